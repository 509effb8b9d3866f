#!/usr/bin/env python
"""Benchmark of the all-pairs test engine on B200 (driver contract: one JSON line).

Metric (BASELINE.json): variable-pairs x samples per second per test
(Pearson, Spearman, chi-squared) at 1/2/4/8 B200.  Homogeneous pairs
P = F(F-1)/2, mixed pairs P = F_C * F_Q, samples = all samples S.

Default workload: config 5 -- the scale run the 1/2/4/8-GPU metric is defined
on (Pearson 20,000 x 10^5 fp64, 30% MCAR, global BH; the largest config and
it fits one B200).  Its Spearman (config 5s, 2000 x 5*10^4) and a chi-squared
(config 3, 500 x 5*10^4) leg run in the same invocation and are reported under
``legs``.  ``--config 1|2|3|4|5s`` measures another config alone.

* value   -- device-resident: inputs already in HBM (N > 1: each rank holds
             its 1/N row shard); one step = [N > 1: NCCL all-gather of the
             input shards] + prepare (validity bits, presort) + the test's
             block over the rank's range + [N > 1: all-gather of the packed
             p cells] + the config's adjustments, all on the device.  CUDA
             events on the launching stream, L2 flushed (512 MiB write)
             between steps outside the events; max over ranks.
* e2e     -- through the public API from host numpy: ``run()`` at N = 1,
             ``dist.sharded_run(..., assemble="owned")`` at N > 1 (each rank
             H2Ds its shard, gets its own rows back); H2D + D2H inside the
             timed region, max over ranks.
* roofline-- dominant kernel, algorithmic bytes/flops per launch / its
             event-timed busy time, against the measured peak.
* cpu_baseline -- the C oracle port (oracle/, OpenMP, all host cores): the
             reference's block kernel timed on a bounded slice of the same
             inputs (triangle rows from row 0), extrapolated by pair count,
             plus the one-off presort for rank tests.

``--impl reference`` times the reference's CPU algorithm (the oracle port; the
reference itself is numba-in-Python and cannot travel) with all host threads,
on the same config dict; under torchrun only rank 0 runs it.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import workloads  # noqa: E402

MEASURED = ROOT / "MEASURED_PEAKS.json"
PROFILES = ROOT / "profiles"

# Roofline bookkeeping per test: (bound, unit, work per pair-sample, kernel name)
ROOF = {
    "pearson": ("tensor", "TFLOP/s", 10.0, "pearson_tile"),      # 5 masked FP64 MACs (DMMA)
    "spearman": ("smem", "GB/s", 24.0, "spearman_walk"),         # 24 B/pair-sample
    "chi2": ("tensor", "TFLOP/s", None, "chi2_gemm"),            # 2 k_g k_h int8 ops
    "anova": ("tensor", "TFLOP/s", None, "group_gemm"),
    "ttest": ("tensor", "TFLOP/s", 8.0, "group_gemm"),
    "kruskal": ("smem", "GB/s", 12.0, "rank_mixed_walk"),
    "mwu": ("smem", "GB/s", 12.0, "rank_mixed_walk"),
}
OUTPUTS = {
    1: ("stat", "p", "p_bonferroni", "p_bh"),
    2: ("rho", "p", "p_bonferroni", "p_bh"),
    3: ("stat", "p", "cramers_v"),
    4: ("stat", "p", "p_bh"),
    5: ("stat", "p", "p_bonferroni", "p_bh"),
    "5s": ("rho", "p", "p_bonferroni", "p_bh"),
}
LEGS = {5: [("5s", "spearman"), (3, "chi2")]}


def parse_config(v: str):
    return v if v == "5s" else int(v)


def load_peaks() -> dict:
    try:
        return json.loads(MEASURED.read_text())
    except Exception:
        return {}


def device_peaks(peaks: dict) -> dict:
    """Peak denominators: measured where the driver measured them, else our
    own microbenchmarks (profiles/peaks_r01.json), else nominal."""
    out = {"hbm_gbs": peaks.get("hbm_gbs", 6650.0), "sm_max_mhz": peaks.get("sm_max_mhz", 1965.0)}
    mb = {}
    for name in ("peaks_r01.json", "peaks_r02.json"):  # later rounds add / override
        f = PROFILES / name
        if f.exists():
            try:
                mb.update(json.loads(f.read_text()))
            except Exception:
                pass
    out["dmma_tflops"] = mb.get("dmma_tflops", 37.0)
    out["imma_tops"] = mb.get("imma_mma_sync_tops", 1127.0)
    out["tcgen05_i8_tops"] = mb.get("tcgen05_i8_tops", 4500.0)  # measured: tools/microbench/tc05_peak.cu
    # the same loop back to back for 4 s: the denominator of a kernel timed inside a long step
    out["tcgen05_i8_tops_sustained"] = mb.get("tcgen05_i8_tops_sustained", out["tcgen05_i8_tops"])
    # SMEM: the measured conflict-free load bandwidth (tools/microbench/
    # smem_peak.cu, profiles/peaks_r02.json), else 148 SMs x 128 B/clk x clock
    if "smem_gbs" in mb:
        out["smem_gbs"], out["smem_source"] = mb["smem_gbs"], "measured (tools/microbench/smem_peak.cu)"
    else:
        out["smem_gbs"] = 148 * 128 * out["sm_max_mhz"] * 1e6 / 1e9
        out["smem_source"] = "derived 148 x 128 B/clk x max clock"
    return out


# ---------------------------------------------------------------- workloads

class Workload:
    """One (config, test) workload as THIS rank sees it: host row shards of
    the inputs (rank r holds rows row_shards(F, world)[r]) plus the metadata
    of the whole matrices.  Config 5 generates only the rank's rows."""

    def __init__(self, cfg_key, test: str, rank: int, world: int):
        from paper_2505_00448_b200 import dist

        self.key, self.test = cfg_key, test
        if cfg_key == 5:
            F, S = 20000, 100000
            _, sh = dist.row_shards(F, world)
            r0, r1 = sh[rank]
            self.a_rows = workloads.config5_rows(F, S, r0, r1)
            self.desc = f"pearson scale {F}x{S} 30% MCAR"
            self.Fa, self.Fb, self.S = F, None, S
            self.kind_a, self.kind_b = "continuous", None
            self.a_full = self.a_rows if world == 1 else None
            self.b_full = None
            self.cat_a = None
        else:
            cfg = workloads.config(cfg_key)
            a, b = cfg["a"], cfg["b"]
            ka, kb = cfg["kind_a"], cfg["kind_b"]
            if test in ("ttest", "mwu"):
                a = np.ascontiguousarray(a[cfg["two_level_rows"]])
                ka = "dichotomous"
            self.desc = cfg["desc"]
            self.kind_a, self.kind_b = ka, kb
            self.a_full, self.b_full = a, b
            self.Fa, self.Fb, self.S = a.shape[0], (b.shape[0] if b is not None else None), a.shape[1]
            self.cat_a = label_counts(a) if ka != "continuous" else None
            _, sh = dist.row_shards(self.Fa, world)
            self.a_rows = a[sh[rank][0]:sh[rank][1]]
        self.b_rows = None
        if self.b_full is not None:
            _, sh = dist.row_shards(self.Fb, world)
            self.b_rows = self.b_full[sh[rank][0]:sh[rank][1]]
        self.r0_a = dist.row_shards(self.Fa, world)[1][rank][0]
        self.r0_b = dist.row_shards(self.Fb, world)[1][rank][0] if self.Fb else 0
        self.outputs = OUTPUTS[cfg_key] if cfg_key != 4 else ("stat", "p", "p_bh")

    @property
    def homogeneous(self) -> bool:
        return self.test in ("pearson", "spearman", "chi2")

    @property
    def pairs(self) -> int:
        if self.homogeneous:
            return self.Fa * (self.Fa - 1) // 2
        return self.Fa * self.Fb

    @property
    def shape(self):
        return (self.Fa, self.Fa) if self.homogeneous else (self.Fa, self.Fb)

    def sharded_inputs(self):
        from paper_2505_00448_b200 import dist

        sa = dist.ShardedInput(self.a_rows, self.r0_a, self.Fa, self.S, self.kind_a, workloads.SENTINEL, self.cat_a)
        sb = None
        if self.b_rows is not None:
            sb = dist.ShardedInput(self.b_rows, self.r0_b, self.Fb, self.S, self.kind_b, workloads.SENTINEL, None)
        return sa, sb

    def datamatrices(self):
        import paper_2505_00448_b200 as ps

        if getattr(self, "_mats", None) is None:
            ma = ps.make_matrix(self.a_full, self.kind_a, na_sentinel=workloads.SENTINEL)
            mb = (ps.make_matrix(self.b_full, self.kind_b, na_sentinel=workloads.SENTINEL)
                  if self.b_full is not None else None)
            self._mats = (ma, mb)
        return self._mats


def default_test(cfg_key) -> str:
    """The (first) test of a config (workloads.config(k)["tests"][0])."""
    return {1: "pearson", 2: "spearman", 3: "chi2", 4: "anova", 5: "pearson", "5s": "spearman"}[cfg_key]


def label_counts(raw: np.ndarray) -> np.ndarray:
    pres = raw != workloads.SENTINEL
    out = np.zeros(raw.shape[0], dtype=np.int64)
    for f in range(raw.shape[0]):
        r = raw[f][pres[f]]
        out[f] = int(r.max()) + 1 if r.size else 0
    return out


def config_dict(wl: Workload, world: int) -> dict:
    """The config object of the JSON line -- identical for both arms."""
    return {"workload": wl.desc, "config": wl.key, "test": wl.test, "pairs": wl.pairs, "samples": wl.S,
            "outputs": list(wl.outputs), "l2": "flushed (512 MiB write) between steps",
            "parallelism": f"pair-shard x{world}"}


# ---------------------------------------------------------------- clocks

class ClockSampler:
    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None
        self.first = 0  # rows before mark() predate the timed region

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms",
                 os.environ.get("PS_BENCH_SMI_MS", "100"),
                 "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def mark(self):
        self.first = len(self.rows)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        self.rows = self.rows[self.first:]
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i - 2] for r in self.rows if len(r) >= 6 for i in range(2, 6)
                          if r[i].lower().startswith("active")})
        loaded = [v for v in sm if mx and v > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- CPU legs

def cpu_baseline(wl: Workload, target_s: float, mat_a, mat_b, t_variant="student"):
    """The reference's block kernel (C oracle port, OpenMP on all host cores)
    on a bounded slice of the workload, extrapolated by pair count.

    Homogeneous tests run triangle rows [0, k) (the longest rows first); mixed
    tests run whole work units (label rows x every feature for ttest / anova,
    continuous features for mwu / kruskal).  The one-off presort of the rank
    tests (engine.py:379-400) is timed separately and added once."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle

    pyoracle.build()
    threads = os.cpu_count() or 1
    test, S = wl.test, wl.S
    prep, run = pyoracle.block_runner(test, mat_a, mat_b, wanted=("stat", "p"), t_variant=t_variant,
                                      threads=threads)
    if wl.homogeneous:
        F = wl.Fa
        units_total, unit_pairs = F, None

        def pairs_of(k):  # off-diagonal pairs of triangle rows [0, k)
            return k * F - k * (k + 1) // 2

        def run_units(k):
            return run(0, k)
    else:
        if test in ("mwu", "kruskal"):
            units_total = wl.Fb

            def pairs_of(k):
                return k * wl.Fa

            def run_units(k):
                return run(0, k)
        else:
            units_total = wl.Fa

            def pairs_of(k):
                return k * wl.Fb

            def run_units(k):
                return run(0, k * wl.Fb)
    # at least one unit per thread: the reference (and the port) parallelise
    # over triangle rows / units, so fewer units would idle cores
    k = min(units_total, threads)
    dt = run_units(k)
    while dt < 0.3 and k < units_total:
        k = min(units_total, k * 2)
        dt = run_units(k)
    rate = pairs_of(k) / dt
    k2 = k
    while k2 < units_total and pairs_of(k2) < rate * target_s:
        k2 = min(units_total, max(k2 + 1, int(k2 * 1.25)))
    if k2 != k:
        dt = run_units(k2)
    total_s = prep + dt * wl.pairs / max(1, pairs_of(k2))
    value = wl.pairs * S / total_s
    what = "triangle rows" if wl.homogeneous else ("continuous features" if test in ("mwu", "kruskal")
                                                   else "label rows")
    sample = (f"{what} [0,{k2}) of {units_total}: {pairs_of(k2)} of {wl.pairs} pairs x {S} samples in {dt:.2f} s"
              + (f" + presort {prep:.2f} s" if prep > 0 else "") + ", extrapolated by pair count")
    return {"value": value, "unit": "pair-samples/s", "cores": threads, "kind": "port", "sample": sample,
            "sample_seconds": dt}


def run_reference_arm(args):
    import paper_2505_00448_b200 as ps  # noqa: F401  (make_matrix, no device use)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    cfg_key = args.config
    test = args.test or default_test(cfg_key)
    wl = Workload(cfg_key, test, 0, 1)
    mat_a, mat_b = wl.datamatrices()
    per_step = float(os.environ.get("REF_STEP_SECONDS", "6"))
    vals, base = [], None
    for i in range(args.warmup + args.steps):
        base = cpu_baseline(wl, per_step, mat_a, mat_b)
        if i >= args.warmup:
            vals.append(base["value"])
    value = statistics.mean(vals)
    base["value"] = value
    legs = {}
    if not args.no_legs:
        for key, t in LEGS.get(cfg_key, []):
            lw = Workload(key, t, 0, 1)
            la, lb = lw.datamatrices()
            b = cpu_baseline(lw, 3.0, la, lb)
            legs[f"{t} (config {key})"] = {"value": b["value"], "unit": "pair-samples/s", "cpu_baseline": b,
                                           "config": config_dict(lw, world)}
    line = {
        "metric": f"pair-samples/s ({test}, config {cfg_key})",
        "impl": "reference",
        "value": value,
        "unit": "pair-samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "dtype": "f64",
        "data": "synthetic (seeded BASELINE recipe, SURVEY 8d; CHRIS cohort unavailable)",
        "config": config_dict(wl, world),
        "cpu_baseline": base,
        "e2e": {"value": value, "unit": "pair-samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "legs": legs,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm

def moments_path(wl: Workload) -> int:
    """Pearson contraction path (library rule, ps_pearson_moments_used): 0 FP64
    DMMA, 1 int8 moments + DMMA Sxy, 2 everything on the int8 tensor cores."""
    from paper_2505_00448_b200 import _lib

    return int(_lib.load().ps_pearson_moments_used(wl.Fa, wl.S))


def roofline_moments(wl: Workload, kern_ms: float, kern_n: int, steps: int, world: int, peaks: dict):
    """The int8 moment contractions of large-F Pearson (ps_moments.cu): 2 moments
    x 8 digits x 2 ops per ORDERED pair-sample, digit expansion included."""
    if not kern_n:
        return None
    launch_ms = kern_ms / steps
    ops = 2 * 8 * 2.0 * wl.Fa * wl.Fa * wl.S / world
    achieved = ops / (launch_ms / 1e3) / 1e12
    peak = peaks["tcgen05_i8_tops"]
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS", "frac": achieved / peak,
            "kernel": "pearson_moments", "launch_ms": launch_ms, "launches_per_step": kern_n / steps,
            "work_per_ordered_pair_sample": "32 int8 ops (tcgen05 kind::i8, 8-digit expansion of x' and x'^2)"}


def roofline(wl: Workload, kern_ms: float, kern_n: int, steps: int, world: int, peaks: dict):
    if not kern_n:
        return None
    test, S = wl.test, wl.S
    bound, unit, per_ps, kname = ROOF[test]
    launch_ms = kern_ms / steps  # kernel busy ms per step (all of its launches)
    units = wl.pairs * S / world
    if test == "chi2":
        ks = wl.cat_a.astype(np.float64)
        per_launch = (ks.sum() ** 2 - (ks * ks).sum()) * S / world  # 2 k_g k_h over g < h
        peak, achieved = peaks["tcgen05_i8_tops"], None
        desc = "2 k_g k_h int8 ops (tcgen05 kind::i8)"
        achieved = per_launch / (launch_ms / 1e3) / 1e12
    elif test == "anova":
        per_launch = 4.0 * float(wl.cat_a.sum()) * wl.Fb * S / world
        peak = peaks["dmma_tflops"]
        achieved = per_launch / (launch_ms / 1e3) / 1e12
        desc = "4 k_g FP64 flops"
    elif test == "pearson" and moments_path(wl) == 2:
        # every contraction on the int8 tensor cores (prof region pearson_moments):
        # Sx, Sxx over ordered pairs (7 + 8 digits x 2 ops), Sxy over the
        # triangle (36 digit products x 2 ops), pair counts (2 ops)
        # (S < 2^17: the symmetric form, 16 sum-plane products + 8 squares)
        F = wl.Fa
        sym = S <= (2 ** 31 - 1) // 16384 and os.environ.get("PS_SXY_SYM", "1")[:1] != "0"
        nxy = 24 if sym else 36
        b256 = S <= (2 ** 31 - 1) // 128 and os.environ.get("PS_MOMENTS_B256", "1")[:1] != "0"
        nmo = 13 if b256 else 15  # moment planes per ordered pair: base 256 (6 + 7) or base 128 (7 + 8)
        ops = (nmo * 2.0 * F * F + (nxy * 2.0 + 2.0) * F * (F + 1) / 2) * S / world
        # a ~1 s phase under the power cap: the sustained microbenchmark figure (burst: 4610)
        peak = peaks["tcgen05_i8_tops_sustained"]
        achieved = ops / (launch_ms / 1e3) / 1e12
        bound, unit = "tensor", "TOPS"
        desc = (f"{2 * (2 * nmo + nxy + 1)} int8 ops per pair-sample (tcgen05 kind::i8 exact digit contractions: "
                + ("Sx, Sy 6 base-256 digits, Sxx, Syy 7" if b256 else "Sx, Sy 7 base-128 digits, Sxx, Syy 8")
                + ", Sxy " + ("16 sum-plane products (D_s + D_t)(D_s + D_t)^T + 8 squares "
                "= the 36 digit products s + t <= 9" if sym else "36 digit products s + t <= 9") + ", n)")
    elif bound == "tensor":
        if test == "pearson" and moments_path(wl) == 1:
            per_ps = 2.0  # Sxy alone on DMMA; Sx, Sxx, Sy, Syy on the int8 tensor cores
        per_launch = per_ps * units
        peak = peaks["dmma_tflops"]
        achieved = per_launch / (launch_ms / 1e3) / 1e12
        desc = f"{per_ps:g} FP64 flops"
        if test == "pearson" and moments_path(wl) == 1:
            desc += " (Sxy on DMMA; masked moments on int8 tcgen05: roofline_moments)"
    else:
        per_launch = per_ps * units
        peak = peaks["smem_gbs"]
        achieved = per_launch / (launch_ms / 1e3) / 1e9
        desc = f"{per_ps:g} B smem ({peaks['smem_source']})"
    traffic = None
    for tf in sorted(PROFILES.glob("traffic_r0*.json"), reverse=True):
        try:
            traffic = json.loads(tf.read_text()).get(f"{wl.key}:{test}")
        except Exception:
            traffic = None
        if traffic is not None:
            break
    out = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
           "traffic": traffic, "kernel": kname, "launch_ms": launch_ms, "launches_per_step": kern_n / steps,
           "work_per_pair_sample": desc}
    if test == "pearson" and moments_path(wl) == 2:
        out["peak_kind"] = ("tcgen05 kind::i8 sustained (tools/microbench/tc05_peak.cu, 4 s back to back; burst "
                            f"{peaks['tcgen05_i8_tops']:.0f} TOPS -> frac {achieved / peaks['tcgen05_i8_tops']:.3f})")
    return out


def _reduce(vals, op):
    import torch
    import torch.distributed as tdist

    dev = "cuda" if tdist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=op)
    return [float(x) for x in t.cpu()]


def reduce_max(vals):
    import torch.distributed as tdist

    return _reduce(vals, tdist.ReduceOp.MAX)


def reduce_sum(vals):
    import torch.distributed as tdist

    return _reduce(vals, tdist.ReduceOp.SUM)


def measure_device(wl: Workload, steps: int, warmup: int, world: int, rank: int, local: int, peaks: dict,
                   clocks=None):
    """Device-resident steps; returns (ms_per_step, roofline, launches, clock summary)."""
    import torch

    import paper_2505_00448_b200 as ps
    from paper_2505_00448_b200 import _lib, blocks, dist

    lib = _lib.load()
    test, S = wl.test, wl.S
    stream = torch.cuda.current_stream()
    dev = torch.device("cuda", local)
    Sp = ((S + 31) // 32) * 32
    ca, _ = dist.row_shards(wl.Fa, world)
    shard_a = dist.upload_rows(wl.a_rows, 0, wl.a_rows.shape[0], ca if world > 1 else wl.Fa, Sp, dev, stream)
    shard_b = None
    if wl.b_rows is not None:
        cb, _ = dist.row_shards(wl.Fb, world)
        shard_b = dist.upload_rows(wl.b_rows, 0, wl.b_rows.shape[0], cb if world > 1 else wl.Fb, Sp, dev, stream)
    blocks.sync(stream)
    ranges = dist.plan(test, wl.Fa, wl.Fb, world)
    lo, hi = ranges[rank]
    shape = wl.shape
    n_canon = 2 + len(ps.EFFECTS_BY_TEST[test])
    outs = [torch.empty(shape, dtype=torch.float64, device=dev) if i < 2 else None for i in range(n_canon)]
    if test == "chi2" and "cramers_v" in wl.outputs:
        outs[3] = torch.empty(shape, dtype=torch.float64, device=dev)
    adj_methods = [m for m, k in (("bonferroni", "p_bonferroni"), ("bh", "p_bh"), ("by", "p_by"))
                   if k in wl.outputs]
    adj_outs = [torch.empty(shape, dtype=torch.float64, device=dev) for _ in adj_methods]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        xa = dist.gather_input(shard_a, wl.Fa)          # NCCL all-gather of the shards (N > 1)
        xb = dist.gather_input(shard_b, wl.Fb) if shard_b is not None else None
        shard_presort = world > 1 and S <= 65535  # sharded tables are 16-bit
        if shard_presort and test == "spearman":
            # each rank presorts 1/world of the features; NCCL all-gathers the tables
            da = blocks.DeviceMatrix(xa, wl.kind_a, workloads.SENTINEL, wl.cat_a, n_samples=S, stream=stream)
            da.presort_sharded(rank, world, stream=stream,
                               gather=lambda name, full, local_: dist.all_gather(full, local_))
        else:
            da = blocks.DeviceMatrix(xa, wl.kind_a, workloads.SENTINEL, wl.cat_a, n_samples=S,
                                     presort=test == "spearman", stream=stream)
        db = None
        if xb is not None:
            rank_walk = test in ("mwu", "kruskal")
            db = blocks.DeviceMatrix(xb, wl.kind_b, workloads.SENTINEL, None, n_samples=S,
                                     presort=rank_walk and not shard_presort, stream=stream)
            if rank_walk and shard_presort:  # the walk only touches this rank's features
                db.presort_rows_only(lo, hi, stream=stream)
        blocks.block(test, da, db, lo, hi, outs, stream=stream)
        if adj_methods:
            dist.exchange_adjust(test, outs[1], shape, ranges, adj_methods, adj_outs, stream)
        da.close()
        if db is not None:
            db.close()

    for _ in range(warmup):
        step()
    blocks.sync(stream)
    torch.cuda.synchronize()
    lib.ps_profile_enable(1)
    _lib.profile_collect(ROOF[test][3])
    _lib.profile_collect("pearson_moments")
    lib.ps_reset_kernel_launches()
    if clocks is not None:
        clocks.mark()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    times = []
    for _ in range(steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        if os.environ.get("PS_BENCH_VERBOSE"):
            print("step ms %.3f" % times[-1], file=sys.stderr)
    blocks.sync(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches = int(lib.ps_kernel_launches())
    clk = clocks.stop() if clocks is not None else None
    lib.ps_profile_enable(0)
    # busy time of the dominant kernel (union over its launches: incremental
    # launches of one step run concurrently on several streams)
    pearson_path = moments_path(wl) if test == "pearson" else 0
    kname = "pearson_moments" if pearson_path == 2 else ROOF[test][3]
    kern_ms, kern_n = _lib.profile_collect_union(kname)
    total_ms = sum(times)
    if world > 1:
        total_ms, kern_ms = reduce_max([total_ms, kern_ms])
    del outs, adj_outs, flush, shard_a, shard_b
    torch.cuda.empty_cache()
    roof = roofline(wl, kern_ms, kern_n, steps, world, peaks)
    if roof is not None and pearson_path == 2:
        roof["kernel"] = "pearson_moments (moment_gemm_mc, cross_gemm_mc)"
    if pearson_path == 1 and roof is not None:
        mom_ms, mom_n = _lib.profile_collect_union("pearson_moments")
        if world > 1:
            mom_ms = reduce_max([mom_ms])[0]
        rm = roofline_moments(wl, mom_ms, mom_n, steps, world, peaks)
        if rm is not None:
            roof["moments"] = rm
    return total_ms / steps, roof, launches, clk


def measure_e2e(wl: Workload, steps: int, warmup: int, world: int):
    """The public API from host numpy: run() (N = 1) or dist.sharded_run with
    each rank's shard (N > 1); max over ranks."""
    import torch

    import paper_2505_00448_b200 as ps
    from paper_2505_00448_b200 import dist

    req = ps.TestRequest(wl.test, wl.outputs)
    if world == 1:
        mat_a, mat_b = wl.datamatrices()

        def call():
            return ps.run(req, mat_a, mat_b)
    else:
        sa, sb = wl.sharded_inputs()

        def call():
            return dist.sharded_run(req, sa, sb, assemble="owned")
    for _ in range(warmup):
        call()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        t1 = time.perf_counter()
        res = call()
        if os.environ.get("PS_BENCH_VERBOSE"):
            print("e2e step ms %.3f" % ((time.perf_counter() - t1) * 1e3), file=sys.stderr)
    dt = (time.perf_counter() - t0) / steps
    d2h = sum(np.asarray(res[n]).nbytes for n in wl.outputs)
    h2d = wl.a_rows.nbytes + (wl.b_rows.nbytes if wl.b_rows is not None else 0)
    if world > 1:
        (dt,) = reduce_max([dt])
        d2h, h2d = reduce_sum([float(d2h), float(h2d)])
    return {"value": wl.pairs * wl.S / dt, "unit": "pair-samples/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": dt * 1e3,
            "api": "run()" if world == 1 else "dist.sharded_run(assemble='owned')"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=parse_config, default=5)
    ap.add_argument("--test", default=None, help="test within a multi-test config (config 4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-legs", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--e2e-warmup", type=int, default=None)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch

    from paper_2505_00448_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one rank per GPU over NCCL; PS_BENCH_BACKEND=gloo + PS_BENCH_DEVICE=0
    # run the N > 1 code path with every rank on one device (a functional
    # check on a one-GPU box -- its timings mean nothing)
    local = int(os.environ.get("PS_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    backend = os.environ.get("PS_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    _lib.check(_lib.load().ps_set_device(local))
    if world > 1:
        import torch.distributed as tdist

        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group(backend)

    cfg_key = args.config
    test = args.test or default_test(cfg_key)
    big = cfg_key == 5
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else (3 if big else 5)
    e2e_warmup = args.e2e_warmup if args.e2e_warmup is not None else (1 if big else 3)
    peaks = device_peaks(load_peaks())

    wl = Workload(cfg_key, test, rank, world)
    # nvidia-smi is started before the warm-up: its start-up (NVML init) can
    # stall this process's CUDA calls for ~15 ms; only rows sampled inside the
    # timed region are kept (mark)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.5)
    ms, roof, launches, clk = measure_device(wl, args.steps, args.warmup, world, rank, local, peaks, clocks)
    value = wl.pairs * wl.S / (ms / 1e3)

    e2e = measure_e2e(wl, e2e_steps, e2e_warmup, world) if e2e_steps > 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        mat_a, mat_b = wl.datamatrices()
        cpu = cpu_baseline(wl, args.cpu_seconds, mat_a, mat_b)
        del mat_a, mat_b
    wl._mats = None

    legs = {}
    if not args.no_legs:
        for key, t in LEGS.get(cfg_key, []):
            lw = Workload(key, t, rank, world)
            lms, lroof, _, _ = measure_device(lw, 3, 3, world, rank, local, peaks)
            legs[f"{t} (config {key})"] = {
                "value": lw.pairs * lw.S / (lms / 1e3), "unit": "pair-samples/s", "ms_per_step": lms,
                "steps": 3, "warmup": 3, "roofline": lroof, "config": config_dict(lw, world)}

    if rank == 0:
        line = {
            "metric": f"pair-samples/s ({test}, config {cfg_key})",
            "value": value,
            "unit": "pair-samples/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": ("u8/i32" if test == "chi2" else
                      "i8/i32 -> f64 (exact digit contractions)" if test == "pearson" and moments_path(wl) == 2
                      else "f64"),
            "data": "synthetic (seeded BASELINE recipe, SURVEY 8d; CHRIS cohort unavailable)",
            "config": config_dict(wl, world),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "legs": legs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
