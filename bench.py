#!/usr/bin/env python
"""Benchmark of the all-pairs test engine on B200 (driver contract: one JSON line).

Metric (BASELINE.json): variable-pairs x samples per second for one test on one
BASELINE config; homogeneous pairs P = F(F-1)/2, mixed pairs P = F_C * F_Q,
samples = all samples S.  Default workload: configs[1] (config 2, Spearman
1000 x 10^4), the config the metric is quoted on.

* value   -- device-resident: inputs already in HBM; one step = prepare
             (validity bits, presort) + the test's block over the full range +
             the config's adjustments, all on the device.  CUDA events on the
             launching stream, L2 flushed (512 MiB write) between steps outside
             the events; max over ranks.
* e2e     -- the public API ``run(TestRequest, DataMatrix)`` from host numpy
             inputs to host ResultSet (H2D + D2H inside the timed region).
* roofline-- dominant kernel, algorithmic bytes/flops per launch / its
             event-timed duration, against the measured peak.
* cpu_baseline -- the C oracle port (oracle/, OpenMP, all host cores) on a
             bounded slice of the same inputs.

``--impl reference`` times the reference's CPU algorithm (the oracle port; the
reference itself is numba-in-Python and cannot travel) with all host threads.
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
    f = PROFILES / "peaks_r01.json"
    if f.exists():
        try:
            mb = json.loads(f.read_text())
        except Exception:
            mb = {}
    out["dmma_tflops"] = mb.get("dmma_tflops", 37.0)
    out["imma_tops"] = mb.get("imma_mma_sync_tops", 1127.0)
    out["tcgen05_i8_tops"] = mb.get("tcgen05_i8_tops", 4500.0)  # measured: tools/microbench/tc05_peak.cu
    # SMEM crossbar: 148 SMs x 128 B/clk at the max SM clock
    out["smem_gbs"] = 148 * 128 * out["sm_max_mhz"] * 1e6 / 1e9
    return out


def pair_count(cfg: dict, test: str) -> int:
    if test in ("pearson", "spearman", "chi2"):
        F = cfg["F"]
        return F * (F - 1) // 2
    rows = cfg["two_level_rows"].size if test in ("ttest", "mwu") else cfg["F"]
    return rows * cfg["Fq"]


def label_counts(raw: np.ndarray) -> np.ndarray:
    pres = raw != workloads.SENTINEL
    out = np.zeros(raw.shape[0], dtype=np.int64)
    for f in range(raw.shape[0]):
        r = raw[f][pres[f]]
        out[f] = int(r.max()) + 1 if r.size else 0
    return out


def build_inputs(cfg: dict, test: str):
    """Host raw matrices (a, b) for `test`, plus kinds and category counts."""
    a, b = cfg["a"], cfg["b"]
    if test in ("ttest", "mwu"):
        a = np.ascontiguousarray(a[cfg["two_level_rows"]])
        return a, b, "dichotomous", "continuous"
    return a, b, cfg["kind_a"], cfg["kind_b"]


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
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100",
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

def cpu_baseline(cfg: dict, test: str, target_s: float, mat_a, mat_b, t_variant="student"):
    """Oracle port (C + OpenMP, all host cores) on a bounded slice of rows."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle

    pyoracle.build()
    threads = os.cpu_count() or 1
    S = mat_a.n_samples
    if test in ("pearson", "spearman", "chi2"):
        F = mat_a.n_features
        total_pairs = F * (F - 1) // 2

        def slice_pairs(k):  # rows [0, k) of the triangle, off-diagonal pairs
            return k * F - k * (k + 1) // 2

        def run_rows(k):
            t0 = time.perf_counter()
            pyoracle.compute(test, mat_a, None, wanted={"stat", "p"}, threads=threads, lo=0, hi=k)
            return time.perf_counter() - t0

        k = max(1, F // 100)
        dt = run_rows(k)
        while dt < 0.5 and k < F:
            k = min(F, k * 4)
            dt = run_rows(k)
        rate = slice_pairs(k) * S / dt
        k2 = k
        want_pairs = rate * target_s / S
        while k2 < F and slice_pairs(k2) < want_pairs:
            k2 += max(1, F // 200)
        k2 = min(k2, F)
        dt = run_rows(k2)
        pairs = slice_pairs(k2)
        sample = f"triangle rows [0,{k2}) of {F}: {pairs} of {total_pairs} pairs x {S} samples"
    else:
        Fq = mat_b.n_features
        rows = mat_a.n_features
        per_unit = rows  # pairs per continuous feature (mwu/kruskal) or per grid row

        def run_units(u):
            t0 = time.perf_counter()
            if test in ("mwu", "kruskal"):
                pyoracle.compute(test, mat_a, mat_b, wanted={"stat", "p"}, threads=threads, lo=0, hi=u)
            else:
                pyoracle.compute(test, mat_a, mat_b, wanted={"stat", "p"}, threads=threads, lo=0,
                                 hi=u * Fq, t_variant=t_variant)
            return time.perf_counter() - t0

        units_total = Fq if test in ("mwu", "kruskal") else rows
        u = max(1, units_total // 100)
        dt = run_units(u)
        while dt < 0.5 and u < units_total:
            u = min(units_total, u * 4)
            dt = run_units(u)
        pairs_u = per_unit if test in ("mwu", "kruskal") else Fq
        rate = u * pairs_u * S / dt
        u2 = min(units_total, max(u, int(rate * target_s / (pairs_u * S))))
        dt = run_units(u2)
        pairs = u2 * pairs_u
        sample = f"{u2} of {units_total} work units: {pairs} pairs x {S} samples"
    value = pairs * S / dt
    return {"value": value, "unit": "pair-samples/s", "cores": threads, "kind": "port",
            "sample": sample + f" ({dt:.1f} s)"}


def run_reference_arm(args, cfg, test):
    import paper_2505_00448_b200 as ps

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    a, b, ka, kb = build_inputs(cfg, test)
    mat_a = ps.make_matrix(a, ka, na_sentinel=workloads.SENTINEL)
    mat_b = ps.make_matrix(b, kb, na_sentinel=workloads.SENTINEL) if b is not None else None
    per_step = float(os.environ.get("REF_STEP_SECONDS", "6"))
    vals = []
    base = None
    for i in range(args.warmup + args.steps):
        base = cpu_baseline(cfg, test, per_step, mat_a, mat_b)
        if i >= args.warmup:
            vals.append(base["value"])
    value = statistics.mean(vals)
    base["value"] = value
    line = {
        "metric": f"pair-samples/s ({test}, config {args.config})",
        "impl": "reference",
        "value": value,
        "unit": "pair-samples/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "dtype": "f64",
        "data": "synthetic (seeded BASELINE recipe, SURVEY 8d)",
        "config": {"workload": cfg["desc"], "config": args.config, "test": test},
        "cpu_baseline": base,
        "e2e": {"value": value, "unit": "pair-samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=parse_config, default=2)
    ap.add_argument("--test", default=None, help="test within a multi-test config (config 4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--e2e-warmup", type=int, default=3)
    args = ap.parse_args()

    cfg = workloads.config(args.config)
    test = args.test or cfg["tests"][0]
    if args.impl == "reference":
        run_reference_arm(args, cfg, test)
        return

    import torch
    import paper_2505_00448_b200 as ps
    from paper_2505_00448_b200 import _lib, blocks, dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    _lib.check(_lib.load().ps_set_device(local))
    if world > 1:
        import torch.distributed as tdist

        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))

    a, b, ka, kb = build_inputs(cfg, test)
    sentinel = workloads.SENTINEL
    S = a.shape[1]
    cat_a = label_counts(a) if ka != "continuous" else None
    outputs = OUTPUTS[args.config]
    if args.config == 4:
        outputs = ("stat", "p", "p_bh")
    P = pair_count(cfg, test)
    work_units = P * S
    peaks = device_peaks(load_peaks())

    stream = torch.cuda.current_stream()
    Sp = ((S + 31) // 32) * 32

    def to_dev(x):
        t = torch.zeros((x.shape[0], Sp), dtype=torch.float64, device="cuda")
        t[:, :S] = torch.from_numpy(x)
        return t

    xa = to_dev(a)
    xb = to_dev(b) if b is not None else None
    plan = dist.plan(test, a.shape[0], None if b is None else b.shape[0], world)
    lo, hi = plan[rank]
    homog = test in ("pearson", "spearman", "chi2")
    shape = (a.shape[0], a.shape[0]) if homog else (a.shape[0], b.shape[0])
    n_canon = 2 + len(ps.EFFECTS_BY_TEST[test])
    want = {"stat"} | {"p"}
    outs = [torch.empty(shape, dtype=torch.float64, device="cuda") if i < 2 else None
            for i in range(n_canon)]
    adj_methods = [m for m, k in (("bonferroni", "p_bonferroni"), ("bh", "p_bh"), ("by", "p_by"))
                   if k in outputs]
    if test == "chi2":
        outs[3] = torch.empty(shape, dtype=torch.float64, device="cuda")  # cramers_v
    adj_out = torch.empty(shape, dtype=torch.float64, device="cuda") if adj_methods else None
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    del want

    def step():
        if world > 1 and test == "spearman":
            # each rank presorts 1/world of the features; NCCL all-gathers the tables
            da = blocks.DeviceMatrix(xa, ka, sentinel, cat_a, n_samples=S, stream=stream)
            da.presort_sharded(rank, world, stream=stream)
        else:
            da = blocks.DeviceMatrix(xa, ka, sentinel, cat_a, n_samples=S,
                                     presort=test == "spearman", stream=stream)
        db = None
        if xb is not None:
            rank_walk = test in ("mwu", "kruskal")
            db = blocks.DeviceMatrix(xb, kb, sentinel, None, n_samples=S,
                                     presort=rank_walk and world == 1, stream=stream)
            if rank_walk and world > 1:  # the walk only touches this rank's features
                db.presort_rows_only(lo, hi, stream=stream)
        blocks.block(test, da, db, lo, hi, outs, stream=stream)
        if adj_methods:
            dist.adjust_gathered(test, outs[1], shape, plan, adj_methods, adj_out, stream)
        da.close()
        if db is not None:
            db.close()

    lib = _lib.load()
    # nvidia-smi is started before the warm-up: its start-up (NVML init) can
    # stall this process's CUDA calls for ~15 ms; only rows sampled inside the
    # timed region are kept (mark)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.5)
    for _ in range(args.warmup):
        step()
    blocks.sync(stream)
    torch.cuda.synchronize()
    lib.ps_profile_enable(1)
    _lib.profile_collect(ROOF[test][3])
    lib.ps_reset_kernel_launches()
    clocks.mark()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
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
    clk = clocks.stop()
    lib.ps_profile_enable(0)
    # busy time of the dominant kernel (union over its launches: incremental
    # launches of one step run concurrently on several streams)
    kern_ms, kern_n = _lib.profile_collect_union(ROOF[test][3])
    total_ms = sum(times)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = work_units / (ms_per_step / 1e3)

    # ---------------- roofline of the dominant kernel
    bound, unit, per_ps, _kname = ROOF[test]
    roof = None
    if kern_n:
        launch_ms = kern_ms / args.steps  # kernel busy ms per step (all of its launches)
        units_per_launch = work_units / world
        if test == "chi2":
            ks = cat_a
            ksum = float(ks.sum())
            per_launch = 2.0 * (ksum * ksum - float((ks * ks).sum())) / 2.0 * S / world
            peak = peaks["tcgen05_i8_tops"]
            achieved = per_launch / (launch_ms / 1e3) / 1e12
            per_ps_desc = "2 k_g k_h int8 ops (tcgen05 kind::i8)"
        elif test == "anova":
            ksum = float(cat_a.sum())
            per_launch = 4.0 * ksum * b.shape[0] * S / world
            peak = peaks["dmma_tflops"]
            achieved = per_launch / (launch_ms / 1e3) / 1e12
            per_ps_desc = "4 k_g FP64 flops"
        elif bound == "tensor":
            per_launch = per_ps * units_per_launch
            peak = peaks["dmma_tflops"]
            achieved = per_launch / (launch_ms / 1e3) / 1e12
            per_ps_desc = f"{per_ps:g} FP64 flops"
        else:
            per_launch = per_ps * units_per_launch
            peak = peaks["smem_gbs"]
            achieved = per_launch / (launch_ms / 1e3) / 1e9
            per_ps_desc = f"{per_ps:g} B smem"
        traffic = None
        tf = PROFILES / "traffic_r01.json"
        if tf.exists():
            try:
                traffic = json.loads(tf.read_text()).get(f"{args.config}:{test}")
            except Exception:
                traffic = None
        roof = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                "frac": achieved / peak, "traffic": traffic, "kernel": ROOF[test][3],
                "launch_ms": launch_ms, "launches_per_step": kern_n / args.steps,
                "work_per_pair_sample": per_ps_desc}

    # ---------------- end to end through run()
    e2e = None
    if rank == 0 and world == 1 and args.e2e_steps > 0:
        mat_a = ps.make_matrix(a, ka, na_sentinel=sentinel)
        mat_b = ps.make_matrix(b, kb, na_sentinel=sentinel) if b is not None else None
        req = ps.TestRequest(test, outputs)
        for _ in range(args.e2e_warmup):  # warm-up (pool growth, first-touch of the pinned ring)
            ps.run(req, mat_a, mat_b)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            t1 = time.perf_counter()
            res = ps.run(req, mat_a, mat_b)
            if os.environ.get("PS_BENCH_VERBOSE"):
                print("e2e step ms %.3f" % ((time.perf_counter() - t1) * 1e3), file=sys.stderr)
        dt = (time.perf_counter() - t0) / args.e2e_steps
        h2d = a.nbytes + (b.nbytes if b is not None else 0)
        d2h = sum(res[n].nbytes for n in outputs)
        e2e = {"value": work_units / dt, "unit": "pair-samples/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": dt * 1e3}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        mat_a = ps.make_matrix(a, ka, na_sentinel=sentinel)
        mat_b = ps.make_matrix(b, kb, na_sentinel=sentinel) if b is not None else None
        cpu = cpu_baseline(cfg, test, args.cpu_seconds, mat_a, mat_b)

    if rank == 0:
        line = {
            "metric": f"pair-samples/s ({test}, config {args.config})",
            "value": value,
            "unit": "pair-samples/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64" if test != "chi2" else "u8/i32",
            "data": "synthetic (seeded BASELINE recipe, SURVEY 8d; CHRIS cohort unavailable)",
            "config": {"workload": cfg["desc"], "config": args.config, "test": test,
                       "pairs": P, "samples": S, "outputs": list(outputs),
                       "l2": "flushed (512 MiB write) between steps",
                       "parallelism": f"pair-shard x{world}"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
