"""Multi-GPU sharding: one process per GPU, pairs partitioned, no host round trips.

The reference parallelises by static, disjoint pair ranges over threads
(``engine.py:70-125`` partitions, ``:360-376`` dispatch); cells are
independent, so results never depend on the partition (``SPEC.md:469``).
Here the same ranges are handed to ranks (``torch.distributed``: NCCL over
NVLink on GPUs, gloo in the CPU tests) and every exchange stays on the device:

* **input** -- rank r uploads only its 1/N row shard of each host matrix
  (pinned all-core staging, ``ps_copy_h2d_2d``) and the ranks all-gather the
  shards over NVLink into the full device matrix ("each GPU
  H2D's 1/8 over its own PCIe link, then ncclAllGather");
* **presort** (Spearman) -- each rank presorts 1/N of the features and the
  tables are all-gathered (``blocks.DeviceMatrix.presort_sharded``);
* **p-values** -- each rank packs the family cells of its range
  (``ps_cells_pack``: 8 bytes per owned cell, half an all-reduce of dense
  matrices), the ranks all-gather the vectors, every rank adjusts the whole
  family on its device (BH / BY / Bonferroni) and unpacks its own segment;
* **results** -- ``assemble="full"`` all-gathers the packed raw / adjusted
  cells so every rank holds the full matrices; ``assemble="owned"`` returns
  each rank's own rows only (1/N of the device-to-host bytes per rank).

Determinism: a cell's k-order never depends on the range that computes it
(split-K factors are functions of the whole matrices), and BH / BY /
Bonferroni are order-insensitive, so 1/2/4/8-GPU results are bitwise equal.
"""

from __future__ import annotations

import ctypes
import math
from typing import Callable

import numpy as np

HOMOGENEOUS = ("pearson", "spearman", "chi2")


def partition_range(count: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous near-equal chunks (engine.py:70-90)."""
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    base, extra = divmod(count, parts)
    out, lo = [], 0
    for w in range(parts):
        hi = lo + base + (1 if w < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def partition_triangle_rows(n: int, parts: int) -> list[tuple[int, int]]:
    """Row ranges with near-equal upper-triangle pair counts (engine.py:93-125)."""
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    total = n * (n + 1) // 2
    out, cum, row = [], 0, 0
    for w in range(1, parts):
        lo = row
        while row < n and (cum + n - row) * parts <= total * w:
            cum += n - row
            row += 1
        out.append((lo, row))
    out.append((row, n))
    return out


def plan(test: str, n_a: int, n_b: int | None, world: int) -> list[tuple[int, int]]:
    """Per-rank work ranges in the reference's units for `test`."""
    if test in HOMOGENEOUS:
        return partition_triangle_rows(n_a, world)
    if test in ("ttest", "anova"):
        return partition_range(n_a * n_b, world)
    return partition_range(n_b, world)


def row_shards(n_rows: int, world: int) -> tuple[int, list[tuple[int, int]]]:
    """Equal input row shards for the all-gather: (rows per shard c, [(r0, r1)]);
    the last shards may be short or empty (padded to c rows on the device)."""
    c = max(1, -(-n_rows // world))
    return c, [(min(n_rows, r * c), min(n_rows, (r + 1) * c)) for r in range(world)]


def owned_mask(test: str, shape: tuple[int, int], lo: int, hi: int) -> np.ndarray:
    """Cells a rank writes for its range (both triangles for homogeneous tests)."""
    rows, cols = shape
    m = np.zeros(shape, dtype=bool)
    if test in HOMOGENEOUS:
        g = np.arange(rows)[:, None]
        h = np.arange(cols)[None, :]
        up = (g >= lo) & (g < hi) & (h >= g)
        m |= up
        m |= up.T
    elif test in ("ttest", "anova"):
        flat = m.reshape(-1)
        flat[lo:hi] = True
    else:
        m[:, lo:hi] = True
    return m


def owned_block(test: str, shape: tuple[int, int], lo: int, hi: int) -> tuple[slice, slice]:
    """The (rows, cols) block of the result matrix that holds a rank's cells."""
    rows, cols = shape
    if test in HOMOGENEOUS:
        return slice(lo, hi), slice(0, cols)
    if test in ("ttest", "anova"):
        return (slice(lo // cols, -(-hi // cols)) if hi > lo else slice(0, 0)), slice(0, cols)
    return slice(0, rows), slice(lo, hi)


def _world():
    import torch.distributed as tdist

    if tdist.is_available() and tdist.is_initialized():
        return tdist, tdist.get_world_size(), tdist.get_rank()
    return None, 1, 0


def all_gather(out, inp) -> None:
    """``out`` (world x n) <- every rank's ``inp`` (n); NCCL moves device
    tensors over NVLink, gloo (CPU tests) goes through host copies."""
    tdist, world, _ = _world()
    if world == 1:
        out.copy_(inp.reshape(out.shape))
        return
    if tdist.get_backend() == "nccl":
        tdist.all_gather_into_tensor(out, inp)
        return
    # gloo: flat host buffers (its all-gather wants matching 1-D chunks)
    o = out.detach().cpu().reshape(-1) if out.is_cuda else out.reshape(-1)
    tdist.all_gather_into_tensor(o, inp.detach().cpu().reshape(-1).contiguous())
    if out.is_cuda or o.data_ptr() != out.data_ptr():
        out.copy_(o.view(out.shape))


# --------------------------------------------------------------------------
# device-side exchanges (C ABI ps_cells_* ; no host round trips)

def cells_count(test: str, diag: bool, shape, lo: int, hi: int) -> int:
    from . import _lib

    n = ctypes.c_int64(0)
    _lib.check(_lib.load().ps_cells_count(_lib.TEST_CODES[test], 1 if diag else 0, shape[0], shape[1], lo, hi,
                                          ctypes.byref(n)))
    return int(n.value)


def _pack(test, diag, mat, shape, lo, hi, vec, stream):
    from . import _lib
    from .blocks import _ptr, _stream_ptr

    _lib.check(_lib.load().ps_cells_pack(_lib.TEST_CODES[test], 1 if diag else 0, _ptr(mat), shape[0], shape[1],
                                         lo, hi, _ptr(vec), _stream_ptr(stream)))


def _unpack(test, diag, vec, shape, lo, hi, mat, stream):
    from . import _lib
    from .blocks import _ptr, _stream_ptr

    _lib.check(_lib.load().ps_cells_unpack(_lib.TEST_CODES[test], 1 if diag else 0, _ptr(vec), shape[0], shape[1],
                                           lo, hi, _ptr(mat), _stream_ptr(stream)))


def _gather_cells(test, diag, mat, shape, ranges, rank, stream):
    """Pack this rank's cells, all-gather every rank's vector (padded to the
    longest with NaN): returns (gathered (world, n_max) tensor, counts)."""
    import torch

    from . import blocks

    counts = [cells_count(test, diag, shape, lo, hi) for lo, hi in ranges]
    nmax = max(1, max(counts))
    lo, hi = ranges[rank]
    local = torch.full((nmax,), math.nan, dtype=torch.float64, device=mat.device)
    _pack(test, diag, mat, shape, lo, hi, local, stream)
    gathered = torch.empty((len(ranges), nmax), dtype=torch.float64, device=mat.device)
    blocks.sync(stream)  # packed before the collective (on its own stream) reads it
    all_gather(gathered, local)
    return gathered, counts


def exchange_adjust(test: str, p, shape, ranges, methods, outs, stream=None) -> None:
    """The global BH / BY / Bonferroni of a sharded p matrix.

    ``p`` holds this rank's cells (device, rows x cols); ``outs[k]`` receives
    the adjusted values of this rank's cells for ``methods[k]`` (mirrored,
    NaN diagonal).  NaN padding of the gathered vectors is not part of any
    family (adjust.py:30-31 drops NaN), so the padded vector adjusts exactly
    as the reference's family."""
    import torch

    from . import blocks

    tdist, world, rank = _world()
    if world == 1:
        for m, o in zip(methods, outs):
            blocks.adjust_device(p, shape[0], shape[1], m, test in HOMOGENEOUS, o, stream)
        return
    gathered, _ = _gather_cells(test, False, p, shape, ranges, rank, stream)
    nmax = gathered.shape[1]
    lo, hi = ranges[rank]
    adj = torch.empty_like(gathered)
    for m, o in zip(methods, outs):
        blocks.adjust_family_device(gathered, gathered.numel(), m, adj, stream)
        _unpack(test, False, adj.view(-1)[rank * nmax:], shape, lo, hi, o, stream)


def gather_full(test: str, mat, shape, ranges, diag: bool = True, stream=None) -> None:
    """In place: every rank's cells of ``mat`` (device) from their owners."""
    tdist, world, rank = _world()
    if world == 1:
        return
    gathered, _ = _gather_cells(test, diag, mat, shape, ranges, rank, stream)
    for r, (lo, hi) in enumerate(ranges):
        if r != rank:
            _unpack(test, diag, gathered[r], shape, lo, hi, mat, stream)


def upload_rows(values: np.ndarray, r0: int, r1: int, c: int, ld: int, device, stream=None):
    """Host rows [r0, r1) -> a zero-padded (c, ld) device tensor (pinned staging)."""
    import torch

    from . import _lib
    from .blocks import _stream_ptr

    t = torch.zeros((c, ld), dtype=torch.float64, device=device)
    if r1 > r0:
        src = np.ascontiguousarray(values[r0:r1], dtype=np.float64)
        _lib.check(_lib.load().ps_copy_h2d_2d(t.data_ptr(), ld * 8, src.ctypes.data, src.shape[1] * 8,
                                              src.shape[1] * 8, r1 - r0, _stream_ptr(stream)))
    return t


def gather_input(shard, n_rows: int):
    """All-gather the per-rank (c, ld) shards into the full (n_rows, ld) matrix."""
    import torch

    _, world, _ = _world()
    c, ld = shard.shape
    if world == 1:
        return shard[:n_rows]
    full = torch.empty((c * world, ld), dtype=shard.dtype, device=shard.device)
    all_gather(full, shard)
    return full[:n_rows]


# --------------------------------------------------------------------------
# the sharded run

class ShardedInput:
    """One rank's view of an input matrix: its own rows [r0, r1) of the host
    values (the rest lives on the other ranks), plus what ``make_matrix``
    knows about the whole matrix.  ``DataMatrix`` inputs are sharded on the
    fly; a ShardedInput lets a rank never materialise the full 16 GB host
    matrix (bench config 5)."""

    def __init__(self, rows: np.ndarray, r0: int, n_features: int, n_samples: int, kind: str,
                 na_sentinel: float = math.nan, category_counts: np.ndarray | None = None):
        self.rows = rows
        self.r0 = r0
        self.n_features = n_features
        self.n_samples = n_samples
        self.kind = kind
        self.na_sentinel = na_sentinel
        self.category_counts = category_counts

    @classmethod
    def from_datamatrix(cls, mat, rank: int, world: int) -> "ShardedInput":
        _, sh = row_shards(mat.n_features, world)
        r0, r1 = sh[rank]
        return cls(mat.values[r0:r1], r0, mat.n_features, mat.n_samples, mat.kind, mat.na_sentinel,
                   mat.category_counts)


def device_inputs(inputs, stream=None):
    """Upload each rank's shard and all-gather: {name: full device tensor}."""
    import torch

    _, world, rank = _world()
    out = []
    for x in inputs:
        if x is None:
            out.append(None)
            continue
        c, sh = row_shards(x.n_features, world)
        r0, r1 = sh[rank]
        assert r0 == x.r0 and r1 - r0 == x.rows.shape[0], "shard does not match the rank's rows"
        ld = -(-x.n_samples // 32) * 32
        dev = torch.device("cuda", torch.cuda.current_device())
        shard = upload_rows(x.rows, 0, r1 - r0, c, ld, dev, stream)
        from . import blocks

        blocks.sync(stream)
        out.append(gather_input(shard, x.n_features))
    return out


def device_compute(request, a_dev, b_dev, a_meta, b_meta, ranges, wanted, stream=None, rank=None, world=None):
    """This rank's block on the full device inputs: {name: device matrix}
    holding the rank's cells (NaN elsewhere).  ``rank``/``world`` default to
    the process group's; a single-process run passes its shard index and
    presorts whole (no collective)."""
    import torch

    from . import blocks
    from .datamodel import EFFECTS_BY_TEST

    if rank is None:
        tdist, world, rank = _world()
        group = True
    else:
        group = False
    test = request.test
    lo, hi = ranges[rank]
    canonical = ("stat", "p") + EFFECTS_BY_TEST[test]
    shape = (a_meta.n_features, a_meta.n_features if b_meta is None else b_meta.n_features)
    S = a_meta.n_samples
    # sharded presort tables are 16-bit (S <= 65535); wider inputs presort whole
    sharded = group and world > 1 and S <= 65535
    da = blocks.DeviceMatrix(a_dev, a_meta.kind, a_meta.na_sentinel, a_meta.category_counts, n_samples=S,
                             presort=test == "spearman" and not sharded, stream=stream)
    if test == "spearman" and sharded:  # 1/world of the presort per rank + all-gather
        da.presort_sharded(rank, world, stream=stream, gather=lambda name, full, local: all_gather(full, local))
    db = None
    if b_dev is not None:
        walk = test in ("mwu", "kruskal")
        db = blocks.DeviceMatrix(b_dev, b_meta.kind, b_meta.na_sentinel, None, n_samples=S,
                                 presort=walk and not sharded, stream=stream)
        if walk and sharded:  # the walk only touches features [lo, hi)
            db.presort_rows_only(lo, hi, stream=stream)
    outs = [torch.full(shape, math.nan, dtype=torch.float64, device=a_dev.device) if n in wanted else None
            for n in canonical]
    blocks.block(test, da, db, lo, hi, outs, t_variant=request.t_variant, u_mode=request.u_mode, stream=stream)
    blocks.sync(stream)
    da.close()
    if db is not None:
        db.close()
    return {n: o for n, o in zip(canonical, outs) if o is not None}


def sharded_run(request, mat_a, mat_b=None, compute: Callable | None = None, adjust_fn: Callable | None = None,
                assemble: str = "full"):
    """Run one request across the ranks of the current process group.

    ``mat_a`` / ``mat_b`` are ``DataMatrix`` objects (every rank uploads only
    its row shard) or :class:`ShardedInput` shards.  ``assemble="full"``
    returns the full result matrices on every rank (a ``ResultSet``);
    ``"owned"`` returns ``{name: block}`` with this rank's block of each
    matrix (``owned_block(...)``; cells other ranks own are NaN).

    ``compute(test, mat_a, mat_b, lo, hi, wanted)`` (CPU tests: the oracle)
    replaces the device path with a host one: it returns full NaN-prefilled
    host matrices with this rank's cells filled, gathered over the group.
    """
    from .datamodel import EFFECTS_BY_TEST, ResultSet
    from .engine import ADJUSTED_OUTPUTS, validate

    test = request.test
    sharded_in = isinstance(mat_a, ShardedInput)
    if not sharded_in:
        shape = validate(request, mat_a, mat_b)
    else:
        shape = (mat_a.n_features, mat_a.n_features if mat_b is None else mat_b.n_features)
    tdist, world, rank = _world()
    ranges = plan(test, mat_a.n_features, None if mat_b is None else mat_b.n_features, world)
    lo, hi = ranges[rank]
    canonical = ("stat", "p") + EFFECTS_BY_TEST[test]
    needed = {n for n in request.outputs if n not in ADJUSTED_OUTPUTS}
    adj_names = [n for n in request.outputs if n in ADJUSTED_OUTPUTS]
    if adj_names:
        needed.add("p")
    if compute is not None:
        return _host_sharded(request, mat_a, mat_b, compute, adjust_fn, shape, ranges, needed, canonical)

    import torch

    from . import _lib

    _lib.require_device()
    stream = torch.cuda.current_stream()
    sa = mat_a if sharded_in else ShardedInput.from_datamatrix(mat_a, rank, world)
    sb = None
    if mat_b is not None:
        sb = mat_b if sharded_in else ShardedInput.from_datamatrix(mat_b, rank, world)
    a_dev, b_dev = device_inputs([sa, sb], stream)
    raw = device_compute(request, a_dev, b_dev, sa, sb, ranges, needed, stream)
    del a_dev, b_dev
    adj = {}
    if adj_names:
        outs = [torch.full(shape, math.nan, dtype=torch.float64, device=raw["p"].device) for _ in adj_names]
        exchange_adjust(test, raw["p"], shape, ranges, [ADJUSTED_OUTPUTS[n] for n in adj_names], outs, stream)
        adj = dict(zip(adj_names, outs))
    result = {}
    if assemble == "owned":
        blk = owned_block(test, shape, lo, hi)
        for name in request.outputs:
            t = adj[name] if name in adj else raw[name]
            result[name] = t[blk].cpu().numpy()
        return result
    for name in request.outputs:
        t = adj[name] if name in adj else raw[name]
        gather_full(test, t, shape, ranges, diag=name not in adj, stream=stream)
        result[name] = t.cpu().numpy()
    torch.cuda.synchronize()
    return ResultSet(matrices=result, shape=shape)


def _host_sharded(request, mat_a, mat_b, compute, adjust_fn, shape, ranges, needed, canonical):
    """Host flavour of the exchange for injected CPU compute (gloo tests):
    owned cells SUM-all-reduced (x + 0.0 == x, NaN stays NaN)."""
    import torch

    from .engine import ADJUSTED_OUTPUTS

    tdist, world, rank = _world()
    test = request.test
    lo, hi = ranges[rank]
    raw = compute(test, mat_a, mat_b, lo, hi, needed)
    own = owned_mask(test, shape, lo, hi)
    full = {}
    for name in canonical:
        if name not in needed:
            continue
        t = torch.from_numpy(np.where(own, raw[name], 0.0))
        if world > 1:
            tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
        full[name] = t.numpy()
    if adjust_fn is None:
        from .adjust import adjust as adjust_fn  # device adjustment
    out = {}
    for name in request.outputs:
        if name in ADJUSTED_OUTPUTS:
            out[name] = adjust_fn(full["p"], ADJUSTED_OUTPUTS[name], test in HOMOGENEOUS)
        else:
            out[name] = full[name]
    return out


# --------------------------------------------------------------------------
# one process, several local GPUs (TestRequest.devices)

def local_run(request, mat_a, mat_b, devices):
    """``run()`` sharded over local GPUs from one process: one host thread per
    device (the library locks per device, so the devices run concurrently).

    Shard r uploads its 1/N rows of each input, the full device inputs are
    assembled from the shards by peer copies (NVLink), shard r computes the
    reference partition ranges[r] of the pairs, packs its p family cells and
    raw outputs (``ps_cells_pack``), and the first device gathers the packed
    vectors (peer copies), adjusts the whole family once and unpacks every
    segment into the full result matrices, which it copies to the host.
    Bitwise identical to the one-device run (partition-independent k-order,
    order-insensitive adjustment).
    """
    import threading

    import torch

    from . import _lib, blocks
    from .datamodel import EFFECTS_BY_TEST, ResultSet
    from .engine import ADJUSTED_OUTPUTS, validate

    shape = validate(request, mat_a, mat_b)
    test = request.test
    n = len(devices)
    ranges = plan(test, mat_a.n_features, None if mat_b is None else mat_b.n_features, n)
    canonical = ("stat", "p") + EFFECTS_BY_TEST[test]
    adj_names = [x for x in request.outputs if x in ADJUSTED_OUTPUTS]
    needed = {x for x in request.outputs if x not in ADJUSTED_OUTPUTS}
    if adj_names:
        needed.add("p")
    raw_names = [x for x in canonical if x in needed]
    S = mat_a.n_samples
    ld = -(-S // 32) * 32
    mats = [mat_a] + ([mat_b] if mat_b is not None else [])
    shards = [[None] * len(mats) for _ in range(n)]
    packs = [None] * n
    errors = [None] * n
    barrier = threading.Barrier(n)
    lib = _lib.load()

    def worker(r):
        try:
            dev = devices[r]
            torch.cuda.set_device(dev)
            _lib.check(lib.ps_set_device(dev))
            stream = torch.cuda.current_stream(dev)
            for i, m in enumerate(mats):  # 1. this shard's rows
                c, sh = row_shards(m.n_features, n)
                r0, r1 = sh[r]
                shards[r][i] = upload_rows(m.values, r0, r1, c, ld, torch.device("cuda", dev), stream)
            blocks.sync(stream)
            barrier.wait()
            full = []
            for i, m in enumerate(mats):  # 2. the full inputs from every shard (peer copies)
                c, _ = row_shards(m.n_features, n)
                t = torch.empty((c * n, ld), dtype=torch.float64, device=dev)
                for q in range(n):
                    t[q * c:(q + 1) * c].copy_(shards[q][i], non_blocking=True)
                full.append(t[:m.n_features])
            torch.cuda.synchronize(dev)
            raw = device_compute(request, full[0], full[1] if len(full) > 1 else None, mat_a, mat_b, ranges,
                                 needed, stream, rank=r, world=n)
            del full
            lo, hi = ranges[r]
            pk = {}
            for name in raw_names:  # 3. this shard's cells, packed
                cnt = cells_count(test, True, shape, lo, hi)
                v = torch.empty(max(1, cnt), dtype=torch.float64, device=dev)
                _pack(test, True, raw[name], shape, lo, hi, v, stream)
                pk[name] = (v, cnt)
            if adj_names:
                cnt = cells_count(test, False, shape, lo, hi)
                v = torch.empty(max(1, cnt), dtype=torch.float64, device=dev)
                _pack(test, False, raw["p"], shape, lo, hi, v, stream)
                pk["__family"] = (v, cnt)
            blocks.sync(stream)
            packs[r] = pk
            barrier.wait()
        except Exception as e:  # noqa: BLE001 -- re-raised in the caller
            errors[r] = e
            barrier.abort()

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(1, n)]
    for t in threads:
        t.start()
    worker(0)
    for t in threads:
        t.join()
    for e in errors:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errors:
        if e is not None:
            raise e
    # 4. assembly on the first device
    dev0 = devices[0]
    torch.cuda.set_device(dev0)
    _lib.check(lib.ps_set_device(dev0))
    stream = torch.cuda.current_stream(dev0)
    result = {}
    for name in raw_names:
        full = torch.full(shape, math.nan, dtype=torch.float64, device=dev0)
        for q, (lo, hi) in enumerate(ranges):
            v, cnt = packs[q][name]
            if cnt:
                _unpack(test, True, v.to(dev0, non_blocking=True), shape, lo, hi, full, stream)
        if name in request.outputs:
            result[name] = full
    if adj_names:
        fam = torch.cat([packs[q]["__family"][0][:packs[q]["__family"][1]].to(dev0) for q in range(n)])
        adj = torch.empty_like(fam)
        offs = np.cumsum([0] + [packs[q]["__family"][1] for q in range(n)])
        for name in adj_names:
            out = torch.full(shape, math.nan, dtype=torch.float64, device=dev0)
            if fam.numel():
                blocks.adjust_family_device(fam, fam.numel(), ADJUSTED_OUTPUTS[name], adj, stream)
            for q, (lo, hi) in enumerate(ranges):
                _unpack(test, False, adj[int(offs[q]):] if fam.numel() else adj, shape, lo, hi, out, stream)
            result[name] = out
    blocks.sync(stream)
    return ResultSet(matrices={k: v.cpu().numpy() for k, v in result.items()}, shape=shape)
