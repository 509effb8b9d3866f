"""Multi-GPU sharding: one process per GPU, pairs partitioned, one exchange.

The reference parallelises by static, disjoint pair ranges over threads
(``engine.py:70-125`` partitions, ``:360-376`` dispatch); cells are
independent, so results never depend on the partition (``SPEC.md:469``).
Here the same ranges are handed to ranks (``torch.distributed``, NCCL on
GPUs, gloo in the CPU tests): each rank runs its block on its own B200 with no
data-path collective.  The single real exchange is the p-value gather that the
global Benjamini-Hochberg / BY family needs (``adjust.py:46-87`` ranks all
defined p-values of the matrix together): every rank contributes its owned
cells (zeros elsewhere) to one SUM all-reduce -- x + 0.0 == x exactly, NaN
stays NaN -- and the adjustment then runs on the device of each rank.

Determinism: a cell's arithmetic never depends on which rank owns it, and the
gathered BH is order-insensitive, so 1/2/4/8-GPU results are bitwise equal.
"""

from __future__ import annotations

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


def _world():
    import torch.distributed as tdist

    if tdist.is_available() and tdist.is_initialized():
        return tdist, tdist.get_world_size(), tdist.get_rank()
    return None, 1, 0


def gather_owned(values, mask_owned) -> None:
    """In-place SUM all-reduce of a tensor holding owned cells and 0 elsewhere."""
    tdist, world, _ = _world()
    if world == 1:
        return
    values.masked_fill_(~mask_owned, 0.0)
    tdist.all_reduce(values, op=tdist.ReduceOp.SUM)


def adjust_gathered(test: str, p, shape, plan_ranges, methods, out, stream=None) -> None:
    """Gather the sharded p matrix (if sharded) and run the device adjustment."""
    from . import blocks

    tdist, world, rank = _world()
    if world > 1:
        import torch

        lo, hi = plan_ranges[rank]
        own = torch.from_numpy(owned_mask(test, tuple(shape), lo, hi)).to(p.device)
        gather_owned(p, own)
    for m in methods:
        blocks.adjust_device(p, shape[0], shape[1], m, test in HOMOGENEOUS, out, stream)


def sharded_run(request, mat_a, mat_b=None,
                compute: Callable | None = None,
                adjust_fn: Callable | None = None) -> dict[str, np.ndarray]:
    """Run one request across the ranks of the current process group.

    ``compute(test, mat_a, mat_b, lo, hi, wanted)`` returns dict name -> full
    NaN-prefilled matrix with this rank's cells filled.  The default computes
    on this rank's B200 via :mod:`.blocks`; the CPU tests inject the oracle.
    Returns the full result matrices (identical on every rank).
    """
    import torch

    from .datamodel import EFFECTS_BY_TEST
    from .engine import ADJUSTED_OUTPUTS, validate

    shape = validate(request, mat_a, mat_b)
    test = request.test
    tdist, world, rank = _world()
    ranges = plan(test, mat_a.n_features, None if mat_b is None else mat_b.n_features, world)
    lo, hi = ranges[rank]
    canonical = ("stat", "p") + EFFECTS_BY_TEST[test]
    needed = {n for n in request.outputs if n not in ADJUSTED_OUTPUTS}
    if any(n in ADJUSTED_OUTPUTS for n in request.outputs):
        needed.add("p")
    if compute is None:
        compute = _device_compute(request)
    raw = compute(test, mat_a, mat_b, lo, hi, needed)
    own = owned_mask(test, shape, lo, hi)
    full = {}
    for name in canonical:
        if name not in needed:
            continue
        t = torch.from_numpy(np.where(own, raw[name], 0.0))
        if world > 1:
            if tdist.get_backend() == "nccl":  # NCCL reduces device tensors (NVLink)
                t = t.cuda()
                tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
                t = t.cpu()
            else:
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


def _device_compute(request):
    def compute(test, mat_a, mat_b, lo, hi, wanted):
        import torch

        from . import blocks
        from .datamodel import EFFECTS_BY_TEST

        canonical = ("stat", "p") + EFFECTS_BY_TEST[test]
        shape = (mat_a.n_features, mat_a.n_features if mat_b is None else mat_b.n_features)
        _, world, rank = _world()
        sharded = world > 1
        da = blocks.DeviceMatrix.from_datamatrix(mat_a, presort=test == "spearman" and not sharded)
        if test == "spearman" and sharded:  # 1/world of the presort per rank + all-gather
            da.presort_sharded(rank, world)
        db = None
        if mat_b is not None:
            walk = test in ("mwu", "kruskal")
            db = blocks.DeviceMatrix.from_datamatrix(mat_b, presort=walk and not sharded)
            if walk and sharded:  # the walk only touches features [lo, hi)
                db.presort_rows_only(lo, hi)
        outs = [torch.full(shape, float("nan"), dtype=torch.float64, device="cuda")
                if n in wanted else None for n in canonical]
        blocks.block(test, da, db, lo, hi, outs, t_variant=request.t_variant,
                     u_mode=request.u_mode)
        blocks.sync()
        da.close()
        if db is not None:
            db.close()
        return {n: (o.cpu().numpy() if o is not None else None) for n, o in zip(canonical, outs)}

    return compute
