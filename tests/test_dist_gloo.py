"""Multi-rank sharding host logic on CPU: world_size 2 over gloo.

dist.sharded_run partitions the pair index space exactly as the reference
partitions it over threads (engine.py:70-125), gathers the owned cells with
one SUM all-reduce and runs the global adjustment.  On the GPU each rank's
shard runs on its own B200; here the per-rank compute and the adjustment are
the CPU oracle, so the test checks the partition / ownership / gather logic:
the assembled result must be bit-identical to a single-process run.
"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]

from paper_2505_00448_b200 import dist  # noqa: E402


def test_partitions_cover_and_balance():
    for n in (1, 7, 100, 1001):
        for parts in (1, 2, 3, 8):
            rows = dist.partition_triangle_rows(n, parts)
            assert rows[0][0] == 0 and rows[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            flat = dist.partition_range(n, parts)
            assert sum(h - l for l, h in flat) == n
    shape = (9, 9)
    owned = sum(dist.owned_mask("pearson", shape, lo, hi).astype(int)
                for lo, hi in dist.partition_triangle_rows(9, 4))
    assert (owned == 1).all()
    owned = sum(dist.owned_mask("anova", (4, 7), lo, hi).astype(int) for lo, hi in dist.partition_range(28, 3))
    assert (owned == 1).all()
    owned = sum(dist.owned_mask("kruskal", (4, 7), lo, hi).astype(int) for lo, hi in dist.partition_range(7, 3))
    assert (owned == 1).all()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, test, out_dir):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as tdist

    import pyoracle
    import workloads
    import paper_2505_00448_b200 as ps

    tdist.init_process_group("gloo", rank=rank, world_size=world)
    kind_a, kind_b = ps.KINDS_BY_TEST[test]
    a = ps.make_matrix(workloads.simulate(11, 120, kind_a, na_ratio=0.2, seed=3), kind_a)
    b = ps.make_matrix(workloads.simulate(6, 120, kind_b, na_ratio=0.2, seed=4), kind_b) if kind_b else None
    req = ps.TestRequest(test, ("stat", "p", "p_bh", "p_bonferroni"))

    def compute(t, ma, mb, lo, hi, wanted):
        return pyoracle.compute(t, ma, mb, wanted=wanted, threads=1, lo=lo, hi=hi)

    res = dist.sharded_run(req, a, b, compute=compute, adjust_fn=pyoracle.adjust)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    tdist.destroy_process_group()


@pytest.mark.parametrize("test", ["pearson", "spearman", "chi2", "anova", "kruskal", "mwu"])
def test_two_rank_gloo_matches_single_process(tmp_path, test):
    sys.path.insert(0, str(ROOT / "oracle"))
    import pyoracle
    import workloads
    import paper_2505_00448_b200 as ps

    pyoracle.build()
    mp.spawn(_worker, args=(2, _free_port(), test, str(tmp_path)), nprocs=2, join=True)
    kind_a, kind_b = ps.KINDS_BY_TEST[test]
    a = ps.make_matrix(workloads.simulate(11, 120, kind_a, na_ratio=0.2, seed=3), kind_a)
    b = ps.make_matrix(workloads.simulate(6, 120, kind_b, na_ratio=0.2, seed=4), kind_b) if kind_b else None
    want = pyoracle.oracle_run(ps.TestRequest(test, ("stat", "p", "p_bh", "p_bonferroni")), a, b, threads=1)
    for rank in (0, 1):
        got = np.load(tmp_path / f"rank{rank}.npz")
        for name, w in want.items():
            g = got[name]
            same = (g.view(np.int64) == w.view(np.int64)) | (np.isnan(g) & np.isnan(w))
            assert same.all(), (rank, name)


def _gather_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch
    import torch.distributed as tdist

    from paper_2505_00448_b200 import dist as d

    tdist.init_process_group("gloo", rank=rank, world_size=world)
    out = torch.empty((world, 3), dtype=torch.float64)
    d.all_gather(out, torch.full((3,), float(rank), dtype=torch.float64))
    torch.save(out, os.path.join(out_dir, f"g{rank}.pt"))
    tdist.destroy_process_group()


def test_all_gather_helper_and_cell_counts(tmp_path):
    """dist.all_gather (the device exchanges' collective) over gloo with 2-D
    outputs, and the packed-cell counts of every partition summing to the
    family (C ABI ps_cells_count, host-only)."""
    import torch

    mp.spawn(_gather_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        g = torch.load(tmp_path / f"g{r}.pt")
        assert g.tolist() == [[0.0] * 3, [1.0] * 3]
    for test, shape in (("pearson", (37, 37)), ("anova", (5, 11)), ("kruskal", (5, 11))):
        units = 37 if test == "pearson" else (55 if test == "anova" else 11)
        fam = 37 * 36 // 2 if test == "pearson" else 55
        for world in (1, 2, 3, 8):
            ranges = dist.plan(test, shape[0], None if test == "pearson" else shape[1], world)
            assert sum(dist.cells_count(test, False, shape, lo, hi) for lo, hi in ranges) == fam
            if test == "pearson":
                assert sum(dist.cells_count(test, True, shape, lo, hi) for lo, hi in ranges) == fam + 37
        assert ranges[-1][1] == units
