"""dist.sharded_run end to end with the DEVICE exchanges, two ranks.

gpurun provides one B200, and NCCL refuses two ranks on one device, so the
two ranks share cuda:0 over a gloo group: each rank uploads only its row
shard of the inputs (pinned staging), the shards are all-gathered, each rank
computes its partition of the pairs on the device, packs its p cells
(``ps_cells_pack``), the packed vectors are all-gathered, every rank adjusts
the whole family on the device and unpacks its segment; ``assemble="full"``
then all-gathers every output's packed cells.  On a multi-GPU box the same
code runs over NCCL.  Results must equal the single-process ``run()`` bit for
bit, and ``assemble="owned"`` blocks must equal the same cells.
"""

from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
TESTS = ("pearson", "spearman", "chi2", "ttest", "anova", "kruskal", "mwu")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(test):
    import workloads
    import paper_2505_00448_b200 as ps

    kind_a, kind_b = ps.KINDS_BY_TEST[test]
    a = workloads.simulate(61, 900, kind_a, categories=5, na_ratio=0.2, seed=31)
    b = workloads.simulate(45, 900, kind_b, na_ratio=0.2, seed=32) if kind_b else None
    if b is not None:
        b[3] = np.round(b[3], 1)
    elif kind_a == "continuous":
        a[3] = np.round(a[3], 1)
    ma = ps.make_matrix(a, kind_a)
    mb = ps.make_matrix(b, kind_b) if b is not None else None
    outs = ("stat", "p", "p_bh", "p_bonferroni", "p_by") + ps.EFFECTS_BY_TEST[test]
    return ps.TestRequest(test, outs), ma, mb


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as tdist

    from paper_2505_00448_b200 import _lib, dist

    torch.cuda.set_device(0)
    _lib.check(_lib.load().ps_set_device(0))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    for test in TESTS:
        req, ma, mb = _inputs(test)
        full = dist.sharded_run(req, ma, mb, assemble="full")
        np.savez(os.path.join(out_dir, f"{test}_full_{rank}.npz"), **{n: full[n] for n in req.outputs})
        owned = dist.sharded_run(req, ma, mb, assemble="owned")
        np.savez(os.path.join(out_dir, f"{test}_owned_{rank}.npz"), **owned)
    tdist.destroy_process_group()


def test_two_ranks_device_exchange_matches_run(tmp_path):
    sys.path.insert(0, str(ROOT))
    import paper_2505_00448_b200 as ps
    from paper_2505_00448_b200 import dist
    from conftest import bitwise_equal

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for test in TESTS:
        req, ma, mb = _inputs(test)
        want = ps.run(req, ma, mb)
        shape = want.shape
        plan = dist.plan(test, ma.n_features, None if mb is None else mb.n_features, world)
        for rank in range(world):
            got = np.load(tmp_path / f"{test}_full_{rank}.npz")
            for n in req.outputs:
                assert bitwise_equal(got[n], want[n]), (test, n, rank, "full")
            own = np.load(tmp_path / f"{test}_owned_{rank}.npz")
            lo, hi = plan[rank]
            blk = dist.owned_block(test, shape, lo, hi)
            mask = dist.owned_mask(test, shape, lo, hi)[blk]
            for n in req.outputs:
                g, w = own[n], want[n][blk]
                assert bitwise_equal(np.where(mask, g, 0.0), np.where(mask, w, 0.0)), (test, n, rank, "owned")
