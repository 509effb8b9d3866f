"""The multi-GPU plumbing on the B200 box: a NCCL process group (one rank --
gpurun provides one GPU) running ``dist.sharded_run`` with the device compute
and device adjustment, checked bit for bit against ``run``.  The 2-rank
exchange itself is covered over gloo in test_dist_gloo.py."""

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


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, str(ROOT))
    import torch
    import torch.distributed as tdist

    import workloads
    import paper_2505_00448_b200 as ps
    from paper_2505_00448_b200 import dist

    torch.cuda.set_device(0)
    tdist.init_process_group("nccl", rank=rank, world_size=1, device_id=torch.device("cuda", 0))
    x = torch.arange(8, dtype=torch.float64, device="cuda")
    tdist.all_reduce(x)  # the collective itself runs on the device
    assert torch.equal(x.cpu(), torch.arange(8, dtype=torch.float64))
    for test in ("spearman", "chi2", "kruskal"):
        kind_a, kind_b = ps.KINDS_BY_TEST[test]
        a = ps.make_matrix(workloads.simulate(23, 700, kind_a, na_ratio=0.2, seed=3), kind_a)
        b = ps.make_matrix(workloads.simulate(9, 700, kind_b, na_ratio=0.2, seed=4), kind_b) if kind_b else None
        req = ps.TestRequest(test, ("stat", "p", "p_bh"))
        res = dist.sharded_run(req, a, b)
        ref = ps.run(req, a, b)
        for name in req.outputs:
            g, w = res[name], ref[name]
            same = (g.view(np.int64) == w.view(np.int64)) | (np.isnan(g) & np.isnan(w))
            assert same.all(), (test, name)
    tdist.destroy_process_group()
    Path(out_dir, "ok").write_text("ok")


def test_nccl_group_sharded_run_matches_run(tmp_path):
    mp.spawn(_worker, args=(_free_port(), str(tmp_path)), nprocs=1, join=True)
    assert (tmp_path / "ok").exists()
