"""Single-process multi-GPU run(): TestRequest.devices (dist.local_run).

One host thread per device; shard r uploads its rows, the inputs are
assembled by peer copies, shard r computes the reference partition r of the
pairs, the first device gathers the packed cells, adjusts the global family
and assembles the matrices.  gpurun provides one B200, so the shards here are
logical (devices=(0, 0, 0): three shards on device 0 -- the same code path
with same-device copies); with more GPUs visible the real multi-device run
is checked too.  Every output must equal the one-device run bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bitwise_equal
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps
from paper_2505_00448_b200 import _lib


def _inputs(test):
    kind_a, kind_b = ps.KINDS_BY_TEST[test]
    a = workloads.simulate(70, 1200, kind_a, categories=5, na_ratio=0.2, seed=61)
    b = workloads.simulate(50, 1200, kind_b, na_ratio=0.2, seed=62) if kind_b else None
    if b is not None:
        b[3] = np.round(b[3], 1)
        b[7] = 0.5
    elif kind_a == "continuous":
        a[3] = np.round(a[3], 1)
    ma = ps.make_matrix(a, kind_a)
    mb = ps.make_matrix(b, kind_b) if b is not None else None
    outs = ("stat", "p", "p_bh", "p_bonferroni", "p_by") + ps.EFFECTS_BY_TEST[test]
    return outs, ma, mb


@pytest.mark.parametrize("devices", [(0, 0), (0, 0, 0)])
@pytest.mark.parametrize("test", ps.TESTS)
def test_logical_shards_match_one_device(test, devices):
    outs, ma, mb = _inputs(test)
    want = ps.run(ps.TestRequest(test, outs), ma, mb)
    got = ps.run(ps.TestRequest(test, outs, devices=devices), ma, mb)
    for n in outs:
        assert bitwise_equal(got[n], want[n]), (test, n, devices)


@pytest.mark.skipif(_lib.device_count() < 2 if _lib.LIB_PATH.exists() else True, reason="one GPU visible")
@pytest.mark.parametrize("test", ps.TESTS)
def test_real_devices_match_one_device(test):
    outs, ma, mb = _inputs(test)
    want = ps.run(ps.TestRequest(test, outs), ma, mb)
    got = ps.run(ps.TestRequest(test, outs, devices=_lib.device_count()), ma, mb)
    for n in outs:
        assert bitwise_equal(got[n], want[n]), (test, n)


def test_devices_validation():
    with pytest.raises(ValueError):
        ps.TestRequest("pearson", ("stat",), devices=0)
    with pytest.raises(ValueError):
        ps.TestRequest("pearson", ("stat",), devices=(0, -1))
    outs, ma, mb = _inputs("pearson")
    with pytest.raises(ValueError, match="not visible"):
        ps.run(ps.TestRequest("pearson", outs, devices=(0, 4096)), ma, mb)
