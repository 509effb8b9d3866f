"""The engine='gpu' row of the reference's timing sweep (benchrows.py;
reference pkg/src/pairstat/bench.py:36-46, :128-242)."""

from __future__ import annotations

import math

import pytest

from paper_2505_00448_b200 import benchrows


def test_row_shape_and_csv_without_device(monkeypatch):
    calls = []
    monkeypatch.setattr(benchrows, "run", lambda req, a, b: calls.append(req.threads))
    rows = benchrows.run_bench(("pearson", "anova"), (6,), (40,), (0.1,), threads=(1, 4), reps=2,
                               baselines={"oracle": lambda req, a, b: sum(range(20000))})
    assert [r.engine for r in rows] == ["oracle", "gpu", "gpu"] * 2
    assert all(r.threads == 1 for r in rows if r.engine == "oracle")
    assert all(math.isnan(r.speedup) for r in rows if r.engine == "oracle")
    assert all(r.speedup > 0 for r in rows if r.engine == "gpu")
    assert calls == [1, 1, 1, 4, 4, 4] * 2  # warm-up + 2 reps per row
    text = benchrows.render_rows(rows)
    lines = text.splitlines()
    assert lines[0] == ",".join(benchrows.BENCH_COLUMNS)
    assert lines[1].startswith("pearson,6,40,0.1,1,oracle,") and len(lines) == 7
    with pytest.raises(ValueError, match="unknown engine"):
        benchrows.run_bench(("pearson",), (6,), (40,), (0.1,), engines=("fast",))
    with pytest.raises(ValueError, match="unknown test"):
        benchrows.run_bench(("nope",), (6,), (40,), (0.1,))


@pytest.mark.gpu
def test_gpu_rows_against_the_oracle_baseline(oracle):
    rows = benchrows.run_bench(("pearson", "spearman", "chi2", "kruskal"), (60,), (2000,), (0.1,), reps=2,
                               baselines={"oracle": lambda req, a, b: oracle.oracle_run(req, a, b, threads=1)})
    gpu = [r for r in rows if r.engine == "gpu"]
    assert len(gpu) == 4 and all(r.mean_seconds > 0 and r.speedup > 1.0 for r in gpu)
