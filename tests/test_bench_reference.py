"""bench.py --impl reference (the driver's reference arm) runs on CPU and
prints the contract JSON line."""

from __future__ import annotations

import json
import subprocess
import sys

import pytest

from conftest import REPO, reference_available


@pytest.mark.skipif(not reference_available(), reason="reference package not installed")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(REPO / "bench.py"), "--impl", "reference", "--univ",
                          "1", "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    # both of the reference's modes were timed; value is the faster one
    assert set(line["modes"]) == {"sequential", "parallel"}
    assert line["value"] == max(m["value"] for m in line["modes"].values())
    assert line["cpu_baseline"]["cpu_model"]
    # the same workload description as the GPU arm
    sys.path.insert(0, str(REPO))
    import bench

    class A:
        univ, seed = 1, 0
    assert line["config"] == bench._config(A, line["config"]["triples"])


def test_algorithmic_bytes_do_not_bill_fused_intermediates():
    """bench.step_bytes: a step fused into the previous kernel reads no left
    table and its predecessor writes none; a filter fused behind an expand
    (possibly a run intersection) bills neither the candidates nor a lookup
    per candidate — the LUBM-1000 c6 shape (2.3G fused candidate rows) must
    not be billed as 55 GB of HBM traffic."""
    from types import SimpleNamespace as NS

    sys.path.insert(0, str(REPO))
    import bench

    def rep(kinds, rows, pre, arities, fused):
        return NS(kinds=kinds, arities=arities, fused=fused,
                  steps=[NS(rows=r, prealloc_total=e) for r, e in zip(rows, pre)])

    # scan -> expand -> filter, the filter fused behind the expand (c6 shape)
    r = rep(["scan", "expand", "filter"], [3, 2_297_671_802, 2_000], [0, 2_297_671_802, 9e9],
            [2, 3, 3], [0, 0, 1])
    b = bench.query_bytes(r, 2)
    assert b == (16 * 3 + 4 * 3 * 2) + 16 * 3 + 4 * 2_000 * 2
    # unfused: every table is read and written
    r = rep(["scan", "expand", "filter"], [10, 50, 20], [0, 50, 50], [2, 3, 3], [0, 0, 0])
    assert bench.query_bytes(r) == (16 * 10 + 4 * 50 + 4 * 10 * 2 + 4 * 50 * 3) + \
        (16 * 50 + 4 * 50 + 4 * 50 * 3 + 4 * 20 * 3)
    # [filter][expand] group: the expand reads no left table, the filter writes none
    r = rep(["scan", "filter", "expand"], [10, 6, 30], [0, 10, 30], [2, 2, 3], [0, 0, 1])
    assert bench.query_bytes(r) == (16 * 10 + 4 * 10 + 4 * 10 * 2) + (16 * 6 + 4 * 30 + 4 * 30 * 3)
