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
