"""bench.py's multi-GPU modes run end to end under torchrun (2 ranks sharing
one GPU over gloo, as on the one-GPU test box; on an 8-GPU node the same
path runs over NCCL with one GPU per rank) and every query's gathered bag
matches the C oracle."""

from __future__ import annotations

import json
import socket
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(900)
@pytest.mark.parametrize("mode,workload,extra", [
    ("partition", "lubm", ["--univ", "2"]),
    ("sharded", "lubm", ["--univ", "2"]),
    ("sharded", "watdiv", ["--scale", "5"]),
    ("partition", "powerlaw", ["--triples", "200000", "--predicates", "8"]),
])
def test_bench_distributed_modes(mode, workload, extra):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(REPO / "bench.py"),
           "--gpus", "2", "--mode", mode, "--workload", workload, *extra, "--backend", "gloo",
           "--share-gpu", "--steps", "2", "--warmup", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=850)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["mode"] == mode
    par = line["parity"]
    assert par["queries"] == len(line["queries"]) > 0
    bad = {k: v for k, v in par["per_query"].items() if v is not True}
    assert not bad, bad
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    if mode == "sharded":
        assert line["exchanged_bytes_per_step"] > 0


@pytest.mark.timeout(900)
def test_bench_replica_mode_two_ranks():
    """The default multi-GPU mode (what `bench.py --gpus N` runs under
    torchrun): every rank serves its own copy of the query stream, timing is
    the max over ranks and `value` the whole job's rows over it."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(REPO / "bench.py"),
           "--gpus", "2", "--backend", "gloo", "--share-gpu", "--univ", "2", "--steps", "3",
           "--warmup", "3", "--no-cpu-baseline", "--no-probe"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=850)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
