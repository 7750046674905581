"""The reference's OWN test suite (/root/reference/pkg/tests, installed next
to the reference as oracle/_ref/gsmat_tests by oracle/build_ref.sh) run
against the drop-in through the maintainer's mode="gpu" patch
(tests/ref_patch.py), with GSMAT_DEVICE=gpu so every
``execute`` of the suite -- sequential and parallel modes, the CLI's query
command included -- runs on the GPU (SURVEY.md §4 plan)."""

from __future__ import annotations

import json
import os
import shutil
import subprocess
import sys

import pytest

from conftest import REPO

import ref_patch

REF = REPO / "oracle" / "_ref"


def _have_reference() -> bool:
    return (REF / "gsmat" / "executor.py").exists() and (REF / "gsmat_tests" / "conftest.py").exists()


def test_patch_applies_and_is_documented(tmp_path):
    """CPU: the patch INTEGRATION.md §2 prints is the one applied, and it
    applies to the installed reference."""
    doc = (REPO / "INTEGRATION.md").read_text()
    assert ref_patch.EXECUTOR_PATCH in doc
    assert ref_patch.CLI_NEW in doc
    if not _have_reference():
        pytest.skip("reference not installed (oracle/build_ref.sh)")
    out = ref_patch.apply(REF / "gsmat", tmp_path)
    text = (out / "executor.py").read_text()
    assert "GSMAT_DEVICE" in text and "import os" in text
    compile(text, str(out / "executor.py"), "exec")


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_reference_suite_on_gpu(tmp_path):
    if not _have_reference():
        pytest.skip("reference not installed (oracle/build_ref.sh)")
    src = tmp_path / "src"
    src.mkdir()
    ref_patch.apply(REF / "gsmat", src)
    shutil.copytree(REF / "gsmat_tests", tmp_path / "tests")
    plug = tmp_path / "plugins"
    plug.mkdir()
    shutil.copy(REPO / "tests" / "ref_suite_plugin.py", plug)
    counts = tmp_path / "counts.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(src), str(REPO), str(plug)])
    env["GSMAT_DEVICE"] = "gpu"
    env["GSM_REF_SUITE_COUNTS"] = str(counts)
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "ref_suite_plugin",
         "-o", "addopts=", str(tmp_path / "tests")],
        cwd=tmp_path, env=env, capture_output=True, text=True)
    tail = proc.stdout[-4000:] + proc.stderr[-2000:]
    assert proc.returncode == 0, tail
    got = json.loads(counts.read_text())
    # the suite's execute() calls reached the device executor and ran kernels
    assert got["execute_calls"] >= 200, got
    assert got["kernels"] > got["execute_calls"], got
    print(tail.strip().splitlines()[-1], got)
