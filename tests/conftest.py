"""Shared fixtures.

CPU tests (``-m "not gpu"``) cover the oracle against the reference's golden
vectors, the host logic (front end, generators, multi-process plumbing) and
the C ABI's exports.  GPU tests (``-m gpu``) are the parity tests proper: they
call the CUDA path through the C ABI and compare with the oracle/goldens.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
for p in (REPO,):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))
_REF = REPO / "oracle" / "_ref"
if _REF.exists() and str(_REF) not in sys.path:
    sys.path.append(str(_REF))  # the installed reference, when present (never /root/reference)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def reference_available() -> bool:
    try:
        import gsmat  # noqa: F401

        return True
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden_dg():
    return json.loads((GOLDEN / "golden_dg.json").read_text())


@pytest.fixture(scope="session")
def golden_c3():
    return json.loads((GOLDEN / "golden_c3.json").read_text())


@pytest.fixture(scope="session")
def golden_lubm1():
    return json.loads((GOLDEN / "golden_lubm1.json").read_text())


@pytest.fixture(scope="session")
def store_factory(tmp_path_factory):
    """Generate (and cache) stores with datagen/gsmgen."""
    from oracle import oracle as orc

    cache: dict[tuple, Path] = {}

    def make(kind: str, **kw) -> Path:
        key = (kind, tuple(sorted(kw.items())))
        if key in cache:
            return cache[key]
        d = tmp_path_factory.mktemp(f"{kind}")
        args = [kind]
        for k, v in kw.items():
            args += [f"--{k.replace('_', '-')}", str(v)]
        args += ["--out", str(d / "store")]
        orc.gsmgen(*args)
        cache[key] = d / "store"
        return cache[key]

    return make


def lubm_queries() -> list[tuple[str, str]]:
    qdir = REPO / "datagen" / "queries" / "lubm"
    return [(f.stem, f.read_text()) for f in sorted(qdir.glob("*.rq"))]
