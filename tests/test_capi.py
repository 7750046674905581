"""The C ABI library loads and exports every symbol include/gsmat_b200.h
declares (no compute calls: runs without a GPU)."""

from __future__ import annotations

import ctypes as C
import re
import subprocess

from conftest import REPO

from paper_1807_07691_b200 import _lib

HEADER = REPO / "include" / "gsmat_b200.h"


def header_symbols() -> set[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(gsm_[a-z_]+)\s*\(", text))


def test_header_and_binding_agree():
    assert header_symbols() == set(_lib.EXPORTS)


def test_library_exports_every_symbol():
    if not _lib.LIB_PATH.exists():
        subprocess.run(["make", "-s", "-C", str(REPO / "paper_1807_07691_b200" / "csrc")], check=True)
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], check=True,
                         capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = header_symbols() - exported
    assert not missing, missing
    L = _lib.lib()
    for name in _lib.EXPORTS:
        assert getattr(L, name) is not None


def test_error_plumbing_without_device():
    L = _lib.lib()
    assert isinstance(_lib.last_error(), str)
    n = C.c_int32(-1)
    L.gsm_device_count(C.byref(n))
    assert n.value >= 0
    assert L.gsm_kernel_launches() >= 0
    # null handles are rejected with GSM_ERR_VALUE, not a crash
    assert L.gsm_store_finalize(None) == _lib.GSM_ERR_VALUE
    assert "null" in _lib.last_error()


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        return  # cuobjdump unavailable
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches
