"""Host logic of left-row chunking (no GPU): the budget rules on summed
counters, DISTINCT across chunks, the host fingerprint twin, chunk counts."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1807_07691_b200 import _lib
from paper_1807_07691_b200 import executor as ex
from paper_1807_07691_b200.errors import DeviceMemoryError, ResourceLimitError

SEQ, PAR = _lib.GSM_BUDGET_SEQUENTIAL, _lib.GSM_BUDGET_PARALLEL


def test_device_memory_error_is_a_resource_limit():
    assert issubclass(DeviceMemoryError, ResourceLimitError)
    with pytest.raises(DeviceMemoryError):
        _lib.raise_status(_lib.GSM_ERR_DEVICE_MEMORY, "intermediate result of 5 rows x 2 columns "
                          "exceeds device memory")


def test_budget_totals_plan_order():
    kinds = ["scan", "expand", "filter", "cross", "expand"]
    rows = [10, 50, 20, 200, 7]
    pre = [0, 50, 60, 0, 900]
    ex._check_budget_totals(kinds, rows, pre, 10**9, SEQ)
    ex._check_budget_totals(kinds, rows, pre, 10**9, PAR)
    with pytest.raises(ResourceLimitError, match=r"^join output exceeds row budget 49$"):
        ex._check_budget_totals(kinds, rows, pre, 49, SEQ)
    with pytest.raises(ResourceLimitError,
                       match=r"^pre-allocated join region of 60 rows exceeds budget 55$"):
        ex._check_budget_totals(kinds, rows, pre, 55, PAR)
    # the cross step: |L| = rows of the previous step, |R| = rows / |L|
    with pytest.raises(ResourceLimitError, match=r"^cross product of 20 x 10 rows exceeds budget 199$"):
        ex._check_budget_totals(kinds, [10, 50, 20, 200, 7], [0, 50, 20, 0, 7], 199, PAR)
    # an empty left side makes the cross product empty: no error
    ex._check_budget_totals(["scan", "cross"], [0, 0], [0, 0], 0, SEQ)
    # a gate (constant pattern) keeps |L| rows or none
    with pytest.raises(ResourceLimitError, match=r"^cross product of 30 x 1 rows exceeds budget 29$"):
        ex._check_budget_totals(["scan", "gate"], [30, 30], [0, 0], 29, SEQ)


def test_dedupe_first_keeps_first_occurrences_in_order():
    a = np.array([[3, 1], [1, 2], [3, 1], [0, 0], [1, 2], [5, 5]], dtype=np.uint32)
    out = ex._dedupe_first(a)
    assert out.tolist() == [[3, 1], [1, 2], [0, 0], [5, 5]]
    z = np.empty((4, 0), dtype=np.uint32)
    assert ex._dedupe_first(z).shape == (1, 0)
    assert ex._dedupe_first(np.empty((0, 3), dtype=np.uint32)).shape == (0, 3)


def test_fingerprint_rows_matches_oracle():
    rng = np.random.default_rng(0)
    for k in (1, 2, 5):
        a = rng.integers(0, 2**32, size=(1000, k), dtype=np.uint64).astype(np.uint32)
        assert ex.fingerprint_rows(a) == orc.fingerprint_array(a)
        assert ex.fingerprint_rows(a[::-1]) == orc.fingerprint_array(a)
    assert ex.fingerprint_rows(np.empty((0, 3), dtype=np.uint32)) == (0, 0, 0)
    e = np.empty((3, 0), dtype=np.uint32)
    assert ex.fingerprint_rows(e) == orc.fingerprint([(), (), ()])


def test_chunk_counts_are_powers_of_two():
    assert [ex._pow2(k) for k in (1, 2, 3, 5, 64, 65)] == [1, 2, 4, 8, 64, 128]
    assert ex._pow2(10**12) == ex._MAX_PARTS
    with pytest.raises(ValueError):
        ex._pow2(0)


def test_first_chunk_count_from_the_overflow_message():
    class _Ctx:  # a store whose context has 1 GiB of capacity
        def context(self):
            return None

    import ctypes as C

    calls = {}

    def cap(ctx, out):
        C.cast(out, C.POINTER(C.c_int64))[0] = 1 << 30
        calls["n"] = calls.get("n", 0) + 1
        return 0

    L = _lib.lib()
    orig = L.gsm_context_capacity
    try:
        L.gsm_context_capacity = cap
        # 10^9 rows x 3 columns x 8 bytes (two arena halves) x 1.25 over 1 GiB -> 28 -> 32
        msg = "intermediate result of 1000000000 rows x 3 columns exceeds device memory"
        assert ex._first_parts(_Ctx(), msg) == 32
        assert ex._first_parts(_Ctx(), "something else") == 2
    finally:
        L.gsm_context_capacity = orig
    assert calls["n"] == 2


def test_chunks_and_partition_do_not_combine():
    class _Q:
        projection = ["?x"]
        distinct = False

    class _P:
        steps = [type("S", (), {"pattern": None})()]

    with pytest.raises(ValueError):
        ex.execute(_Q(), _P(), object(), partition=(0, 2), chunks=2)
