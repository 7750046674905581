"""GPU table-level joins (paper_1807_07691_b200.tables) against the
reference executor's own unit-test vectors (test_executor.py:70-150,
test_acceptance.py:85-97) and a nested-loop restatement on random tables."""

from __future__ import annotations

import random
from collections import Counter

import pytest

pytestmark = pytest.mark.gpu

from paper_1807_07691_b200 import tables as T  # noqa: E402
from paper_1807_07691_b200.errors import ResourceLimitError  # noqa: E402
from paper_1807_07691_b200.executor import BindingTable  # noqa: E402

A = BindingTable(("?a", "?b"), [(10, 20), (10, 30)])  # test_executor.py:72-73
B = BindingTable(("?b", "?c"), [(20, 1), (20, 3), (30, 2), (30, 3)])


def test_chain_join_exact_rows():
    out = T.sm_join(A, B, ["?b"])  # test_executor.py:75-78
    assert out.schema == ("?a", "?b", "?c")
    assert out.rows == [(10, 20, 1), (10, 20, 3), (10, 30, 2), (10, 30, 3)]


def test_match_counts_table4():
    assert T.match_counts(A, B, ["?b"]) == Counter({(10, 1): 1, (10, 2): 1, (10, 3): 2})
    i, k, l, r, s, t = 101, 2, 3, 11, 12, 13  # test_acceptance.py:88-93
    a = BindingTable(("?row", "?mid"), [(i, k), (i, l)])
    b = BindingTable(("?mid", "?col"), [(k, r), (k, t), (l, s), (l, t)])
    assert T.match_counts(a, b, ["?mid"]) == Counter({(i, r): 1, (i, s): 1, (i, t): 2})


def test_empty_cartesian_arity_budget():
    assert T.sm_join(BindingTable(("?a", "?b"), []), B, ["?b"]).rows == []
    left = BindingTable(("?a",), [(1,), (2,)])
    right = BindingTable(("?c",), [(5,)])
    out = T.sm_join(left, right, [])
    assert out.schema == ("?a", "?c") and out.rows == [(1, 5), (2, 5)]
    assert len(T.sm_join(A, B, ["?b"]).schema) == 3
    with pytest.raises(ResourceLimitError, match="join output exceeds row budget 2"):
        T.sm_join(A, B, ["?b"], row_budget=2)
    with pytest.raises(ResourceLimitError, match="pre-allocated join region of 4 rows"):
        T.parallel_sm_join(A, B, ["?b"], row_budget=3)
    with pytest.raises(ResourceLimitError, match="cross product of 2 x 1 rows exceeds budget 1"):
        T.cross_product(left, right, row_budget=1)


def test_prealloc_plans():
    plan = T.preallocate(A, B, "?b")  # test_executor.py:103-109
    assert plan.total == 4 and plan.offsets[0] == 0
    for i in range(1, len(plan.counts)):
        assert plan.offsets[i] == plan.offsets[i - 1] + plan.counts[i - 1]
    empty = T.preallocate(BindingTable(("?a", "?b"), []), B, "?b")
    assert empty.counts == [] and empty.offsets == [] and empty.total == 0
    left = BindingTable(("?x", "?w"), [(1, 2), (1, 3), (6, 3)])  # test_executor.py:111-119
    other = BindingTable(("?z", "?w"), [(1, 2), (1, 3), (6, 3)])
    g = T.regroup(left, "?w")
    p2 = T.preallocate(g, other, "?w")
    assert p2.total == 5 and len(T.sm_join(g, other, ["?w"]).rows) == 5
    assert p2.keys == [2, 3] and p2.counts == [1, 4] and p2.offsets == [0, 1]


def _nested_loop(left, right, jv):
    """executor.sm_join restated as a nested loop (small cases only)."""
    li = [left.schema.index(v) for v in jv]
    ri = [right.schema.index(v) for v in jv]
    rcols = [i for i, v in enumerate(right.schema) if v not in set(left.schema)]
    out = []
    for lr in left.rows:
        for rr in right.rows:
            if all(lr[a] == rr[b] for a, b in zip(li, ri)):
                out.append(tuple(lr) + tuple(rr[i] for i in rcols))
    return out


def test_random_tables_exact_order():
    rng = random.Random(31)
    for trial in range(60):
        nl, nr = rng.randint(0, 300), rng.randint(0, 300)
        dom = rng.choice([3, 10, 50, 1000])
        lv = ["?a", "?b", "?c"][: rng.randint(1, 3)]
        shared = rng.sample(lv, rng.randint(1, len(lv)))
        rv = shared + ["?x", "?y"][: rng.randint(0, 2)]
        rng.shuffle(rv)
        left = BindingTable(tuple(lv), [tuple(rng.randrange(dom) for _ in lv) for _ in range(nl)])
        right = BindingTable(tuple(rv), [tuple(rng.randrange(dom) for _ in rv) for _ in range(nr)])
        jv = [v for v in left.schema if v in set(right.schema)]
        exp = _nested_loop(left, right, jv)
        got = T.sm_join(left, right, jv, row_budget=1 << 40)
        assert got.rows == exp, trial  # the reference's row order
        par = T.parallel_sm_join(T.regroup(left, jv[0]), right, jv, worker_count=8,
                                 row_budget=1 << 40)
        assert Counter(par.rows) == Counter(exp), trial
        plan = T.preallocate(left, right, jv[0])
        e = sum(1 for lr in left.rows for rr in right.rows
                if lr[left.schema.index(jv[0])] == rr[right.schema.index(jv[0])])
        assert plan.total == e and sum(plan.counts) == e, trial


def test_reference_bindingtables_accepted():
    gsmat = pytest.importorskip("gsmat")
    ra = gsmat.executor.BindingTable(("?a", "?b"), [(10, 20), (10, 30)])
    rb = gsmat.executor.BindingTable(("?b", "?c"), [(20, 1), (20, 3), (30, 2), (30, 3)])
    assert T.sm_join(ra, rb, ["?b"]).rows == gsmat.executor.sm_join(ra, rb, ["?b"]).rows
