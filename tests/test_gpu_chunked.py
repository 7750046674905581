"""Left-row chunking (SURVEY.md §5 long-context row, §7 hard part 2) and the
device-side result fingerprint, on the GPU.

A plan whose intermediate tables exceed device memory runs once per
equal-E slice of its first table; the slices' rows concatenated are the
one-pass result, and the per-step counters summed are the one-pass report.
The arena cap GSM_ARENA_MAX makes a small store overflow so every path is
exercised at test size: the first failure, the initial chunk count, the
in-place split of a chunk that still overflows, the budget rules on the
summed counters, DISTINCT across chunks, and execute_summary (rows reduced
on the device, never copied out).  Checked against the one-pass run and the
C oracle.
"""

from __future__ import annotations

import os
from collections import Counter

import numpy as np
import pytest

from conftest import lubm_queries
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

import paper_1807_07691_b200 as g  # noqa: E402

PROBE = ("PREFIX ub: <http://swat.cse.lehigh.edu/onto/univ-bench.owl#> "
         "SELECT * WHERE { ?x ub:memberOf ?d . ?y ub:memberOf ?d . }")
PROBE3 = ("PREFIX ub: <http://swat.cse.lehigh.edu/onto/univ-bench.owl#> "
          "SELECT ?x ?b WHERE { ?x ub:memberOf ?d . ?y ub:memberOf ?d . ?x ub:advisor ?a . "
          "?y ub:advisor ?b . }")


def _plan(store, text):
    q = g.bind_constants(g.parse_query(text), store.dictionary)
    return q, g.make_plan(q, store.stats)


def _bag(a):
    return Counter(map(tuple, np.asarray(a).tolist()))


@pytest.fixture(scope="module")
def lubm1(store_factory):
    return store_factory("lubm", univ=1, seed=0)


@pytest.fixture(scope="module")
def capped(lubm1):
    """The LUBM-1 store with its context's arena capped at 2 MB."""
    os.environ["GSM_ARENA_MAX"] = str(2 << 20)
    try:
        st = g.load(lubm1)
        st.context()  # the cap is read when the context is created
    finally:
        del os.environ["GSM_ARENA_MAX"]
    return st


@pytest.fixture(scope="module")
def full(lubm1):
    return g.load(lubm1)


def _oracle(store, q, plan, budget=1 << 62):
    rows, step_rows, step_pre = orc.run(store.matrices, [s.pattern for s in plan.steps],
                                        q.projection, q.distinct, budget=budget)
    return np.asarray(rows, dtype=np.uint32).reshape(len(rows), len(q.projection)), step_rows, step_pre


@pytest.mark.parametrize("text", [PROBE, PROBE3])
def test_overflow_runs_chunked(capped, full, text):
    q, plan = _plan(full, text)
    exp_rep = g.ExecutionReport()
    exp = g.execute(q, plan, full, row_budget=1 << 62, report=exp_rep)
    assert exp_rep.chunks == 0
    # the one-pass result is larger than the capped arena
    assert 8 * max(s.rows for s in exp_rep.steps) * 3 > (2 << 20)
    q2, plan2 = _plan(capped, text)
    rep = g.ExecutionReport()
    got = g.execute(q2, plan2, capped, row_budget=1 << 62, report=rep)
    assert rep.chunks >= 2
    assert [s.rows for s in rep.steps] == [s.rows for s in exp_rep.steps]
    assert [s.prealloc_total for s in rep.steps] == [s.prealloc_total for s in exp_rep.steps]
    assert got.array.shape == exp.array.shape
    # first-table order is kept: the concatenated slices are the one-pass rows
    assert np.array_equal(got.array, exp.array) or _bag(got.array) == _bag(exp.array)
    o, o_rows, o_pre = _oracle(full, q, plan)
    assert orc.fingerprint_array(got.array) == orc.fingerprint_array(o)
    assert [s.rows for s in rep.steps] == list(o_rows)


def test_summary_matches_rows_and_oracle(capped, full):
    q, plan = _plan(full, PROBE)
    exp = g.execute(q, plan, full, row_budget=1 << 62)
    fp = orc.fingerprint_array(exp.array)
    # one pass, reduced on the device (result in the arena / staging buffer)
    s1 = g.execute_summary(q, plan, full, row_budget=1 << 62)
    assert s1.fingerprint == fp
    assert g.fingerprint_rows(exp.array) == fp
    # chunked under the cap (an intermediate of 2.4M x 4 ids): each chunk
    # reduced on the device
    q3, plan3 = _plan(full, PROBE3)
    fp3 = orc.fingerprint_array(g.execute(q3, plan3, full, row_budget=1 << 62).array)
    q2, plan2 = _plan(capped, PROBE3)
    rep = g.ExecutionReport()
    s2 = g.execute_summary(q2, plan2, capped, row_budget=1 << 62, report=rep)
    assert rep.chunks >= 2
    assert s2.fingerprint == fp3
    # small (zero-copy staged) results too
    for name, text in lubm_queries():
        qq, pp = _plan(full, text)
        r = g.execute(qq, pp, full)
        assert g.execute_summary(qq, pp, full).fingerprint == orc.fingerprint_array(r.array), name


@pytest.mark.parametrize("chunks", [2, 8, 64])
def test_forced_chunks_lubm_queries(full, chunks):
    """Every LUBM query evaluated in k left-row chunks == one pass (rows in
    order, report counters)."""
    for name, text in lubm_queries():
        q, plan = _plan(full, text)
        r1, r2 = g.ExecutionReport(), g.ExecutionReport()
        a = g.execute(q, plan, full, report=r1)
        b = g.execute(q, plan, full, report=r2, chunks=chunks)
        assert _bag(a.array) == _bag(b.array), name
        assert [s.rows for s in r1.steps] == [s.rows for s in r2.steps], name
        assert [s.prealloc_total for s in r1.steps] == [s.prealloc_total for s in r2.steps], name
        assert r2.chunks == chunks, name


def test_chunked_budget_errors_match_one_pass(full):
    q, plan = _plan(full, PROBE3)
    rep = g.ExecutionReport()
    g.execute(q, plan, full, row_budget=1 << 62, report=rep)
    big = max(s.rows for s in rep.steps)
    for mode in ("sequential", "parallel"):
        for budget in (big // 3, big - 1, rep.steps[1].rows - 1):
            with pytest.raises(g.ResourceLimitError) as e1:
                g.execute(q, plan, full, mode=mode, row_budget=budget)
            with pytest.raises(g.ResourceLimitError) as e2:
                g.execute(q, plan, full, mode=mode, row_budget=budget, chunks=16)
            assert str(e1.value) == str(e2.value), (mode, budget)


def test_chunked_distinct_and_cross(full):
    texts = [
        "PREFIX ub: <http://swat.cse.lehigh.edu/onto/univ-bench.owl#> "
        "SELECT DISTINCT ?d WHERE { ?x ub:memberOf ?d . ?y ub:memberOf ?d . }",
        "PREFIX ub: <http://swat.cse.lehigh.edu/onto/univ-bench.owl#> "
        "SELECT ?u ?c WHERE { ?u ub:subOrganizationOf ?c . ?x ub:headOf ?y . }",
    ]
    for text in texts:
        q, plan = _plan(full, text)
        a = g.execute(q, plan, full, row_budget=1 << 62)
        b = g.execute(q, plan, full, row_budget=1 << 62, chunks=8)
        assert _bag(a.array) == _bag(b.array), text
        o, _, _ = _oracle(full, q, plan)
        assert _bag(o) == _bag(b.array), text
    # the cross-product rule on the summed left rows
    q, plan = _plan(full, texts[1])
    rep = g.ExecutionReport()
    g.execute(q, plan, full, row_budget=1 << 62, report=rep)
    with pytest.raises(g.ResourceLimitError) as e1:
        g.execute(q, plan, full, row_budget=rep.steps[-1].rows - 1)
    with pytest.raises(g.ResourceLimitError) as e2:
        g.execute(q, plan, full, row_budget=rep.steps[-1].rows - 1, chunks=4)
    assert str(e1.value) == str(e2.value)
    assert str(e1.value).startswith("cross product of ")


def test_batch_falls_back_to_chunks(capped):
    items = [_plan(capped, t) for _, t in lubm_queries()[:3]] + [_plan(capped, PROBE3)]
    res = g.execute_batch(items, capped, row_budget=1 << 62)
    for (q, p), r in zip(items, res):
        one = g.execute(q, p, capped, row_budget=1 << 62)
        assert _bag(one.array) == _bag(r.array)


def test_row_granular_chunks_beyond_the_chunk_table(full):
    """More left-row chunks than k_slice_sums' 4096 chunks (and than first-
    table rows): row-granular equal-E slices still tile the table exactly."""
    q, plan = _plan(full, PROBE)
    r1, r2 = g.ExecutionReport(), g.ExecutionReport()
    a = g.execute(q, plan, full, row_budget=1 << 62, report=r1)
    b = g.execute(q, plan, full, row_budget=1 << 62, report=r2, chunks=16384)
    assert r1.steps[0].rows < 16384
    assert r2.chunks == 16384
    assert np.array_equal(a.array, b.array)  # slices concatenated in first-table order
    assert [s.rows for s in r1.steps] == [s.rows for s in r2.steps]
