"""Pin the C oracle (oracle/gsm_oracle.c) to the reference's golden vectors.

The goldens were produced by the reference itself (tests/golden/make_golden.py);
these tests need no GPU and no reference install.  The oracle must match the
reference ROW FOR ROW (same order), step report and budget errors included.
"""

from __future__ import annotations

import pytest

from conftest import GOLDEN
from hoststore import HostStore, plan_for
from oracle import oracle as orc


@pytest.fixture(scope="module")
def dg_store():
    return HostStore(GOLDEN / "d_g")


def _run(store, text, mode, budget):
    q, plan = plan_for(store, text)
    prep = orc.PreparedStore(store.matrices)
    return q, plan, orc.run(prep, [s.pattern for s in plan.steps], q.projection, q.distinct,
                            budget=budget, mode=mode)


def test_dg_golden_rows_and_reports(dg_store, golden_dg):
    for case in golden_dg:
        exp = case["expected"]
        budget = case["budget"] if case["budget"] is not None else 10**8
        if "error" in exp:
            with pytest.raises(orc.OracleResourceError) as ei:
                _run(dg_store, case["query"], case["mode"], budget)
            assert str(ei.value) == exp["message"], case["name"]
            continue
        q, plan, (rows, srows, spre) = _run(dg_store, case["query"], case["mode"], budget)
        assert [s.pattern.source.text() for s in plan.steps] == exp["plan"], case["name"]
        assert rows == [tuple(r) for r in exp["rows"]], case["name"]
        assert srows == exp["step_rows"], case["name"]
        assert spre == exp["step_prealloc"], case["name"]


def test_fig_query_worked_example(dg_store):
    """test_acceptance.py:58-66: rows == [(1, 4, 6, 3)] = ids of (A, B, C, I2)."""
    q, plan, (rows, _, _) = _run(dg_store, "SELECT ?x ?y ?z ?w WHERE { ?x <:follows> ?y . "
                                 "?y <:follows> ?z . ?x <:likes> ?w . ?z <:likes> ?w . }",
                                 "sequential", 10**8)
    assert rows == [(1, 4, 6, 3)]
    assert [dg_store.dictionary.decode_node(v) for v in rows[0]] == ["A", "B", "C", "I2"]


def test_c3_campaign_golden(golden_c3, store_factory):
    """The reference's 200-trial acceptance campaign (test_acceptance.py:135-174)."""
    for t in golden_c3:
        d = store_factory("powerlaw", triples=t["triples"], predicates=t["predicates"],
                          zipf=t["zipf"], seed=t["seed"])
        store = HostStore(d)
        q, plan, (rows, srows, spre) = _run(store, t["query"], "sequential", 10**8)
        assert [s.pattern.source.text() for s in plan.steps] == t["plan"], t["trial"]
        assert len(rows) == t["count"], t["trial"]
        assert [str(v) for v in orc.fingerprint(rows)] == t["fingerprint"], t["trial"]
        if "rows" in t:
            assert rows == [tuple(r) for r in t["rows"]], t["trial"]
        assert srows == t["step_rows"], t["trial"]
        assert spre == t["step_prealloc"], t["trial"]


def test_lubm1_golden(golden_lubm1, store_factory):
    store = HostStore(store_factory("lubm", univ=1, seed=0))
    from conftest import lubm_queries

    texts = dict(lubm_queries())
    prep = orc.PreparedStore(store.matrices)
    for g in golden_lubm1:
        q, plan = plan_for(store, texts[g["name"]])
        rows, srows, spre = orc.run(prep, [s.pattern for s in plan.steps], q.projection, q.distinct)
        assert len(rows) == g["count"], g["name"]
        assert [str(v) for v in orc.fingerprint(rows)] == g["fingerprint"], g["name"]
        if "rows" in g:
            assert rows == [tuple(r) for r in g["rows"]], g["name"]
        assert srows == g["step_rows"] and spre == g["step_prealloc"], g["name"]


def test_fingerprint_array_matches_scalar():
    import numpy as np

    rows = [(1, 2, 3), (4, 5, 6), (1, 2, 3), (7, 8, 9)]
    assert orc.fingerprint(rows) == orc.fingerprint_array(np.array(rows))
    assert orc.fingerprint([]) == orc.fingerprint_array(np.zeros((0, 3)))


def test_watdiv_oracle_matches_reference(store_factory):
    """WatDiv-style store + the 20 L/S/F/C templates: the C oracle equals the
    reference executor row for row (skipped without the reference install)."""
    gsmat = pytest.importorskip("gsmat")
    from gsmat import executor, planner, qparser, storage

    from conftest import REPO

    d = store_factory("watdiv", scale=2, seed=0)
    host = HostStore(d)
    ref = storage.load(d)
    prep = orc.PreparedStore(host.matrices)
    for f in sorted((REPO / "datagen" / "queries" / "watdiv").glob("*.rq")):
        text = f.read_text()
        q, plan = plan_for(host, text)
        rows, srows, spre = orc.run(prep, [s.pattern for s in plan.steps], q.projection, q.distinct)
        rq = qparser.bind_constants(qparser.parse_query(text), ref.dictionary)
        rp = planner.make_plan(rq, ref.stats)
        rep = executor.ExecutionReport()
        res = executor.execute(rq, rp, ref, row_budget=1 << 62, report=rep)
        assert rows == res.rows, f.stem
        assert srows == [s.rows for s in rep.steps], f.stem
        assert spre == [s.prealloc_total for s in rep.steps], f.stem
