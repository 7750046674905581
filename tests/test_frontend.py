"""The restated front end (parse/bind/plan) equals the reference's.

Plan order decides the intermediate tables and therefore the per-step
report, so it must be identical (planner.py:113-166)."""

from __future__ import annotations

import random

import pytest

from conftest import GOLDEN, lubm_queries, reference_available
from hoststore import HostStore, plan_for
from paper_1807_07691_b200 import frontend
from paper_1807_07691_b200.errors import ParseError, UnsupportedFeatureError


def test_plans_match_golden_campaign(golden_c3, store_factory):
    for t in golden_c3[:60]:
        store = HostStore(store_factory("powerlaw", triples=t["triples"],
                                        predicates=t["predicates"], zipf=t["zipf"], seed=t["seed"]))
        _, plan = plan_for(store, t["query"])
        assert [s.pattern.source.text() for s in plan.steps] == t["plan"]


def test_plans_match_golden_dg(golden_dg):
    store = HostStore(GOLDEN / "d_g")
    for case in golden_dg:
        exp = case["expected"]
        if "plan" not in exp:
            continue
        _, plan = plan_for(store, case["query"])
        assert [s.pattern.source.text() for s in plan.steps] == exp["plan"], case["name"]


@pytest.mark.parametrize("text,exc", [
    ("SELECT ?x WHERE { ?x ?p ?y . }", UnsupportedFeatureError),
    ("SELECT WHERE { ?x <p> ?y . }", ParseError),
    ("SELECT ?x WHERE { ?x a <C> . }", ParseError),
    ("SELECT ?x WHERE { ?x <p> ?y ; <q> ?z . }", ParseError),
    ("SELECT ?z WHERE { ?x <p> ?y . }", ParseError),
    ("SELECT ?x WHERE { }", ParseError),
    ("SELECT ?x WHERE { ?x pre:p ?y . }", ParseError),
    ("SELECT ?x WHERE { ?x <p> ?y . } extra", ParseError),
    ("SELECT ?x WHERE { ?x <p> \"bad\\q\" . }", ParseError),
])
def test_parse_errors(text, exc):
    with pytest.raises(exc):
        frontend.parse_query(text)


def test_literals_and_prefixes():
    g = frontend.parse_query('PREFIX ub: <http://x#> SELECT DISTINCT * WHERE { '
                             '?x ub:name "a\\"b\\u00e9"@en . ?x ub:age "3"^^<http://int> . '
                             '?x ub:knows _:b1 . }')
    assert g.distinct and g.projection == ["?x"]
    assert g.patterns[0].o == '"a"bé"@en'
    assert g.patterns[1].o == '"3"^^<http://int>'
    assert g.patterns[2].o == "_:b1"
    assert g.patterns[0].text() == '?x <http://x#name> "a\\"bé"@en'


@pytest.mark.skipif(not reference_available(), reason="reference package not installed")
def test_parse_bind_plan_equal_reference(store_factory):
    from gsmat import planner, qparser

    store = HostStore(store_factory("lubm", univ=1, seed=0))
    texts = [t for _, t in lubm_queries()]
    rng = random.Random(4)
    preds = list(store.dictionary.pred_index)
    for _ in range(200):  # random BGPs over the LUBM vocabulary, incl. disconnected ones
        n = rng.randint(1, 5)
        vars_ = [f"?v{i}" for i in range(4)]
        pats = []
        for _ in range(n):
            s = rng.choice(vars_ + ["<http://www.University0.edu>"])
            o = rng.choice(vars_ + ["<http://www.Department0.University0.edu>", '"xxx-xxx-xxxx"'])
            pats.append(f"{s} <{rng.choice(preds)}> {o} .")
        texts.append("SELECT * WHERE { " + " ".join(pats) + " }")
    for text in texts:
        g_ref = qparser.parse_query(text)
        g_our = frontend.parse_query(text)
        assert [(p.s, p.p, p.o) for p in g_ref.patterns] == [(p.s, p.p, p.o) for p in g_our.patterns]
        assert g_ref.projection == g_our.projection and g_ref.distinct == g_our.distinct
        q_ref = qparser.bind_constants(g_ref, store.dictionary)
        q_our = frontend.bind_constants(g_our, store.dictionary)
        p_ref = planner.make_plan(q_ref, store.stats)
        p_our = frontend.make_plan(q_our, store.stats)
        key = lambda st: (st.pattern.s, st.pattern.p, st.pattern.o, st.pattern.empty,  # noqa: E731
                          st.estimate, st.join_vars)
        assert [key(s) for s in p_ref.steps] == [key(s) for s in p_our.steps], text
        assert p_ref.warnings == p_our.warnings
