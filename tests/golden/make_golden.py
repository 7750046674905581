"""Generate the golden vectors under tests/golden/ from the REFERENCE itself.

Run in a container where the reference is present (it imports the unmodified
``gsmat`` package from oracle/_ref or /root/reference/pkg/src and the
reference test-suite helpers from /root/reference/pkg/tests):

    python tests/golden/make_golden.py

Outputs (committed; nothing at test time reads /root/reference):
  d_g/               the paper's 9-triple example store (Fig. 8, conftest.py:13-23),
                     built and persisted by the reference (storage.py:165-219)
  golden_dg.json     reference executor results/reports/errors on that store
  golden_c3.json     the reference's acceptance campaign c3/c4
                     (test_acceptance.py:135-174, seed 20240817, 200 trials),
                     replayed: generator parameters, query text, expected bag
                     (count + fingerprint + rows when small), per-step report
  golden_lubm1.json  LUBM-1 (datagen/gsmgen lubm --univ 1 --seed 0), Q1-Q14
"""

from __future__ import annotations

import json
import random
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
for p in (REF_SRC, REPO / "oracle" / "_ref", REPO):
    if p.exists() and str(p) not in sys.path:
        sys.path.insert(0, str(p))
if REF_TESTS.exists():  # appended: its oracle.py must not shadow our oracle package
    sys.path.append(str(REF_TESTS))

from gsmat import executor, generate, planner, qparser, storage  # noqa: E402
from gsmat.dictionary import TermDictionary  # noqa: E402
from gsmat.errors import ResourceLimitError  # noqa: E402

from oracle.oracle import fingerprint  # noqa: E402

D_G_TRIPLES = [
    ("A", ":likes", "I1"),
    ("A", ":likes", "I2"),
    ("A", ":follows", "B"),
    ("B", ":related", "h"),
    ("B", ":follows", "C"),
    ("B", ":follows", "D"),
    ("C", ":likes", "I2"),
    ("C", ":follows", "D"),
    ("D", ":related", "h"),
]

FIG_QUERY = """SELECT ?x ?y ?z ?w
WHERE {
  ?x <:follows> ?y .
  ?y <:follows> ?z .
  ?x <:likes> ?w .
  ?z <:likes> ?w .
}"""

DG_QUERIES = [
    ("fig_query", FIG_QUERY),
    ("scan_both_vars", "SELECT * WHERE { ?x <:likes> ?w . }"),
    ("scan_const_subject", "SELECT * WHERE { <A> <:likes> ?w . }"),
    ("scan_const_object", "SELECT * WHERE { ?x <:follows> <D> . }"),
    ("scan_self_loop", "SELECT * WHERE { ?x <:likes> ?x . }"),
    ("scan_unknown_subject", "SELECT * WHERE { <Z> <:likes> ?w . }"),
    ("scan_both_const_hit", "SELECT * WHERE { <A> <:likes> <I1> . }"),
    ("scan_both_const_miss", "SELECT * WHERE { <A> <:likes> <h> . }"),
    ("unknown_predicate_first", "SELECT ?a ?b WHERE { ?a <:nope> ?b . ?a <:likes> ?c . }"),
    ("all_distinct_predicates",
     "SELECT * WHERE { ?a <:likes> ?b . ?a <:follows> ?c . ?c <:related> ?d . }"),
    ("cross_product", "SELECT * WHERE { ?a <:related> ?b . ?c <:related> ?d . }"),
    ("distinct", "SELECT DISTINCT ?w WHERE { ?x <:likes> ?w . }"),
    ("chain_follows_related", "SELECT * WHERE { ?a <:follows> ?b . ?b <:related> ?c . }"),
    ("two_hop_follows", "SELECT * WHERE { ?a <:follows> ?b . ?b <:follows> ?c . }"),
    ("triangle_cycle", "SELECT * WHERE { ?a <:follows> ?b . ?b <:follows> ?c . ?a <:follows> ?c . }"),
    ("both_vars_shared",
     "SELECT * WHERE { ?a <:follows> ?b . ?b <:follows> ?c . ?c <:follows> ?a . }"),
    ("semi_join_const_object", "SELECT * WHERE { ?x <:likes> ?w . ?x <:follows> <B> . }"),
    ("semi_join_const_subject", "SELECT * WHERE { ?x <:follows> ?y . <B> <:follows> ?y . }"),
    ("const_connected_cross",
     "SELECT * WHERE { <A> <:likes> ?w . <A> <:follows> ?y . }"),
    ("gate_true", "SELECT * WHERE { ?x <:likes> ?w . <A> <:follows> <B> . }"),
    ("gate_false", "SELECT * WHERE { ?x <:likes> ?w . <A> <:follows> <C> . }"),
    ("empty_join_right", "SELECT * WHERE { ?x <:likes> ?w . ?w <:nope> ?z . }"),
    ("self_loop_join", "SELECT * WHERE { ?x <:follows> ?y . ?y <:likes> ?y . }"),
    ("select_star_all_constants", "SELECT * WHERE { <A> <:likes> <I1> . <C> <:likes> <I2> . }"),
    ("distinct_pair", "SELECT DISTINCT ?x ?y WHERE { ?x <:follows> ?y . ?y <:follows> ?z . }"),
    ("star3", "SELECT * WHERE { ?x <:likes> ?a . ?x <:follows> ?b . ?x <:likes> ?c . }"),
    ("chain3", "SELECT * WHERE { ?x <:follows> ?y . ?y <:follows> ?z . ?z <:related> ?w . }"),
]

BUDGET_CASES = [
    ("fig_query", FIG_QUERY, 1),
    ("fig_query", FIG_QUERY, 4),
    ("cross_product", "SELECT * WHERE { ?a <:related> ?b . ?c <:related> ?d . }", 3),
    ("two_hop_follows", "SELECT * WHERE { ?a <:follows> ?b . ?b <:follows> ?c . }", 2),
]


def run_reference(store, text, mode="sequential", budget=executor.DEFAULT_ROW_BUDGET):
    g = qparser.parse_query(text)
    q = qparser.bind_constants(g, store.dictionary)
    plan = planner.make_plan(q, store.stats)
    rep = executor.ExecutionReport()
    try:
        res = executor.execute(q, plan, store, mode=mode, worker_count=2, row_budget=budget,
                               report=rep)
    except ResourceLimitError as exc:
        return {"error": "ResourceLimitError", "message": str(exc)}
    return {
        "schema": list(res.schema),
        "rows": [list(r) for r in res.rows],
        "step_rows": [s.rows for s in rep.steps],
        "step_prealloc": [s.prealloc_total for s in rep.steps],
        "preparations": rep.preparations,
        "uses": rep.uses,
        "plan": [s.pattern.source.text() for s in plan.steps],
    }


def build_from_strings(triples):
    d = TermDictionary()
    enc = [storage.EncodedTriple(d.encode_node(s), d.encode_predicate(p), d.encode_node(o))
           for s, p, o in triples]
    return storage.build_store(d, enc)


def make_dg() -> None:
    store = build_from_strings(D_G_TRIPLES)
    out = HERE / "d_g"
    shutil.rmtree(out, ignore_errors=True)
    storage.persist(store, out)
    cases = []
    for name, text in DG_QUERIES:
        for mode in ("sequential", "parallel"):
            cases.append({"name": name, "query": text, "mode": mode, "budget": None,
                          "expected": run_reference(store, text, mode)})
    for name, text, budget in BUDGET_CASES:
        for mode in ("sequential", "parallel"):
            cases.append({"name": f"{name}_budget{budget}", "query": text, "mode": mode,
                          "budget": budget, "expected": run_reference(store, text, mode, budget)})
    (HERE / "golden_dg.json").write_text(json.dumps(cases, indent=1))


def query_text(graph) -> str:
    def show(t):
        return t if t.startswith("?") else f"<{t}>"

    body = " ".join(f"{show(p.s)} {show(p.p)} {show(p.o)} ." for p in graph.patterns)
    return f"SELECT * WHERE {{ {body} }}"


def make_c3() -> None:
    from conftest import random_connected_query  # reference tests/conftest.py:69-93

    rng = random.Random(20240817)  # test_acceptance.py:138
    trials = []
    for trial in range(200):
        cfg = generate.GenConfig(triples=rng.randint(50, 1000), predicates=rng.randint(2, 8),
                                 zipf_s=1.0, seed=trial)
        triples = list(generate.generate_triples(cfg))
        store = build_from_strings(triples)
        graph = random_connected_query(rng, triples, rng.randint(1, 6), rng.randint(0, 2))
        text = query_text(graph)
        assert qparser.parse_query(text).patterns == graph.patterns
        exp = run_reference(store, text)
        par = run_reference(store, text, mode="parallel")
        rows = [tuple(r) for r in exp.pop("rows")]
        assert sorted(rows) == sorted(tuple(r) for r in par["rows"])
        entry = {"trial": trial, "triples": cfg.triples, "predicates": cfg.predicates,
                 "zipf": 1.0, "seed": trial, "query": text, "count": len(rows),
                 "fingerprint": [str(v) for v in fingerprint(rows)], **exp}
        if len(rows) <= 200:
            entry["rows"] = [list(r) for r in rows]
        trials.append(entry)
    (HERE / "golden_c3.json").write_text(json.dumps(trials, indent=0))


def make_lubm1() -> None:
    gen = REPO / "oracle" / "_build" / "gsmgen"
    subprocess.run(["make", "-s", "-C", str(REPO / "oracle")], check=True)
    with tempfile.TemporaryDirectory() as tmp:
        d = Path(tmp) / "lubm1"
        subprocess.run([str(gen), "lubm", "--univ", "1", "--seed", "0", "--out", str(d)],
                       check=True, stdout=subprocess.DEVNULL)
        store = storage.load(d)
        out = []
        for qf in sorted((REPO / "datagen" / "queries" / "lubm").glob("*.rq")):
            text = qf.read_text()
            exp = run_reference(store, text)
            rows = [tuple(r) for r in exp.pop("rows")]
            entry = {"name": qf.stem, "count": len(rows),
                     "fingerprint": [str(v) for v in fingerprint(rows)], **exp}
            if len(rows) <= 100:
                entry["rows"] = [list(r) for r in rows]
            out.append(entry)
    (HERE / "golden_lubm1.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    make_dg()
    make_c3()
    make_lubm1()
    print("golden vectors written to", HERE)
