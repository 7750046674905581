"""Small workload for compute-sanitizer (SURVEY.md §5 race-detection row):
the D_G goldens in both budget modes (errors included), the first trials of
the reference's c3 campaign, LUBM-1 Q1-Q14 one by one (first run captures
the CUDA graph, the second replays it; PDL on) and as one execute_batch
(batch graph, concurrent streams, zero-copy results), DISTINCT, cross
products, and the table-level joins (counts-only preallocate included).
Every result is checked against the goldens so a sanitizer run is also a
parity run.  Usage: compute-sanitizer --tool memcheck python tools/sanitize_cases.py [n_c3]
"""

from __future__ import annotations

import json
import sys
import tempfile
from collections import Counter
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(REPO), str(REPO / "tests")]

import paper_1807_07691_b200 as g  # noqa: E402
from paper_1807_07691_b200 import tables as T  # noqa: E402
from oracle import oracle as orc  # noqa: E402

GOLDEN = REPO / "tests" / "golden"


def bag(rows):
    return Counter(tuple(int(v) for v in r) for r in rows)


def plan(store, text):
    q = g.bind_constants(g.parse_query(text), store.dictionary)
    return q, g.make_plan(q, store.stats)


def main() -> None:
    n_c3 = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    checks = 0
    dg = g.load(GOLDEN / "d_g")
    for case in json.loads((GOLDEN / "golden_dg.json").read_text()):
        exp = case["expected"]
        q, p = plan(dg, case["query"])
        budget = case["budget"] if case["budget"] is not None else 10**8
        try:
            res = g.execute(q, p, dg, mode=case["mode"], row_budget=budget)
            assert "error" not in exp and bag(res.rows) == bag(exp["rows"]), case["name"]
        except g.ResourceLimitError as e:
            assert exp.get("message") == str(e), case["name"]
        checks += 1
    with tempfile.TemporaryDirectory() as tmp:
        made = {}
        for t in json.loads((GOLDEN / "golden_c3.json").read_text())[:n_c3]:
            key = (t["triples"], t["predicates"], t["zipf"], t["seed"])
            if key not in made:
                d = f"{tmp}/pl{len(made)}"
                orc.gsmgen("powerlaw", "--triples", str(t["triples"]), "--predicates",
                           str(t["predicates"]), "--zipf", str(t["zipf"]), "--seed", str(t["seed"]),
                           "--out", d)
                made[key] = g.load(d)
            st = made[key]
            q, p = plan(st, t["query"])
            for mode in ("sequential", "parallel"):
                res = g.execute(q, p, st, mode=mode)
                assert [str(v) for v in orc.fingerprint_array(res.array)] == t["fingerprint"], t["trial"]
                checks += 1
        orc.gsmgen("lubm", "--univ", "1", "--seed", "0", "--out", f"{tmp}/lubm1")
        st = g.load(f"{tmp}/lubm1")
        gold = {x["name"]: x for x in json.loads((GOLDEN / "golden_lubm1.json").read_text())}
        items = []
        for f in sorted((REPO / "datagen" / "queries" / "lubm").glob("*.rq")):
            q, p = plan(st, f.read_text())
            items.append((q, p))
            for _ in range(3):  # capture, re-capture with grids from the rows seen, warm replay
                res = g.execute(q, p, st)
                assert [str(v) for v in orc.fingerprint_array(res.array)] == gold[f.stem]["fingerprint"]
                checks += 1
        # batch: capture, hinted re-capture, warm replay (k_init nodes off),
        # then one member's context runs another plan (its k_init back on)
        for rnd in range(5):
            if rnd == 3:
                g.execute_batch([items[0]], st)
            outs = g.execute_batch(items, st)
            for (q, p), res, f in zip(items, outs, sorted((REPO / "datagen" / "queries" / "lubm").glob("*.rq"))):
                assert [str(v) for v in orc.fingerprint_array(res.array)] == gold[f.stem]["fingerprint"]
                checks += 1
        # left-row chunks (forced), with the device fingerprint
        q, p = items[8]
        exp = gold[sorted((REPO / "datagen" / "queries" / "lubm").glob("*.rq"))[8].stem]["fingerprint"]
        res = g.execute(q, p, st, chunks=8)
        assert [str(v) for v in orc.fingerprint_array(res.array)] == exp
        assert [str(v) for v in g.execute_summary(q, p, st, chunks=4).fingerprint] == exp
        checks += 2
        ub = "PREFIX ub: <http://swat.cse.lehigh.edu/onto/univ-bench.owl#> "
        rdf = "PREFIX rdf: <http://www.w3.org/1999/02/22-rdf-syntax-ns#> "
        prep = orc.PreparedStore(st.matrices)
        for text in (ub + "SELECT DISTINCT ?d WHERE { ?x ub:memberOf ?d . ?x ub:takesCourse ?c . }",
                     rdf + ub + "SELECT * WHERE { ?x rdf:type ub:FullProfessor . ?y rdf:type ub:Course . }",
                     ub + "SELECT * WHERE { ?x ub:takesCourse ?c . ?y ub:takesCourse ?c . }"):
            q, p = plan(st, text)
            rows, _, _ = orc.run(prep, [s.pattern for s in p.steps], q.projection, q.distinct)
            res = g.execute(q, p, st, row_budget=1 << 62)
            assert bag(res.rows) == bag(rows)
            checks += 1
    a = g.BindingTable(("?a", "?b"), [(10, 20), (10, 30), (11, 20)])
    b = g.BindingTable(("?b", "?c"), [(20, 1), (20, 3), (30, 2), (30, 3)])
    assert T.sm_join(a, b, ["?b"]).rows == [(10, 20, 1), (10, 20, 3), (10, 30, 2), (10, 30, 3),
                                            (11, 20, 1), (11, 20, 3)]
    pp = T.preallocate(a, b, "?b")
    assert pp.total == 6 and pp.counts == [4, 2]
    assert len(T.cross_product(a, b)) == 12
    checks += 3
    print(f"sanitize cases ok: {checks} checks")


if __name__ == "__main__":
    main()
