import sys, os
sys.path.insert(0, ".")
import paper_1807_07691_b200 as g
st = g.load("tests/golden/d_g")
text = "SELECT ?x ?y ?z ?w WHERE { ?x <:follows> ?y . ?y <:follows> ?z . ?x <:likes> ?w . ?z <:likes> ?w . }"
q = g.bind_constants(g.parse_query(text), st.dictionary); p = g.make_plan(q, st.stats)
for rep in (None, g.ExecutionReport()):
    try:
        print("rep" if rep else "norep", g.execute(q, p, st, report=rep).rows)
    except Exception as e:
        print("ERR", rep is not None, e)
