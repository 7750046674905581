import sys, os, json, subprocess
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1807_07691_b200 as g
from oracle import oracle as orc
subprocess.run(["oracle/_build/gsmgen", "lubm", "--univ", "2", "--seed", "4", "--out", "/tmp/l2"], check=True, stdout=subprocess.DEVNULL)
st = g.load("/tmp/l2")
prep = orc.PreparedStore(st.matrices)
qs = sorted(["datagen/queries/lubm/" + f for f in os.listdir("datagen/queries/lubm")]) + sorted(["datagen/queries/lubm_complex/" + f for f in os.listdir("datagen/queries/lubm_complex")])
for f in qs:
    q = g.bind_constants(g.parse_query(open(f).read()), st.dictionary); p = g.make_plan(q, st.stats)
    runs = []
    try:
        for _ in range(2):
            rep = g.ExecutionReport()
            r = g.execute(q, p, st, report=rep, row_budget=1 << 62)
            runs.append((orc.fingerprint_array(r.array), [s.rows for s in rep.steps], [s.prealloc_total for s in rep.steps], rep.kinds))
    except Exception as e:
        print("EXC", f, e); continue
    rows, sr, sp = orc.run(prep, [s.pattern for s in p.steps], q.projection, q.distinct)
    import numpy as np
    fo = orc.fingerprint_array(np.asarray(rows, dtype=np.uint32).reshape(len(rows), len(q.projection)))
    ok = runs[0][0] == runs[1][0] == fo and runs[0][1] == runs[1][1] == sr and runs[0][2] == runs[1][2] == sp
    print("OK " if ok else "BAD", f.split("/")[-1], runs[0][1:], "oracle", sr, sp, "" if ok else (runs[0][0], runs[1][0], fo))
