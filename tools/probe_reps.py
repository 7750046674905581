#!/usr/bin/env python
"""Per-repetition device time of the bench's expand probes (the first run is
the single-pass kernel, later runs may take the chunk-balanced path)."""
import sys
import tempfile
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
import bench  # noqa: E402
import paper_1807_07691_b200 as g  # noqa: E402

with tempfile.TemporaryDirectory() as tmp:
    store = g.load(bench._gen_store(Path(tmp), 10, 0), device=0)
    for name, text in bench.PROBES:
        q = g.bind_constants(g.parse_query(text), store.dictionary)
        plan = g.make_plan(q, store.stats)
        ts = []
        for _ in range(6):
            rep = g.ExecutionReport()
            g.execute(q, plan, store, report=rep, row_budget=1 << 62)
            ts.append(round(rep.steps[1].seconds * 1e6, 1))
        print(name, "expand step us per rep:", ts, "kernels", rep.kernels)
