#!/usr/bin/env python
"""Golden stores for the ingest path, built by the REFERENCE ``gsmat build``
(cli._cmd_build, /root/reference/pkg/src/gsmat/cli.py:64-82) from the
installed reference (oracle/_ref).  Writes <name>.nt and <name>_store/ next
to this script; tests/test_ingest.py requires our build to reproduce every
file byte for byte.  Run here (the reference is importable); commit outputs.
    python tests/golden/ingest/make_ingest_golden.py
"""
from __future__ import annotations

import random
import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[2]
sys.path.append(str(REPO / "oracle" / "_ref"))

from gsmat import cli  # noqa: E402

TRICKY = r'''# comment line
<http://ex.org/s1> <http://ex.org/p1> <http://ex.org/o1> .
<http://ex.org/s1> <http://ex.org/p1> <http://ex.org/o1> .
_:b1 <http://ex.org/p2> "plain" .
_:b1 <http://ex.org/p2> "with \"quotes\" and \\ backslash" .
_:b1 <http://ex.org/p2> "multi\nline\ttab\rcr"@en-GB .
<http://ex.org/s2>	<http://ex.org/p3>   "1"^^<http://www.w3.org/2001/XMLSchema#int>  .   # trailing comment
   <http://ex.org/s2> <http://ex.org/p1> _:b2.
<http://ex.org/s3> <http://ex.org/p2> "café \U0001F600 \b\f\'" .
<http://ex.org/o1> <http://ex.org/p1> <http://ex.org/s1> .
<http://ex.org/s1> <http://ex.org/p3> <http://ex.org/s1> .
_:b2 <http://ex.org/p3> _:b1 .

<http://ex.org/s4> <http://ex.org/p4> "tab\tin literal"@de .
<http://ex.org/s4> <http://ex.org/p4> "" .
<http://ex.org/s5> <http://ex.org/p1> <http://ex.org/s4> .
<http://ex.org/ünï> <http://ex.org/p1> <http://ex.org/s5> .
_:a.b-c_d <http://ex.org/p4> _:x.y .
'''


def random_nt(rng: random.Random, n: int) -> str:
    nodes = [f"<http://ex.org/n{i}>" for i in range(n // 6)] + [f"_:b{i}" for i in range(20)]
    preds = [f"<http://ex.org/p{i}>" for i in range(9)]
    lits = ['"v%d"' % i for i in range(40)] + ['"t%d"@en' % i for i in range(5)] + \
        ['"%d"^^<http://www.w3.org/2001/XMLSchema#int>' % i for i in range(5)] + \
        ['"esc\\t%d\\n"' % i for i in range(3)]
    lines = []
    for _ in range(n):
        s = rng.choice(nodes[: len(nodes) // 2 + 5] if rng.random() < 0.7 else nodes)
        p = preds[min(int(rng.expovariate(0.6)), len(preds) - 1)]
        o = rng.choice(lits) if rng.random() < 0.2 else rng.choice(nodes)
        lines.append(f"{s} {p} {o} .")
        if rng.random() < 0.03:
            lines.append(lines[rng.randrange(len(lines))])  # duplicates
        if rng.random() < 0.01:
            lines.append("# comment")
    return "\n".join(lines) + "\n"


def make(name: str, text: str, newline: str = "\n") -> None:
    nt = HERE / f"{name}.nt"
    nt.write_bytes(text.replace("\n", newline).encode("utf-8"))
    out = HERE / f"{name}_store"
    if out.exists():
        shutil.rmtree(out)
    assert cli.main(["build", "--input", str(nt), "--out", str(out)]) == 0


if __name__ == "__main__":
    make("tricky", TRICKY)
    make("tricky_crlf", TRICKY, newline="\r\n")
    make("random", random_nt(random.Random(20240817), 4000))
