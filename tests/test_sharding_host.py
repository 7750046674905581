"""Host-side logic of the sharded mode (no GPU): the id-range owner function
(must match the device's shard_of) and the exchange schedule."""

from __future__ import annotations

import numpy as np

from paper_1807_07691_b200 import _lib
from paper_1807_07691_b200.sharded import exchange_plan, pattern_vars
from paper_1807_07691_b200.storage import shard_owner


def _pat(s, o, pid=1):
    p = _lib.Pattern()
    p.s_var, p.o_var = (s, o)
    p.s_const = 7 if s < 0 else 0
    p.o_const = 9 if o < 0 else 0
    p.pid = pid
    return p


def test_shard_owner_ranges():
    n = 1000
    ids = np.arange(1, n + 1)
    for parts in (1, 2, 3, 7, 8):
        o = shard_owner(ids, n, parts)
        assert o.min() == 0 and o.max() == parts - 1
        assert np.all(np.diff(o) >= 0)  # contiguous id ranges
        counts = np.bincount(o, minlength=parts)
        assert counts.max() - counts.min() <= 1  # balanced
        # the device formula: (id - 1) * parts / node_count
        assert np.array_equal(o, ((ids - 1) * parts) // n)


def test_exchange_schedule():
    x, y, z, w = 0, 1, 2, 3
    # star on ?x after an R1 scan partitioned by ?x: no exchange at all
    star = [_pat(x, y), _pat(x, z, 2), _pat(x, w, 3)]
    assert [s["exchange"] for s in exchange_plan(star)] == [False, False]
    # chain ?x p ?y . ?y q ?z . ?z r ?w: every step re-keys
    chain = [_pat(x, y), _pat(y, z, 2), _pat(z, w, 3)]
    sched = exchange_plan(chain)
    assert [s["key"] for s in sched] == [y, z]
    assert [s["exchange"] for s in sched] == [True, True]
    assert sched[-1]["schema"] == [x, y, z, w]
    # R2 first step (?x p C) lives on the owner of C: the first join exchanges
    r2 = [_pat(x, -1), _pat(x, y, 2)]
    assert exchange_plan(r2)[0]["exchange"] is True
    # no shared variable -> cross product, no exchange
    cross = [_pat(x, y), _pat(z, w, 2)]
    assert exchange_plan(cross)[0]["kind"] == "cross"
    # join vars in left-schema order: J[0] decides the key (executor.py:343)
    tri = [_pat(x, y), _pat(y, z, 2), _pat(z, x, 3)]
    assert [s["key"] for s in exchange_plan(tri)] == [y, x]
    assert pattern_vars(_pat(x, x)) == [x]


def test_shard_byte_range_reads_match_owner_mask(store_factory):
    """load(shard=(i, n)) reads one contiguous byte range per pair file
    (storage._read_shard); it must select exactly the rows whose key the
    shard owns, and the shards must tile every file."""
    from pathlib import Path

    from paper_1807_07691_b200.storage import _read_shard, shard_id_range

    d = Path(store_factory("lubm", univ=1, seed=0))
    node_count = int((d / "meta").read_text().split()[3])
    for f in sorted(d.glob("p*.[so][os]")):
        full = np.fromfile(f, dtype="<u8").reshape(-1, 2)
        for parts in (1, 2, 3, 8):
            got = []
            for i in range(parts):
                lo, hi = shard_id_range(i, parts, node_count)
                part = _read_shard(f, lo, hi)
                exp = full[shard_owner(full[:, 0], node_count, parts) == i]
                assert np.array_equal(part, exp), (f.name, parts, i)
                got.append(part)
            assert sum(len(p) for p in got) == len(full)
