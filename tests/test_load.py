"""storage.load: the reference's StoreFormatError checks (storage.py:222-271,
test_storage.py:116-131) and the loader fast path (gsm_store_load_files).

Host-side checks (missing store, bad magic, truncated pair file, count
mismatches) raise before any device work and run on CPU; the checks the
device makes while streaming the pair files (key order -> the reference's
ValueError "not sorted", value order, ids >= 2^32) and the agreement of the
fast path with the array upload path need the GPU.
"""

from __future__ import annotations

import shutil

import numpy as np
import pytest

import paper_1807_07691_b200 as g
from conftest import GOLDEN, lubm_queries
from oracle import oracle as orc


def _copy_dg(tmp_path, name="s"):
    d = tmp_path / name
    shutil.copytree(GOLDEN / "d_g", d)
    return d


def test_load_missing_and_bad_magic(tmp_path):
    with pytest.raises(g.StoreFormatError, match="missing"):
        g.load(tmp_path / "nowhere")
    bad = tmp_path / "bad"
    bad.mkdir()
    (bad / "meta").write_text("WRONG9\n")
    with pytest.raises(g.StoreFormatError, match="bad magic"):
        g.load(bad)


def test_load_truncated_pair_file(tmp_path):
    d = _copy_dg(tmp_path)
    so = d / "p1.so"
    so.write_bytes(so.read_bytes()[:-5])
    with pytest.raises(g.StoreFormatError, match="truncated|pairs"):
        g.load(d)


def test_load_count_mismatches(tmp_path):
    d = _copy_dg(tmp_path, "a")
    so = d / "p1.so"
    so.write_bytes(so.read_bytes()[:-16])  # one pair fewer than stats declares
    with pytest.raises(g.StoreFormatError, match="stats declares"):
        g.load(d)
    d = _copy_dg(tmp_path, "b")
    os_ = d / "p2.os"
    os_.write_bytes(os_.read_bytes() + os_.read_bytes()[:16])
    with pytest.raises(g.StoreFormatError, match="pairs but"):
        g.load(d)
    d = _copy_dg(tmp_path, "c")
    (d / "p3.so").unlink()
    with pytest.raises(g.StoreFormatError, match="missing pair files"):
        g.load(d)


def _rewrite(path, fn):
    a = np.fromfile(path, dtype="<u8").reshape(-1, 2)
    fn(a)
    a.astype("<u8").tofile(path)


@pytest.mark.gpu
def test_load_device_checks(tmp_path):
    # key order broken -> build_aux's ValueError (storage.py:44-45)
    d = _copy_dg(tmp_path, "k")
    _rewrite(d / "p1.so", lambda a: a.__setitem__(slice(None), a[::-1].copy()))
    with pytest.raises(ValueError, match="not sorted"):
        g.load(d)
    # value order inside a run broken -> StoreFormatError
    d = _copy_dg(tmp_path, "v")
    a = np.fromfile(d / "p1.so", dtype="<u8").reshape(-1, 2)
    keys, counts = np.unique(a[:, 0], return_counts=True)
    k = keys[np.argmax(counts)]
    assert counts.max() >= 2
    idx = np.nonzero(a[:, 0] == k)[0]

    def swap(x):
        x[idx[0], 1], x[idx[1], 1] = x[idx[1], 1], x[idx[0], 1]
    _rewrite(d / "p1.so", swap)
    with pytest.raises(g.StoreFormatError, match="not sorted by"):
        g.load(d)
    # ids beyond 2^32
    d = _copy_dg(tmp_path, "w")
    _rewrite(d / "p2.os", lambda x: x.__setitem__((-1, 1), np.uint64(1) << np.uint64(33)))
    with pytest.raises(g.StoreFormatError, match="2\\^32"):
        g.load(d)


@pytest.mark.gpu
def test_fast_loader_matches_array_upload(store_factory):
    """load() streams the pair files (gsm_store_load_files); load(shard=(0, 1))
    uploads host arrays (gsm_store_put_predicate_shard).  Same device bytes,
    same answers, same host aux (constant scans), same host views."""
    d = store_factory("lubm", univ=2, seed=4)
    a = g.load(d)
    b = g.load(d, shard=(0, 1))
    assert a.device_bytes() == b.device_bytes()
    for pid in a.matrices:
        assert np.array_equal(np.asarray(a.matrices[pid].so), b.matrices[pid].so)
        assert np.array_equal(np.asarray(a.matrices[pid].os), b.matrices[pid].os)
    for _, text in lubm_queries():
        qa = g.bind_constants(g.parse_query(text), a.dictionary)
        pa = g.make_plan(qa, a.stats)
        ra, rb = g.ExecutionReport(), g.ExecutionReport()
        x = g.execute(qa, pa, a, report=ra).array
        y = g.execute(qa, pa, b, report=rb).array
        assert orc.fingerprint_array(x) == orc.fingerprint_array(y)
        assert [s.rows for s in ra.steps] == [s.rows for s in rb.steps]


@pytest.mark.gpu
def test_fast_loader_multi_chunk(store_factory):
    """Predicates larger than one 2M-pair chunk, and more chunks than the
    loader's 8 pinned slots, so chunk boundaries and slot reuse are crossed."""
    d = store_factory("powerlaw", triples=20_000_000, predicates=3, seed=1)
    a = g.load(d)
    b = g.load(d, shard=(0, 1))
    assert max(m.cardinality for m in a.matrices.values()) > (1 << 21)
    assert sum(-(-2 * m.cardinality // (1 << 21)) for m in a.matrices.values()) > 8
    text = "SELECT * WHERE { ?x <p1> ?y . ?y <p2> ?z . }"
    qa = g.bind_constants(g.parse_query(text), a.dictionary)
    pa = g.make_plan(qa, a.stats)
    x = g.execute(qa, pa, a, row_budget=1 << 62).array
    y = g.execute(qa, pa, b, row_budget=1 << 62).array
    assert len(x) > 0
    assert orc.fingerprint_array(x) == orc.fingerprint_array(y)
