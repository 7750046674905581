"""datagen/gsmgen writes the reference store format, byte-identical to what
the reference's own ``gsmat build`` produces from the same N-Triples, and its
power-law mode reproduces ``gsmat gen`` (generate.py) bit for bit."""

from __future__ import annotations

import subprocess
import sys

import numpy as np
import pytest

from conftest import REPO, reference_available
from oracle import oracle as orc


def _store_files(d):
    return sorted(p.name for p in d.iterdir())


def _check_invariants(d):
    """SPEC.md:155-162 / storage.py invariants on a persisted store."""
    meta = (d / "meta").read_text().splitlines()
    assert meta[0] == "GSMAT1"
    triples, preds, nodes = (int(x) for x in meta[1:4])
    node_lines = (d / "nodes.dict").read_bytes().count(b"\n")
    assert node_lines == nodes
    total = 0
    for raw in (d / "stats.tsv").read_text().splitlines():
        pid, card, ds, do = (int(x) for x in raw.split("\t"))
        so = np.fromfile(d / f"p{pid}.so", dtype="<u8").reshape(-1, 2)
        os_ = np.fromfile(d / f"p{pid}.os", dtype="<u8").reshape(-1, 2)
        assert so.shape[0] == card == os_.shape[0]
        key_so = so[:, 0] * (1 << 32) + so[:, 1]
        key_os = os_[:, 0] * (1 << 32) + os_[:, 1]
        assert np.all(np.diff(key_so.astype(np.uint64)) > 0)  # sorted, no duplicates
        assert np.all(np.diff(key_os.astype(np.uint64)) > 0)
        assert len(np.unique(so[:, 0])) == ds and len(np.unique(os_[:, 0])) == do
        assert set(map(tuple, so.tolist())) == {(s, o) for o, s in os_.tolist()}
        assert so.min() >= 1 and so.max() <= nodes
        total += card
    assert total == triples
    assert len([l for l in (d / "stats.tsv").read_text().splitlines() if l]) == preds


@pytest.mark.parametrize("kind,args", [
    ("lubm", ["--univ", "1", "--seed", "0"]),
    ("lubm", ["--univ", "2", "--seed", "5"]),
    ("powerlaw", ["--triples", "5000", "--predicates", "7", "--seed", "11"]),
    ("watdiv", ["--scale", "1", "--seed", "2"]),
])
def test_generated_store_invariants(tmp_path, kind, args):
    d = tmp_path / "s"
    orc.gsmgen(kind, *args, "--out", str(d))
    _check_invariants(d)


def test_lubm_deterministic(tmp_path):
    a, b = tmp_path / "a", tmp_path / "b"
    orc.gsmgen("lubm", "--univ", "1", "--seed", "3", "--out", str(a))
    orc.gsmgen("lubm", "--univ", "1", "--seed", "3", "--out", str(b))
    for f in _store_files(a):
        assert (a / f).read_bytes() == (b / f).read_bytes()


@pytest.mark.skipif(not reference_available(), reason="reference package not installed")
@pytest.mark.parametrize("kind,args", [
    ("lubm", ["--univ", "1", "--seed", "0"]),
    ("powerlaw", ["--triples", "20000", "--predicates", "6", "--seed", "3"]),
    ("watdiv", ["--scale", "1", "--seed", "0"]),
])
def test_byte_identical_to_reference_build(tmp_path, kind, args):
    mine, ref = tmp_path / "mine", tmp_path / "ref"
    nt = tmp_path / "data.nt"
    orc.gsmgen(kind, *args, "--out", str(mine), "--nt", str(nt))
    env_path = str(REPO / "oracle" / "_ref")
    subprocess.run([sys.executable, "-c",
                    f"import sys; sys.path.insert(0, {env_path!r}); from gsmat import cli; "
                    f"sys.exit(cli.main(['build', '--input', {str(nt)!r}, '--out', {str(ref)!r}]))"],
                   check=True, stdout=subprocess.DEVNULL)
    assert _store_files(mine) == _store_files(ref)
    for f in _store_files(ref):
        assert (mine / f).read_bytes() == (ref / f).read_bytes(), f


@pytest.mark.skipif(not reference_available(), reason="reference package not installed")
def test_powerlaw_matches_reference_generator(tmp_path):
    """gsmgen powerlaw == generate.generate_ntriples (CPython MT19937 restated)."""
    from gsmat import generate

    nt = tmp_path / "mine.nt"
    orc.gsmgen("powerlaw", "--triples", "30000", "--predicates", "9", "--zipf", "1.0",
               "--seed", "12345678901", "--out", str(tmp_path / "s"), "--nt", str(nt))
    cfg = generate.GenConfig(30000, 9, 1.0, seed=12345678901)
    ref = "".join(line + "\n" for line in generate.generate_ntriples(cfg))
    assert nt.read_text() == ref
