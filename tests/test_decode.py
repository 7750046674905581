"""Result decoding (gsm_store_put_dictionary / gsm_decode_rows) against the
reference CLI's output rules (cli.py:101-105, qparser.format_term
qparser.py:71-78, dictionary.unescape_term dictionary.py:28-43)."""

from __future__ import annotations

import shutil

import numpy as np
import pytest

import paper_1807_07691_b200 as g
from conftest import GOLDEN, lubm_queries, reference_available
from paper_1807_07691_b200.dictionary import escape_term

# Terms exercising every rendering rule: IRIs, blank nodes, literals with
# escapes inside the quotes, language tags / datatypes after the last quote,
# quotes inside the lexical form, stored escapes (\\ \n \r \t) and edge cases.
TRICKY = [
    "http://example.org/a",
    "_:b0",
    '"plain"',
    '"with \\"quotes\\" inside"@en',
    '"multi\nline\ttab\rcr"^^http://www.w3.org/2001/XMLSchema#string',
    '"back\\\\slash"',
    '"',
    '"unterminated',
    '""',
    "_",
    "_:",
    'iri"with"quote',
    "tab\tin\niri",
    '"a"b"c"@de',
    "",
    "x" * 300,
    '"' + "y\\" * 70 + '"@en-GB',
]


def test_format_term_matches_reference():
    if not reference_available():
        pytest.skip("reference package not installed")
    from gsmat import qparser

    for t in TRICKY:
        assert g.format_term(t) == qparser.format_term(t)


def _store_with_terms(tmp_path, terms):
    """The D_G store with its nodes.dict replaced by `terms` (ids unchanged
    for the first len(D_G) nodes; the pair files still refer to ids 1..9)."""
    d = tmp_path / "s"
    shutil.copytree(GOLDEN / "d_g", d)
    old = (d / "nodes.dict").read_text(encoding="utf-8").splitlines()
    lines = old + [escape_term(t) for t in terms]
    (d / "nodes.dict").write_text("\n".join(lines) + "\n", encoding="utf-8")
    meta = (d / "meta").read_text().splitlines()
    meta[3] = str(len(lines))
    (d / "meta").write_text("\n".join(meta) + "\n")
    return d, len(old)


@pytest.mark.gpu
def test_decode_worked_example():
    """test_cli.py:38-46: the fig query prints ?x ?y ?z ?w / <A> <B> <C> <I2>."""
    store = g.load(GOLDEN / "d_g")
    text = ("SELECT ?x ?y ?z ?w WHERE { ?x <:follows> ?y . ?y <:follows> ?z . "
            "?x <:likes> ?w . ?z <:likes> ?w . }")
    q = g.bind_constants(g.parse_query(text), store.dictionary)
    res = g.execute(q, g.make_plan(q, store.stats), store)
    assert g.result_tsv(res, store).splitlines() == ["?x\t?y\t?z\t?w", "<A>\t<B>\t<C>\t<I2>"]
    import io
    buf = io.BytesIO()
    assert g.write_tsv(res, store, buf) == len(buf.getvalue())
    assert buf.getvalue().decode("utf-8") == g.result_tsv(res, store)


@pytest.mark.gpu
def test_decode_rendering_rules(tmp_path):
    d, base = _store_with_terms(tmp_path, TRICKY)
    store = g.load(d)
    n = store.dictionary.node_count
    ids = np.arange(1, n + 1, dtype=np.uint32)
    rng = np.random.default_rng(3)
    for k in (1, 2, 3):
        rows = rng.choice(ids, size=(257, k)).astype(np.uint32)
        rows[: min(257, n), 0] = ids[: min(257, n)]
        body = g.decode_rows(store, rows).decode("utf-8")
        exp = "".join("\t".join(g.format_term(store.dictionary.decode_node(int(v))) for v in r) + "\n"
                      for r in rows)
        assert body == exp
    assert g.decode_rows(store, np.zeros((0, 2), np.uint32)) == b""
    assert g.decode_rows(store, np.zeros((3, 0), np.uint32)) == b"\n\n\n"
    with pytest.raises(g.UnknownIdError):
        g.decode_rows(store, np.array([[1, n + 1]], dtype=np.uint32))
    with pytest.raises(g.UnknownIdError):
        g.decode_rows(store, np.array([[0]], dtype=np.uint32))


@pytest.mark.gpu
def test_decode_lubm_results(store_factory):
    """Every LUBM query's decoded result equals the CLI's per-cell loop."""
    store = g.load(store_factory("lubm", univ=1, seed=0))
    dec = store.dictionary.decode_node
    for name, text in lubm_queries():
        q = g.bind_constants(g.parse_query(text), store.dictionary)
        res = g.execute(q, g.make_plan(q, store.stats), store)
        got = g.result_tsv(res, store)
        exp = "\t".join(res.schema) + "\n" + "".join(
            "\t".join(g.format_term(dec(v)) for v in row) + "\n" for row in res.rows)
        assert got == exp, name
