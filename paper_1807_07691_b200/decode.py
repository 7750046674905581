"""Result decoding on the device.

The reference CLI prints a result as TSV, one ``format_term(decode_node(v))``
per cell (/root/reference/pkg/src/gsmat/cli.py:101-105, dictionary.py:84-87,
qparser.py:71-78) — a Python loop over every cell.  Here the node dictionary
is uploaded once (raw ``nodes.dict`` bytes + line offsets), every term is
rendered on the device, and a result table becomes its TSV body in one call
(``gsm_decode_rows``: per-row byte counts, scan, warp-per-row copy).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .dictionary import escape_term


def _escape_literal(text: str) -> str:
    """qparser._escape_literal (qparser.py:60-67)."""
    return (text.replace("\\", "\\\\").replace('"', '\\"').replace("\n", "\\n")
            .replace("\r", "\\r").replace("\t", "\\t"))


def format_term(term: str) -> str:
    """qparser.format_term (qparser.py:71-78): a canonical term in N-Triples
    surface syntax (host restatement, used by the tests as the checker)."""
    if term.startswith('"'):
        end = term.rfind('"')
        return '"' + _escape_literal(term[1:end]) + '"' + term[end + 1:]
    if term.startswith("_:"):
        return term
    return f"<{term}>"


def _node_lines(dictionary) -> tuple[bytes, np.ndarray, np.ndarray]:
    nodes = getattr(dictionary, "_nodes", None)
    if nodes is not None:  # StoreDictionary: the nodes.dict file as read
        return nodes.buf, nodes.starts, nodes.ends
    # a reference TermDictionary: re-escape its terms into nodes.dict form
    lines = [escape_term(t).encode("utf-8") for t in dictionary.node_terms]
    lens = np.fromiter((len(x) for x in lines), dtype=np.int64, count=len(lines))
    ends = np.cumsum(lens + 1) - 1
    starts = ends - lens
    return b"\n".join(lines) + (b"\n" if lines else b""), starts, ends


def upload_dictionary(store) -> None:
    """Render the store's node terms on its device (once per store)."""
    if getattr(store, "_dict_on_device", False):
        return
    buf, starts, ends = _node_lines(store.dictionary)
    starts = np.ascontiguousarray(starts, dtype=np.int64)
    ends = np.ascontiguousarray(ends, dtype=np.int64)
    _lib.check(_lib.lib().gsm_store_put_dictionary(
        store._handle, buf, len(buf), starts.ctypes.data, ends.ctypes.data, len(starts)))
    store._dict_on_device = True


class _Text:
    """A decoded TSV body held by the library (gsm_text): ``view`` is a
    memoryview of its bytes, valid until ``close()``."""

    def __init__(self, store, rows: np.ndarray):
        from .storage import from_store

        store = from_store(store)
        upload_dictionary(store)
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        if rows.ndim != 2:
            raise ValueError("rows must be a 2-D (n, k) array")
        n, k = rows.shape
        self._L = _lib.lib()
        self._txt = C.c_void_p()
        _lib.check(self._L.gsm_decode_rows(store._handle, rows.ctypes.data if rows.size else None,
                                           n, k, C.byref(self._txt)))
        data, nbytes = C.c_void_p(), C.c_int64()
        _lib.check(self._L.gsm_text_data(self._txt, C.byref(data), C.byref(nbytes)))
        self.nbytes = int(nbytes.value)
        self.view = (memoryview((C.c_char * self.nbytes).from_address(data.value)).cast("B")
                     if self.nbytes else memoryview(b""))

    def close(self) -> None:
        if self._txt:
            self.view.release()
            self._L.gsm_text_free(self._txt)
            self._txt = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def decode_rows(store, rows: np.ndarray) -> bytes:
    """TSV body of a (n, k) node-id table: per row the k rendered terms joined
    by tabs and a newline (cli.py:103-105).  Raises UnknownIdError for an id
    outside the dictionary (dictionary.py:84-87)."""
    with _Text(store, rows) as t:
        return t.view.tobytes()


def write_tsv(result, store, fh) -> int:
    """Write what ``gsmat query`` prints (cli.py:101-105) to a binary file
    object without building a Python str or bytes: the library's decoded
    buffer is written as it is; returns the bytes written."""
    head = ("\t".join(result.schema) + "\n").encode("utf-8")
    fh.write(head)
    with _Text(store, result.array) as t:
        fh.write(t.view)
        return len(head) + t.nbytes


def result_tsv(result, store) -> str:
    """What ``gsmat query`` prints for a result (cli.py:101-105): the schema
    line, then one decoded line per row."""
    with _Text(store, result.array) as t:
        body = str(t.view, "utf-8")  # decoded straight from the library's buffer
    return "\t".join(result.schema) + "\n" + body
