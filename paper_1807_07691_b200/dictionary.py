"""Read-only, array-backed term dictionary over a store's ``*.dict`` files.

Same lookup/decode contract as the reference's TermDictionary
(/root/reference/pkg/src/gsmat/dictionary.py:46-125): dense 1-based ids in
file line order, ``lookup_*`` returns None for unknown terms, ``decode_*``
raises UnknownIdError.  It does not build a Python dict of every node (the
reference's costs ~115 B per node): nodes.dict is kept as one
bytes buffer plus a numpy line-offset array; lookups search the buffer.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from .errors import StoreFormatError, UnknownIdError

NODES_FILE = "nodes.dict"
PREDS_FILE = "preds.dict"

_ESC = {"\\": "\\", "n": "\n", "r": "\r", "t": "\t"}


def escape_term(term: str) -> str:
    """dictionary.escape_term (dictionary.py:18-25)."""
    return (
        term.replace("\\", "\\\\").replace("\n", "\\n").replace("\r", "\\r").replace("\t", "\\t")
    )


def unescape_term(text: str) -> str:
    """dictionary.unescape_term (dictionary.py:28-43)."""
    if "\\" not in text:
        return text
    out: list[str] = []
    i, n = 0, len(text)
    while i < n:
        c = text[i]
        if c == "\\" and i + 1 < n:
            out.append(_ESC.get(text[i + 1], text[i + 1]))
            i += 2
        else:
            out.append(c)
            i += 1
    return "".join(out)


class _TermFile:
    """One ``*.dict`` file: bytes + start offset of every line."""

    def __init__(self, path: Path):
        if not path.exists():
            raise StoreFormatError(f"missing dictionary file {path}")
        self.buf = path.read_bytes()
        arr = np.frombuffer(self.buf, dtype=np.uint8)
        nl = np.flatnonzero(arr == 10)
        ends = nl
        if len(self.buf) and (len(nl) == 0 or nl[-1] != len(self.buf) - 1):
            ends = np.append(nl, len(self.buf))  # last line without newline
        self.ends = ends.astype(np.int64)
        self.starts = np.concatenate(([0], self.ends[:-1] + 1)).astype(np.int64) if len(ends) else np.zeros(0, np.int64)
        self.count = int(len(self.ends))
        self._cache: dict[str, int | None] = {}

    def term(self, id_: int) -> str:
        a, b = int(self.starts[id_ - 1]), int(self.ends[id_ - 1])
        return unescape_term(self.buf[a:b].decode("utf-8"))

    def lookup(self, term: str) -> int | None:
        hit = self._cache.get(term, -1)
        if hit != -1:
            return hit  # type: ignore[return-value]
        needle = escape_term(term).encode("utf-8")
        found: int | None = None
        if self.buf.startswith(needle + b"\n") or self.buf == needle:
            found = 1
        else:
            pos = self.buf.find(b"\n" + needle + b"\n")
            if pos < 0 and self.buf.endswith(b"\n" + needle):
                pos = len(self.buf) - len(needle) - 1
            if pos >= 0:
                found = int(np.searchsorted(self.starts, pos + 1)) + 1
        self._cache[term] = found
        return found


class StoreDictionary:
    """Drop-in for TermDictionary on a persisted store (read-only)."""

    def __init__(self, directory: Path | str):
        directory = Path(directory)
        self._nodes = _TermFile(directory / NODES_FILE)
        self._preds = _TermFile(directory / PREDS_FILE)
        self.pred_index = {self._preds.term(i): i for i in range(1, self._preds.count + 1)}

    @property
    def node_count(self) -> int:
        return self._nodes.count

    @property
    def predicate_count(self) -> int:
        return self._preds.count

    def lookup_node(self, term: str) -> int | None:
        return self._nodes.lookup(term)

    def lookup_predicate(self, term: str) -> int | None:
        return self.pred_index.get(term)

    def decode_node(self, id_: int) -> str:
        if not 1 <= id_ <= self._nodes.count:
            raise UnknownIdError("node", id_)
        return self._nodes.term(id_)

    def decode_predicate(self, id_: int) -> str:
        if not 1 <= id_ <= self._preds.count:
            raise UnknownIdError("predicate", id_)
        return self._preds.term(id_)

    def save(self, directory: Path | str) -> None:
        """TermDictionary.save (dictionary.py:95-104): the files as read."""
        directory = Path(directory)
        for name, tf in ((NODES_FILE, self._nodes), (PREDS_FILE, self._preds)):
            data = tf.buf
            if data and not data.endswith(b"\n"):
                data += b"\n"
            (directory / name).write_bytes(data)


class TermDictionary:
    """dictionary.TermDictionary (dictionary.py:46-125): two first-occurrence
    ordered bijections (nodes, predicates), dense 1-based ids, the reference's
    one-term-per-line persistence.  Host-side state of the build path
    (:func:`paper_1807_07691_b200.storage.build_store`)."""

    def __init__(self) -> None:
        self.node_terms: list[str] = []
        self.pred_terms: list[str] = []
        self.node_index: dict[str, int] = {}
        self.pred_index: dict[str, int] = {}

    def encode_node(self, term: str) -> int:
        nid = self.node_index.get(term)
        if nid is None:
            self.node_terms.append(term)
            nid = len(self.node_terms)
            self.node_index[term] = nid
        return nid

    def encode_predicate(self, term: str) -> int:
        pid = self.pred_index.get(term)
        if pid is None:
            self.pred_terms.append(term)
            pid = len(self.pred_terms)
            self.pred_index[term] = pid
        return pid

    def lookup_node(self, term: str) -> int | None:
        return self.node_index.get(term)

    def lookup_predicate(self, term: str) -> int | None:
        return self.pred_index.get(term)

    def decode_node(self, id_: int) -> str:
        if not 1 <= id_ <= len(self.node_terms):
            raise UnknownIdError("node", id_)
        return self.node_terms[id_ - 1]

    def decode_predicate(self, id_: int) -> str:
        if not 1 <= id_ <= len(self.pred_terms):
            raise UnknownIdError("predicate", id_)
        return self.pred_terms[id_ - 1]

    @property
    def node_count(self) -> int:
        return len(self.node_terms)

    @property
    def predicate_count(self) -> int:
        return len(self.pred_terms)

    def save(self, directory: Path | str) -> None:
        directory = Path(directory)
        for name, terms in ((NODES_FILE, self.node_terms), (PREDS_FILE, self.pred_terms)):
            with open(directory / name, "w", encoding="utf-8", newline="\n") as fh:
                for term in terms:
                    fh.write(escape_term(term))
                    fh.write("\n")

    @classmethod
    def load(cls, directory: Path | str) -> "TermDictionary":
        directory = Path(directory)
        d = cls()
        for name, encode in ((NODES_FILE, d.encode_node), (PREDS_FILE, d.encode_predicate)):
            path = directory / name
            if not path.exists():
                raise StoreFormatError(f"missing dictionary file {path}")
            with open(path, encoding="utf-8", newline="\n") as fh:
                for raw in fh:
                    encode(unescape_term(raw.rstrip("\n")))
        return d
