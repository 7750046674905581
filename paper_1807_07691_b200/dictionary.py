"""Read-only, array-backed term dictionary over a store's ``*.dict`` files.

Same lookup/decode contract as the reference's TermDictionary
(/root/reference/pkg/src/gsmat/dictionary.py:46-125) for a persisted store:
dense 1-based ids in file line order, ``lookup_*`` returns None for unknown
terms, ``decode_*`` raises UnknownIdError.  Building a dictionary (encoding
new terms) is out of scope: ``build_store`` takes the caller's dictionary.  It does not build a Python dict of every node (the
reference's costs ~115 B per node): nodes.dict is kept as one
bytes buffer plus a numpy line-offset array; lookups search the buffer.
"""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np

from .errors import StoreFormatError, UnknownIdError

NODES_FILE = "nodes.dict"
PREDS_FILE = "preds.dict"

# One-term-per-line file format of nodes.dict / preds.dict
# (/root/reference/pkg/src/gsmat/dictionary.py:18-43): backslash, newline,
# carriage return and tab are written as two-character escapes; on reading,
# a backslash takes the next character literally unless it names one of
# those escapes, and a trailing lone backslash stays as it is.
_TO_FILE = str.maketrans({"\\": "\\\\", "\n": "\\n", "\r": "\\r", "\t": "\\t"})
_FROM_FILE = {"n": "\n", "r": "\r", "t": "\t"}
_ESCAPED = re.compile(r"\\(.)", re.S)


def escape_term(term: str) -> str:
    """A term as one line of a ``*.dict`` file."""
    return term.translate(_TO_FILE)


def unescape_term(text: str) -> str:
    """The term one line of a ``*.dict`` file encodes."""
    if "\\" not in text:
        return text
    return _ESCAPED.sub(lambda m: _FROM_FILE.get(m.group(1), m.group(1)), text)


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
