"""Store build from N-Triples: the drop-in for ``gsmat build``
(/root/reference/pkg/src/gsmat/cli.py:64-82).

``build(input, out)`` writes the same store directory as the reference's
``gsmat build --input input --out out`` — byte for byte — with the parse on
the host threads and the dictionary encoding and per-predicate
sort/deduplication on the GPU (csrc/gsm_ingest.cu).  ``parse_ntriples``
exposes the parse stage (qparser.read_ntriples, qparser.py:80-111).
"""

from __future__ import annotations

import ctypes as C
import struct
from pathlib import Path

from . import _lib


def parse_ntriples(data: str | bytes, threads: int = 0) -> list[tuple[str, str, str]]:
    """Canonical (subject, predicate, object) terms of every statement, in
    input order; ParseError("line N: ...") on the first malformed one."""
    buf = data.encode("utf-8") if isinstance(data, str) else bytes(data)
    L = _lib.lib()
    txt = C.c_void_p()
    _lib.check(L.gsm_ntriples_parse(buf, len(buf), int(threads), C.byref(txt)))
    try:
        ptr, n = C.c_void_p(), C.c_int64()
        _lib.check(L.gsm_text_data(txt, C.byref(ptr), C.byref(n)))
        raw = C.string_at(ptr, n.value) if n.value else b""
    finally:
        L.gsm_text_free(txt)
    terms = []
    i = 0
    while i < len(raw):
        (ln,) = struct.unpack_from("<I", raw, i)
        terms.append(raw[i + 4:i + 4 + ln].decode("utf-8"))
        i += 4 + ln
    return [tuple(terms[k:k + 3]) for k in range(0, len(terms), 3)]


def parse_ntriples_line(line: str, lineno: int | None = None):
    """qparser.parse_ntriples_line (qparser.py:80-104): the canonical triple
    of one statement, None for a blank or comment line."""
    text = ("\n" * ((lineno or 1) - 1)) + line.rstrip("\n") + "\n"
    try:
        got = parse_ntriples(text, threads=1)
    except Exception as e:  # keep the reference's "line N" only when a number was given
        from .errors import ParseError

        if isinstance(e, ParseError) and lineno is None:
            raise ParseError(str(e).split(": ", 1)[1] if ": " in str(e) else str(e)) from None
        raise
    return got[0] if got else None


def read_ntriples(lines):
    """qparser.read_ntriples (qparser.py:107-111) over an iterable of lines
    (e.g. an open text file): all statements parsed in one call."""
    text = "".join(line if line.endswith("\n") else line + "\n" for line in lines)
    yield from parse_ntriples(text)


def build(input_path: Path | str, out_dir: Path | str, device: int = 0,
          threads: int = 0) -> tuple[int, int, int]:
    """``gsmat build`` (cli._cmd_build): returns (triples, predicates, nodes),
    the numbers the reference prints."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)  # persist(): mkdir(parents=True, exist_ok=True)
    counts = (C.c_int64 * 3)()
    _lib.check(_lib.lib().gsm_build_store(str(input_path).encode(), str(out).encode(), int(device),
                                          int(threads), counts))
    return int(counts[0]), int(counts[1]), int(counts[2])
