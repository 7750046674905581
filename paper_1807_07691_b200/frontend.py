"""Query front end of the drop-in: BGP parsing, constant binding, planning.

These are host-side and OUT of the accelerated path;
they are restated here only so the package runs stand-alone where the
reference is not installed (e.g. the GPU box).  They accept the reference's
query grammar and produce the same encoded patterns and the same plan order:

  parse_query     qparser.py:231-297  PREFIX* SELECT [DISTINCT] (?v+|*) WHERE {(s p o .)+}
  bind_constants  qparser.py:334-353  unknown predicate/constant -> id 0 + empty flag
  make_plan       planner.py:138-166  per connected component: ascending estimate,
                                      greedy connected choice; components by their
                                      cheapest pattern (planner.py:58-135)

tests/test_frontend.py checks equality with the reference's own functions on
the reference's randomized query campaign and on every LUBM query.
:func:`paper_1807_07691_b200.executor.execute` accepts plans from either.
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field

from .errors import ParseError, UnsupportedFeatureError

# ---------------------------------------------------------------------------
# terms
# ---------------------------------------------------------------------------
_IRI_CHARS = r'[^<>"{}|^`\\\x00-\x20]*'
_LIT_BODY = r'"(?:[^"\\\n]|\\.)*"'
_LANG = r"@[A-Za-z]+(?:-[A-Za-z0-9]+)*"
_LITERAL_RE = re.compile(rf"({_LIT_BODY})(?:\^\^<({_IRI_CHARS})>|({_LANG}))?")

_SCANNER = re.compile(
    "|".join(
        (
            rf"(?P<iri><{_IRI_CHARS}>)",
            rf"(?P<literal>{_LIT_BODY}(?:\^\^<{_IRI_CHARS}>|{_LANG})?)",
            r"(?P<var>[?$][A-Za-z_][A-Za-z0-9_]*)",
            r"(?P<punct>[{}.*;,])",
            r"(?P<pname>[A-Za-z_][A-Za-z0-9_.-]*:[A-Za-z0-9_.-]*|_:[A-Za-z0-9_.-]+|:[A-Za-z0-9_.-]*)",
            r"(?P<word>[A-Za-z]+)",
            r"(?P<comment>#[^\n]*)",
            r"(?P<ws>\s+)",
            r"(?P<bad>.)",
        )
    ),
    re.DOTALL,
)

_SIMPLE_ESC = {'"': '"', "\\": "\\", "n": "\n", "r": "\r", "t": "\t", "b": "\b", "f": "\f", "'": "'"}


def _unescape(body: str, line: int | None) -> str:
    """Literal escapes as qparser._unescape_literal (qparser.py:34-58)."""
    if "\\" not in body:
        return body
    parts: list[str] = []
    i = 0
    while i < len(body):
        ch = body[i]
        if ch != "\\":
            parts.append(ch)
            i += 1
            continue
        nxt = body[i + 1]
        if nxt in _SIMPLE_ESC:
            parts.append(_SIMPLE_ESC[nxt])
            i += 2
        elif nxt in "uU":
            width = 4 if nxt == "u" else 8
            parts.append(chr(int(body[i + 2 : i + 2 + width], 16)))
            i += 2 + width
        else:
            raise ParseError(f"bad literal escape \\{nxt}", line)
    return "".join(parts)


def format_term(term: str) -> str:
    """Canonical term -> surface syntax (qparser.py:71-78)."""
    if term.startswith('"'):
        cut = term.rfind('"')
        lex = (
            term[1:cut]
            .replace("\\", "\\\\")
            .replace('"', '\\"')
            .replace("\n", "\\n")
            .replace("\r", "\\r")
            .replace("\t", "\\t")
        )
        return f'"{lex}"{term[cut + 1:]}'
    if term.startswith("_:"):
        return term
    return f"<{term}>"


def is_var(term: str) -> bool:
    return term.startswith("?")


# ---------------------------------------------------------------------------
# query graph
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class TriplePattern:
    s: str
    p: str
    o: str
    ordinal: int

    def variables(self) -> list[str]:
        return [t for t in (self.s, self.o) if is_var(t)]

    def text(self) -> str:
        show = lambda t: t if is_var(t) else format_term(t)  # noqa: E731
        return f"{show(self.s)} {show(self.p)} {show(self.o)}"


@dataclass
class QueryGraph:
    patterns: list[TriplePattern]
    projection: list[str]
    select_all: bool = False
    distinct: bool = False
    variables: set[str] = field(default_factory=set)

    def __post_init__(self) -> None:
        if not self.variables:
            self.variables = {v for p in self.patterns for v in p.variables()}
        if self.select_all:
            order: list[str] = []
            for p in self.patterns:
                for v in p.variables():
                    if v not in order:
                        order.append(v)
            self.projection = order


class _Tokens:
    def __init__(self, text: str):
        self.items: list[tuple[str, str, int]] = []
        line = 1
        for m in _SCANNER.finditer(text):
            kind, value = m.lastgroup, m.group()
            if kind == "bad":
                raise ParseError(f"unexpected character {value!r}", line)
            if kind not in ("ws", "comment"):
                self.items.append((kind, value, line))
            line += value.count("\n")
        self.i = 0

    def peek(self):
        return self.items[self.i] if self.i < len(self.items) else None

    def take(self, keyword: str | None = None):
        tok = self.peek()
        if tok is None:
            raise ParseError("unexpected end of query")
        if keyword is not None and tok[1].upper() != keyword:
            raise ParseError(f"expected {keyword!r}, found {tok[1]!r}", tok[2])
        self.i += 1
        return tok

    def at(self, value: str) -> bool:
        tok = self.peek()
        return tok is not None and tok[1].upper() == value


def _term(toks: _Tokens, prefixes: dict[str, str]) -> str:
    kind, value, line = toks.take()
    if kind == "var":
        return "?" + value[1:]
    if kind == "iri":
        return value[1:-1]
    if kind == "literal":
        m = _LITERAL_RE.fullmatch(value)
        assert m is not None
        body, dtype, lang = m.groups()
        term = '"' + _unescape(body[1:-1], line) + '"'
        if dtype is not None:
            term += f"^^<{dtype}>"
        elif lang is not None:
            term += lang
        return term
    if kind == "pname":
        if value.startswith("_:"):
            return value
        prefix, _, local = value.partition(":")
        if prefix not in prefixes:
            raise ParseError(f"unknown prefix {prefix!r}:", line)
        return prefixes[prefix] + local
    raise ParseError(f"expected a term, found {value!r}", line)


def parse_query(text: str) -> QueryGraph:
    """``PREFIX* SELECT [DISTINCT] (?v+ | *) WHERE { (s p o .)+ }``."""
    toks = _Tokens(text)
    prefixes: dict[str, str] = {}
    while toks.at("PREFIX"):
        toks.take()
        kind, name, line = toks.take()
        if kind != "pname" or not name.endswith(":"):
            raise ParseError(f"expected a prefix declaration, found {name!r}", line)
        kind, iri, line = toks.take()
        if kind != "iri":
            raise ParseError(f"expected an IRI after PREFIX, found {iri!r}", line)
        prefixes[name[:-1]] = iri[1:-1]
    toks.take("SELECT")
    distinct = False
    if toks.at("DISTINCT"):
        toks.take()
        distinct = True
    projection: list[str] = []
    select_all = False
    if toks.peek() is not None and toks.peek()[1] == "*":
        toks.take()
        select_all = True
    else:
        while toks.peek() is not None and toks.peek()[0] == "var":
            projection.append("?" + toks.take()[1][1:])
        if not projection:
            tok = toks.peek()
            raise ParseError("SELECT clause names no variables", tok[2] if tok else None)
    toks.take("WHERE")
    toks.take("{")
    patterns: list[TriplePattern] = []
    while True:
        tok = toks.peek()
        if tok is None:
            raise ParseError("unterminated WHERE block")
        if tok[1] == "}":
            toks.take()
            break
        s = _term(toks, prefixes)
        pline = toks.peek()[2] if toks.peek() else 0
        p = _term(toks, prefixes)
        if is_var(p):
            raise UnsupportedFeatureError("variable predicates are not supported", pline)
        o = _term(toks, prefixes)
        patterns.append(TriplePattern(s, p, o, ordinal=len(patterns) + 1))
        if toks.peek() is not None and toks.peek()[1] == ".":
            toks.take()
    if toks.peek() is not None:
        raise ParseError(f"trailing tokens after query: {toks.peek()[1]!r}", toks.peek()[2])
    if not patterns:
        raise ParseError("WHERE block contains no triple patterns")
    graph = QueryGraph(patterns, projection, select_all=select_all, distinct=distinct)
    missing = [v for v in graph.projection if v not in graph.variables]
    if missing:
        raise ParseError(f"projected variables not bound by any pattern: {', '.join(missing)}")
    return graph


# ---------------------------------------------------------------------------
# constant binding
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class EncodedPattern:
    s: int | str
    p: int
    o: int | str
    ordinal: int
    source: TriplePattern
    empty: bool = False

    def variables(self) -> list[str]:
        return [t for t in (self.s, self.o) if isinstance(t, str)]

    def nodes(self) -> list[int | str]:
        return [self.s, self.o]


@dataclass
class EncodedQuery:
    patterns: list[EncodedPattern]
    projection: list[str]
    distinct: bool
    variables: set[str]


def bind_constants(graph: QueryGraph, dictionary) -> EncodedQuery:
    out: list[EncodedPattern] = []
    for tp in graph.patterns:
        pid = dictionary.lookup_predicate(tp.p)
        empty = pid is None
        ends: list[int | str] = []
        for t in (tp.s, tp.o):
            if is_var(t):
                ends.append(t)
                continue
            nid = dictionary.lookup_node(t)
            if nid is None:
                empty = True
            ends.append(0 if nid is None else nid)
        out.append(EncodedPattern(ends[0], 0 if pid is None else pid, ends[1], tp.ordinal, tp, empty))
    return EncodedQuery(out, list(graph.projection), graph.distinct, set(graph.variables))


# ---------------------------------------------------------------------------
# planning
# ---------------------------------------------------------------------------
_SAT = (1 << 63) - 1


@dataclass
class PlanStep:
    pattern: EncodedPattern
    estimate: int
    join_vars: list[str]


@dataclass
class Plan:
    steps: list[PlanStep]
    warnings: list[str] = field(default_factory=list)

    @property
    def estimates(self) -> list[int]:
        return [s.estimate for s in self.steps]


def estimate_cardinality(pat, stats) -> int:
    """planner.estimate_cardinality (planner.py:58-70)."""
    if pat.empty or pat.p not in stats:
        return 0
    card, ds, do = stats[pat.p]
    est = card
    s_const, o_const = isinstance(pat.s, int), isinstance(pat.o, int)
    if s_const and ds > 0:
        est = -(-est // ds)
    if o_const and do > 0:
        est = -(-est // do)
    return max(est, 1) if (s_const and o_const) else est


def _connected_groups(patterns) -> list[list]:
    """Union-find over shared endpoints, groups ordered by first member."""
    root = list(range(len(patterns)))

    def find(i: int) -> int:
        while root[i] != i:
            root[i] = root[root[i]]
            i = root[i]
        return i

    owner: dict[object, int] = {}
    for i, pat in enumerate(patterns):
        for node in pat.nodes():
            if node in owner:
                root[find(i)] = find(owner[node])
            else:
                owner[node] = i
    groups: dict[int, list] = {}
    for i, pat in enumerate(patterns):
        groups.setdefault(find(i), []).append(pat)
    return list(groups.values())


def make_plan(query, stats) -> Plan:
    if not query.patterns:
        raise ValueError("cannot plan an empty query")
    warnings: list[str] = []
    ordered_groups = []
    for group in _connected_groups(query.patterns):
        ranked = sorted(((estimate_cardinality(p, stats), p) for p in group),
                        key=lambda e: (e[0], e[1].ordinal))
        chain = [ranked.pop(0)]
        touched = set(chain[0][1].nodes())
        while ranked:
            pick = next((i for i, (_, p) in enumerate(ranked) if any(n in touched for n in p.nodes())),
                        None)
            if pick is None:
                pick = 0
                warnings.append("no connected pattern available; Cartesian product forced at "
                                f"pattern {ranked[0][1].ordinal}")
            chosen = ranked.pop(pick)
            touched.update(chosen[1].nodes())
            chain.append(chosen)
        ordered_groups.append(chain)
    ordered_groups.sort(key=lambda c: (c[0][0], c[0][1].ordinal))
    if len(ordered_groups) > 1:
        warnings.append(f"query graph has {len(ordered_groups)} components; "
                        "cross products between components are unavoidable")
    steps: list[PlanStep] = []
    bound: set[str] = set()
    for chain in ordered_groups:
        for est, pat in chain:
            steps.append(PlanStep(pat, est, [v for v in pat.variables() if v in bound]))
            bound.update(pat.variables())
    return Plan(steps, warnings)
