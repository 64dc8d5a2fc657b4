"""SPARQL front-end, greedy planner and dictionary (the step after the hot path).

The paper states queries as SPARQL basic graph patterns — "SELECT ?person WHERE {?person hasJob
?job. ?job workAt "Hospital".}" — and answers them in two steps, partial matching
and the MapReduce-based join.  This module turns query text into the library's
pattern descriptors, orders the joins, runs them on the GPU through the C ABI and decodes the
result.  Host-side orchestration only: every scan, join and projection runs in libmapsq's kernels.

* Grammar (a subset of SPARQL): ``SELECT (?v+ | *) WHERE { p (. p)* [.] }`` with terms
  ``?var``, ``<iri>``, bare identifiers (taken as IRIs, the paper's informal syntax) and quoted
  literals.  Errors carry the 1-based line and column.
* Dictionary: dense uint32 IDs in first-seen order; ``load_ntriples`` keeps the triple
  SET (duplicates dropped).
* Planner: scan every pattern (one fused pass), then a left-deep order that starts
  from the smallest partial-match table and repeatedly appends the smallest table sharing a
  variable with what is joined so far (ties: textual order).  A disconnected pattern is an error
  (cross products are out of scope, reading R9).
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np


class SparqlError(ValueError):
    pass


@dataclass(frozen=True)
class Term:
    """An RDF term: kind 'iri' (``<x>`` or a bare identifier) or 'lit' (a quoted literal)."""
    kind: str
    text: str

    def __str__(self):
        if self.kind == "lit":
            return '"' + self.text.replace("\\", "\\\\").replace('"', '\\"') + '"'
        return (
            self.text if re.fullmatch(r"[A-Za-z_][\w:.\-]*", self.text) else f"<{self.text}>")


@dataclass(frozen=True)
class Var:
    name: str

    def __str__(self):
        return "?" + self.name


@dataclass
class Query:
    projection: Optional[List[str]]          # None = SELECT *
    patterns: List[Tuple[object, object, object]]

    def variables(self) -> List[str]:
        """Variables in first-appearance order."""
        out: List[str] = []
        for pat in self.patterns:
            for x in pat:
                if isinstance(x, Var) and x.name not in out:
                    out.append(x.name)
        return out

    def __str__(self):  # debug printer; parse(str(q)) == q
        proj = "*" if self.projection is None else " ".join("?" + v for v in self.projection)
        body = " . ".join(" ".join(str(x) for x in pat) for pat in self.patterns)
        return f"SELECT {proj} WHERE {{ {body} . }}"


_TOKEN = re.compile(r'''\s*(?:(?P<var>\?[A-Za-z_][\w]*)|(?P<iri><[^<>\s]*>)|(?P<lit>"(?:[^"\\]|\\.)*")|
                        (?P<punct>[{}.*])|(?P<word>[A-Za-z_][\w:.\-]*[\w]|[A-Za-z_]))''', re.X)


def _tokens(text: str):
    pos = 0
    n = len(text)
    while pos < n:
        while pos < n and text[pos].isspace():
            pos += 1
        if pos == n:
            break
        m = _TOKEN.match(text, pos)
        if not m or m.end() == pos:
            raise SparqlError(_where(text, pos) + f": unexpected character {text[pos]!r}")
        kind = m.lastgroup
        start = m.start(kind)
        yield kind, m.group(kind), start
        pos = m.end()


def _where(text: str, pos: int) -> str:
    line = text.count("\n", 0, pos) + 1
    col = pos - (text.rfind("\n", 0, pos) + 1) + 1
    return f"line {line}, column {col}"


def parse_query(text: str) -> Query:
    """Parse the supported SPARQL subset."""
    toks = list(_tokens(text))
    i = 0

    def peek():
        return toks[i] if i < len(toks) else ("eof", "", len(text))

    def expect(kind, value=None):
        nonlocal i
        k, v, p = peek()
        if k != kind or (value is not None and v.upper() != value):
            want = value or kind
            raise SparqlError(_where(text, p) + f": expected {want}, found {v or 'end of input'!r}")
        i += 1
        return v

    expect("word", "SELECT")
    proj: Optional[List[str]] = []
    if peek()[0] == "punct" and peek()[1] == "*":
        i += 1
        proj = None
    else:
        while peek()[0] == "var":
            proj.append(peek()[1][1:])
            i += 1
        if not proj:
            raise SparqlError(_where(text, peek()[2]) + ": expected a variable list or *")
    expect("word", "WHERE")
    expect("punct", "{")
    pats = []
    while True:
        k, v, p = peek()
        if k == "punct" and v == "}":
            break
        pat = []
        for _ in range(3):
            k, v, p = peek()
            if k == "var":
                pat.append(Var(v[1:]))
            elif k == "iri":
                pat.append(Term("iri", v[1:-1]))
            elif k == "lit":
                pat.append(Term("lit", bytes(v[1:-1], "utf-8").decode("unicode_escape")))
            elif k == "word" and v.upper() not in ("SELECT", "WHERE"):
                pat.append(Term("iri", v))
            else:
                raise SparqlError(_where(text, p) + f": expected a term, found {v or 'end of input'!r}")
            i += 1
        pats.append(tuple(pat))
        k, v, p = peek()
        if k == "punct" and v == ".":
            i += 1
        elif not (k == "punct" and v == "}"):
            raise SparqlError(_where(text, p) + f": expected '.' or '}}', found {v or 'end of input'!r}")
    expect("punct", "}")
    if i != len(toks):
        raise SparqlError(_where(text, toks[i][2]) + ": trailing input")
    if not pats:
        raise SparqlError(_where(text, peek()[2]) + ": empty basic graph pattern")
    q = Query(proj, pats)
    if proj is not None:
        vs = set(q.variables())
        for v in proj:
            if v not in vs:
                raise SparqlError(f"projected variable ?{v} appears in no pattern")
    return q


@dataclass
class Dictionary:
    """Dense uint32 term IDs in first-seen order."""
    terms: List[Term] = field(default_factory=list)
    ids: Dict[Term, int] = field(default_factory=dict)

    def intern(self, t: Term) -> int:
        i = self.ids.get(t)
        if i is None:
            i = len(self.terms)
            self.ids[t] = i
            self.terms.append(t)
        return i

    def lookup(self, t: Term) -> Optional[int]:
        return self.ids.get(t)

    def resolve(self, i: int) -> Term:
        return self.terms[i]

    def decode(self, ids: np.ndarray) -> np.ndarray:
        arr = np.empty(len(self.terms), dtype=object)
        arr[:] = self.terms
        return arr[np.asarray(ids, dtype=np.int64)]


_NT = re.compile(r'''\s*(<[^<>]*>|"(?:[^"\\]|\\.)*"|[A-Za-z_][\w:.\-]*)\s+(<[^<>]*>|[A-Za-z_][\w:.\-]*)\s+
                     (<[^<>]*>|"(?:[^"\\]|\\.)*"|[A-Za-z_][\w:.\-]*)\s*\.\s*$''', re.X)


def _term(tok: str) -> Term:
    if tok.startswith("<"):
        return Term("iri", tok[1:-1])
    if tok.startswith('"'):
        return Term("lit", bytes(tok[1:-1], "utf-8").decode("unicode_escape"))
    return Term("iri", tok)


def load_ntriples(lines, dictionary: Optional[Dictionary] = None):
    """N-Triples-like lines (``s p o .``; bare identifiers allowed) -> (dictionary, s, p, o) with
    uint32 columns; the store is a set: duplicate triples are kept once, first
    occurrence order."""
    d = dictionary or Dictionary()
    seen = set()
    rows = []
    for k, line in enumerate(lines, 1):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        m = _NT.match(line)
        if not m:
            raise SparqlError(f"line {k}: not an N-Triples statement")
        tr = tuple(d.intern(_term(x)) for x in m.groups())
        if tr not in seen:
            seen.add(tr)
            rows.append(tr)
    a = np.asarray(rows, dtype=np.uint32).reshape(-1, 3)
    return d, a[:, 0].copy(), a[:, 1].copy(), a[:, 2].copy()


ABSENT = 0xFFFFFFFF  # the ID of a constant missing from the dictionary: it matches nothing


def encode(query: Query, dictionary: Dictionary):
    """Pattern descriptors for the C ABI (variables numbered in first-appearance order) and the
    projection as variable ids."""
    names = query.variables()
    vid = {v: k for k, v in enumerate(names)}
    pats = []
    for pat in query.patterns:
        enc = []
        for x in pat:
            if isinstance(x, Var):
                enc.append(("v", vid[x.name]))
            else:
                i = dictionary.lookup(x)
                enc.append(("c", ABSENT if i is None else i))
        pats.append(tuple(enc))
    proj = names if query.projection is None else query.projection
    return pats, [vid[v] for v in proj], names


def greedy_order(sizes: Sequence[int], pattern_vars: Sequence[Sequence[int]]) -> List[int]:
    """start from the smallest table, then repeatedly the smallest table sharing a
    variable with the joined ones (ties: textual order)."""
    left = list(range(len(sizes)))
    first = min(left, key=lambda k: (sizes[k], k))
    order, have = [first], set(pattern_vars[first])
    left.remove(first)
    while left:
        conn = [k for k in left if have & set(pattern_vars[k])]
        if not conn:
            raise SparqlError("the basic graph pattern is not connected (cross products are "
                              "out of scope)")
        nxt = min(conn, key=lambda k: (sizes[k], k))
        order.append(nxt)
        have |= set(pattern_vars[nxt])
        left.remove(nxt)
    return order


@dataclass
class ResultSet:
    schema: List[str]
    rows: np.ndarray  # (n, len(schema)) object array of Terms


def execute(ctx, store, dictionary: Dictionary, text: str, plan: str = "greedy",
            stream=None) -> ResultSet:
    """Parse, encode, match every pattern (one fused scan or index views), join in the chosen
    order on the GPU, project, decode.  ``store`` = (s, p, o) device tensors or an Index.
    ``plan`` = "greedy" or "textual" (reading R8, what mapsq_query does)."""
    q = parse_query(text)
    pats, proj, names = encode(q, dictionary)
    if plan == "textual":
        rs = ctx.query(store, pats, proj, stream=stream)
        ids = rs.to_numpy()
    else:
        tabs = ctx.scan_patterns(store, pats, stream=stream)
        pv = [t.vars for t in tabs]
        order = greedy_order([t.nrows for t in tabs], pv)
        acc = tabs[order[0]]
        for k in order[1:]:
            acc = ctx.join(acc, tabs[k], stream=stream)
        cols = [acc.columns[acc.vars.index(v)] for v in proj]
        ids = (np.stack([c.view(__import__("torch").int32).cpu().numpy().view(np.uint32)
                         for c in cols], 1) if acc.nrows else np.zeros((0, len(proj)), np.uint32))
    schema = [names[v] for v in proj]
    rows = dictionary.decode(ids.reshape(-1)).reshape(ids.shape) if ids.size else \
        np.empty((0, len(schema)), dtype=object)
    return ResultSet(schema, rows)
