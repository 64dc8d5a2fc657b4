"""CPU oracle for the MapSQ join path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product (``paper_1702_03484_b200``)
never imports it, and the two share no code.  See oracle.h for what each function computes and
which PAPER.md passage it follows; DESIGN.md §2 lists the readings of ambiguous passages.

Tables are ``Table(vars, rows)`` with ``rows`` a row-major ``(nrows, ncols)`` uint32 array.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
MAX_COLS = 16
OK, E_INVALID, E_NO_SHARED, E_NOMEM = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


class _CTable(ctypes.Structure):
    _fields_ = [("nrows", ctypes.c_uint64), ("ncols", ctypes.c_uint32),
                ("var", ctypes.c_int32 * MAX_COLS), ("rows", ctypes.POINTER(ctypes.c_uint32))]


@dataclass
class Table:
    vars: list
    rows: np.ndarray  # (nrows, ncols) uint32

    @property
    def nrows(self) -> int:
        return int(self.rows.shape[0])

    def canonical(self) -> np.ndarray:
        """Rows sorted lexicographically (the canonical form parity is judged on)."""
        return canonical_rows(self.rows)

    def column(self, var: int) -> np.ndarray:
        return self.rows[:, self.vars.index(var)]

    def reorder(self, vars_: list) -> "Table":
        idx = [self.vars.index(v) for v in vars_]
        return Table(list(vars_), np.ascontiguousarray(self.rows[:, idx]))


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            import sys
            sys.path.insert(0, os.path.dirname(_HERE))
            import build  # noqa: E402
            build.build_oracle()
        L = ctypes.CDLL(path)
        P32, PT = ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(_CTable)
        PI32 = ctypes.POINTER(ctypes.c_int32)
        L.oracle_scan.argtypes = [ctypes.c_uint64, P32, P32, P32, PI32, P32, PT]
        L.oracle_join_nested.argtypes = [PT, PT, PT]
        L.oracle_join_sortmerge.argtypes = [PT, PT, PT]
        L.oracle_query.argtypes = [ctypes.c_uint64, P32, P32, P32, PI32, P32, ctypes.c_int, PI32,
                                   ctypes.c_int, PT]
        L.oracle_canonical_sort.argtypes = [PT]
        L.oracle_canonical_sort.restype = None
        L.oracle_free.argtypes = [PT]
        L.oracle_free.restype = None
        PU64 = ctypes.POINTER(ctypes.c_uint64)
        L.oracle_fingerprint.argtypes = [PT, PU64]
        L.oracle_fingerprint.restype = None
        L.oracle_fingerprint_cols.argtypes = [ctypes.c_uint64, ctypes.c_uint32,
                                              ctypes.POINTER(P32), PU64]
        L.oracle_fingerprint_cols.restype = None
        for f in (L.oracle_scan, L.oracle_join_nested, L.oracle_join_sortmerge, L.oracle_query):
            f.restype = ctypes.c_int
        _LIB = L
    return _LIB


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


def _p32(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _to_c(t: Table, keep: list) -> _CTable:
    rows = _u32(t.rows).reshape(t.nrows, len(t.vars))
    keep.append(rows)
    c = _CTable()
    c.nrows, c.ncols = t.nrows, len(t.vars)
    for i, v in enumerate(t.vars):
        c.var[i] = v
    c.rows = _p32(rows)
    return c


def _from_c(c: _CTable) -> Table:
    n, w = int(c.nrows), int(c.ncols)
    if n * w:
        rows = np.ctypeslib.as_array(c.rows, shape=(n * w,)).copy().reshape(n, w)
    else:
        rows = np.zeros((n, w), np.uint32)
    vars_ = [int(c.var[i]) for i in range(w)]
    _lib().oracle_free(ctypes.byref(c))
    return Table(vars_, rows)


def pattern_arrays(pattern) -> tuple:
    """pattern = ((kind, x), (kind, x), (kind, x)) with kind 'v' (variable id) or 'c' (const)."""
    var = (ctypes.c_int32 * 3)()
    ids = (ctypes.c_uint32 * 3)()
    for j, (kind, x) in enumerate(pattern):
        if kind == "v":
            var[j], ids[j] = int(x), 0
        else:
            var[j], ids[j] = -1, int(x)
    return var, ids


def scan(s, p, o, pattern) -> Table:
    s, p, o = _u32(s), _u32(p), _u32(o)
    var, ids = pattern_arrays(pattern)
    out = _CTable()
    rc = _lib().oracle_scan(len(s), _p32(s), _p32(p), _p32(o), var, ids, ctypes.byref(out))
    if rc:
        raise OracleError(rc, "scan")
    return _from_c(out)


def join(a: Table, b: Table, tier: str = "sortmerge") -> Table:
    keep: list = []
    ca, cb = _to_c(a, keep), _to_c(b, keep)
    out = _CTable()
    fn = _lib().oracle_join_nested if tier == "nested" else _lib().oracle_join_sortmerge
    rc = fn(ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(out))
    if rc:
        raise OracleError(rc, f"join[{tier}]")
    return _from_c(out)


def query(s, p, o, patterns, proj=None) -> Table:
    s, p, o = _u32(s), _u32(p), _u32(o)
    k = len(patterns)
    pv = (ctypes.c_int32 * (3 * k))()
    pi = (ctypes.c_uint32 * (3 * k))()
    for i, pat in enumerate(patterns):
        v, d = pattern_arrays(pat)
        for j in range(3):
            pv[3 * i + j], pi[3 * i + j] = v[j], d[j]
    proj = list(proj or [])
    pr = (ctypes.c_int32 * max(1, len(proj)))(*proj)
    out = _CTable()
    rc = _lib().oracle_query(len(s), _p32(s), _p32(p), _p32(o), pv, pi, k, pr, len(proj),
                             ctypes.byref(out))
    if rc:
        raise OracleError(rc, "query")
    return _from_c(out)


def canonical(t: Table) -> Table:
    """Rows sorted lexicographically by the oracle (sorts a private copy in place)."""
    rows = _u32(t.rows).reshape(t.nrows, len(t.vars)).copy()
    c = _CTable()
    c.nrows, c.ncols = t.nrows, len(t.vars)
    c.rows = _p32(rows)
    _lib().oracle_canonical_sort(ctypes.byref(c))
    return Table(list(t.vars), rows)


class Fingerprint:
    """Accumulating multiset fingerprint (count, sum mod 2^64, xor) of per-row splitmix64 hashes
    (definition in oracle.h).  Feed it row-major tables or SoA column chunks
    in any order; equal multisets of rows give equal fingerprints."""

    def __init__(self):
        self.acc = (ctypes.c_uint64 * 3)(0, 0, 0)

    def add_table(self, t: Table) -> "Fingerprint":
        keep: list = []
        c = _to_c(t, keep)
        _lib().oracle_fingerprint(ctypes.byref(c), self.acc)
        return self

    def add_cols(self, cols) -> "Fingerprint":
        cols = [_u32(c) for c in cols]
        n = len(cols[0]) if cols else 0
        assert all(len(c) == n for c in cols)
        arr = (ctypes.POINTER(ctypes.c_uint32) * max(1, len(cols)))(*[_p32(c) for c in cols])
        _lib().oracle_fingerprint_cols(n, len(cols), arr, self.acc)
        return self

    @property
    def value(self) -> tuple:
        return int(self.acc[0]), int(self.acc[1]), int(self.acc[2])


def fingerprint(t: Table) -> tuple:
    return Fingerprint().add_table(t).value


def canonical_rows(rows: np.ndarray) -> np.ndarray:
    """Lexicographic row sort with numpy (used for device results copied to the host)."""
    rows = np.asarray(rows)
    if rows.shape[0] < 2 or rows.shape[1] == 0:
        return rows.copy()
    order = np.lexsort(rows.T[::-1])
    return rows[order]
