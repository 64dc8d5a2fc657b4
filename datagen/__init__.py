"""Seeded synthetic inputs (LUBM-shaped triples, Zipf / uniform (key, value) tables).

Input infrastructure shared by the oracle tests and the GPU path.  It contains none of the join
method's arithmetic; see datagen.h for the contract and DESIGN.md §3 for the recipe.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

LUBM_PRED = dict(type=0, name=1, emailAddress=2, telephone=3, subOrganizationOf=4, worksFor=5,
                 headOf=6, memberOf=7, undergraduateDegreeFrom=8, mastersDegreeFrom=9,
                 doctoralDegreeFrom=10, researchInterest=11, teacherOf=12, takesCourse=13,
                 advisor=14, teachingAssistantOf=15, publicationAuthor=16)
LUBM_CLASS = dict(University=32, Department=33, ResearchGroup=34, FullProfessor=35,
                  AssociateProfessor=36, AssistantProfessor=37, Lecturer=38,
                  UndergraduateStudent=39, GraduateStudent=40, Course=41, GraduateCourse=42,
                  Publication=43)

_STAT_FIELDS = (["n_triples"] + [f"pred_{i}" for i in range(32)]
                + ["n_dept", "n_faculty", "n_ug", "n_grad", "c1_rs", "c2_j1", "c2_j2",
                   "c3_j1", "c3_j2", "c3_j3", "c5_j1", "c5_j2"])


class _Stats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_uint64) for f in _STAT_FIELDS]


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libdatagen.so")
        if not os.path.exists(path):
            import sys
            sys.path.insert(0, os.path.dirname(_HERE))
            import build  # noqa: E402  (repo-root build helper)
            build.build_datagen()
        L = ctypes.CDLL(path)
        u64, u32, p32 = ctypes.c_uint64, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)
        L.lubm_pool_size.restype = u32
        L.lubm_pool_size.argtypes = [u32]
        L.lubm_univ_base.restype = u64
        L.lubm_univ_base.argtypes = [u64, u32, u32]
        L.lubm_id_end.restype = u64
        L.lubm_id_end.argtypes = [u64, u32, u32]
        L.lubm_count.restype = u64
        L.lubm_count.argtypes = [u64, u32, u32, u32, ctypes.POINTER(_Stats)]
        L.lubm_generate.restype = u64
        L.lubm_generate.argtypes = [u64, u32, u32, u32, p32, p32, p32, ctypes.POINTER(_Stats)]
        L.zipf_table.restype = None
        L.zipf_table.argtypes = [u64, ctypes.c_int, ctypes.c_double, u32, u64, u64, p32, p32]
        L.zipf_rank.restype = u64
        L.zipf_rank.argtypes = [u64, ctypes.c_int, ctypes.c_double, u32, u64]
        L.uniform_table.restype = None
        L.uniform_table.argtypes = [u64, u64, u32, u32, p32, p32]
        L.datagen_num_threads.restype = ctypes.c_int
        _LIB = L
    return _LIB


def _p32(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _stats_dict(st: _Stats) -> dict:
    d = {f: int(getattr(st, f)) for f in _STAT_FIELDS if not f.startswith("pred_")}
    d["pred_count"] = [int(getattr(st, f"pred_{i}")) for i in range(32)]
    return d


def lubm_count(n_univ: int, u_lo: int = 0, u_hi: int | None = None, seed: int = 42) -> dict:
    u_hi = n_univ if u_hi is None else u_hi
    st = _Stats()
    _lib().lubm_count(seed, n_univ, u_lo, u_hi, ctypes.byref(st))
    return _stats_dict(st)


def lubm(n_univ: int, u_lo: int = 0, u_hi: int | None = None, seed: int = 42, out=None):
    """Triples of universities [u_lo, u_hi) of LUBM(n_univ) as SoA uint32 (s, p, o) + stats.

    ``out`` may supply preallocated (s, p, o) uint32 arrays (e.g. pinned host memory)."""
    u_hi = n_univ if u_hi is None else u_hi
    L = _lib()
    st = _Stats()
    n = L.lubm_count(seed, n_univ, u_lo, u_hi, None)
    if out is None:
        s, p, o = (np.empty(n, np.uint32) for _ in range(3))
    else:
        s, p, o = out
        assert all(a.dtype == np.uint32 and a.size >= n and a.flags.c_contiguous for a in out)
    m = L.lubm_generate(seed, n_univ, u_lo, u_hi, _p32(s), _p32(p), _p32(o), ctypes.byref(st))
    assert m == n
    return s[:n], p[:n], o[:n], _stats_dict(st)


def lubm_id_end(n_univ: int, u_hi: int | None = None, seed: int = 42) -> int:
    return int(_lib().lubm_id_end(seed, n_univ, n_univ if u_hi is None else u_hi))


def lubm_univ_base(n_univ: int, u: int, seed: int = 42) -> int:
    """First dictionary ID of university u's block (entities + literals of u follow)."""
    return int(_lib().lubm_univ_base(seed, n_univ, u))


def lubm_pool_size(n_univ: int) -> int:
    return int(_lib().lubm_pool_size(n_univ))


def zipf(n: int, side: int, seed: int = 1702, s: float = 1.1, kbits: int = 29, i_lo: int = 0,
         out=None):
    """Rows [i_lo, i_lo+n) of one side of the C4 Zipf(s) (key, value) table."""
    if out is None:
        key, val = np.empty(n, np.uint32), np.empty(n, np.uint32)
    else:
        key, val = out
    _lib().zipf_table(seed, side, s, kbits, i_lo, i_lo + n, _p32(key), _p32(val))
    return key[:n], val[:n]


def zipf_rank(i: int, side: int = 0, seed: int = 1702, s: float = 1.1, kbits: int = 29) -> int:
    return int(_lib().zipf_rank(seed, side, s, kbits, i))


def uniform(n: int, key_domain: int, val_domain: int = 1 << 30, seed: int = 7):
    key, val = np.empty(n, np.uint32), np.empty(n, np.uint32)
    _lib().uniform_table(seed, n, key_domain, val_domain, _p32(key), _p32(val))
    return key, val


def num_threads() -> int:
    return int(_lib().datagen_num_threads())
