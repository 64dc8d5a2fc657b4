"""paper_1702_03484_b200 — Python binding of libmapsq.so (MapSQ's join path on B200, sm_100a).

Argument marshalling only: every step of the path runs in the CUDA kernels behind the C ABI
declared in include/mapsq.h (same function names, minus the ``mapsq_`` prefix).  PyTorch is
used for device memory of the inputs, for streams and for ``torch.distributed``.  There is no
CPU fallback: importing works without a GPU (for the host-only ``plan_join``), but every compute
call raises if the CUDA extension or a GPU is missing.

Tables are ``DeviceTable`` objects (SoA uint32 columns + one variable id per column).  Results
own library-allocated device memory and expose their columns as zero-copy torch tensors.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmapsq.so")

MAX_COLS = 16
MAX_PATTERNS = 16
TABLE_BOUNDS = 1
PATH_P64, PATH_KV, PATH_RESIDUAL, PATH_HASH = 0, 1, 2, 3
OPT_WIDE_KEY, WIDE_KEY_RESIDUAL, WIDE_KEY_KV, WIDE_KEY_HASH = 1, 0, 1, 2
OPT_SEMIJOIN, SEMIJOIN_OFF, SEMIJOIN_AUTO, SEMIJOIN_ON = 2, 0, 1, 2
OPT_SMALL_JOIN = 3
OPT_SKEW = 4
OPT_HOST_COMPRESS = 5
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_NO_SHARED", 3: "E_NOMEM", 4: "E_CUDA",
          5: "E_NCCL", 6: "E_UNSUPPORTED"}
DIST_ID_BYTES = 128


class MapsqError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"mapsq {STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class _Table(ctypes.Structure):
    _fields_ = [("nrows", ctypes.c_uint64), ("ncols", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("var", ctypes.c_int32 * MAX_COLS), ("lo", ctypes.c_uint32 * MAX_COLS),
                ("hi", ctypes.c_uint32 * MAX_COLS), ("col", ctypes.c_void_p * MAX_COLS),
                ("owner", ctypes.c_void_p)]


class _Triples(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("s", ctypes.c_void_p), ("p", ctypes.c_void_p),
                ("o", ctypes.c_void_p)]


class _Pattern(ctypes.Structure):
    _fields_ = [("var", ctypes.c_int32 * 3), ("id", ctypes.c_uint32 * 3)]


class JoinPlan(ctypes.Structure):
    _fields_ = [("n1", ctypes.c_uint64), ("n2", ctypes.c_uint64), ("nshared", ctypes.c_uint32),
                ("shared", ctypes.c_int32 * MAX_COLS), ("key_col1", ctypes.c_int32 * MAX_COLS),
                ("key_col2", ctypes.c_int32 * MAX_COLS), ("key_lo", ctypes.c_uint32 * MAX_COLS),
                ("key_hi", ctypes.c_uint32 * MAX_COLS), ("key_bits", ctypes.c_uint32 * MAX_COLS),
                ("key_shift", ctypes.c_uint32 * MAX_COLS), ("nrest1", ctypes.c_uint32),
                ("nrest2", ctypes.c_uint32), ("rest_col1", ctypes.c_int32 * MAX_COLS),
                ("rest_col2", ctypes.c_int32 * MAX_COLS), ("out_ncols", ctypes.c_uint32),
                ("out_var", ctypes.c_int32 * MAX_COLS), ("kb", ctypes.c_uint32),
                ("ib", ctypes.c_uint32), ("path", ctypes.c_uint32), ("passes", ctypes.c_uint32),
                ("disjoint", ctypes.c_uint32), ("packed_mask", ctypes.c_uint32)]


class _KStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_uint64),
                ("total_ms", ctypes.c_double), ("algo_bytes", ctypes.c_uint64)]


class _Stats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_uint64), ("join_in_rows", ctypes.c_uint64),
                ("join_out_rows", ctypes.c_uint64), ("scanned_triples", ctypes.c_uint64),
                ("joins", ctypes.c_uint64), ("scans", ctypes.c_uint64),
                ("last_kb", ctypes.c_uint64), ("last_ib", ctypes.c_uint64),
                ("last_passes", ctypes.c_uint64), ("last_path", ctypes.c_uint64),
                ("last_groups", ctypes.c_uint64), ("last_filtered", ctypes.c_uint64),
                ("filter_accesses", ctypes.c_uint64), ("exchanges", ctypes.c_uint64),
                ("exchange_rows", ctypes.c_uint64), ("exchange_bytes", ctypes.c_uint64),
                ("exchange_recv_rows", ctypes.c_uint64), ("exchange_recv_bytes", ctypes.c_uint64),
                ("skew_keys", ctypes.c_uint64),
                ("nkernels", ctypes.c_uint32), ("kernel", _KStat * 32)]


# mapsq_collectives (include/mapsq.h): host-buffer control-plane callbacks
_AG_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                          ctypes.c_size_t)
_AR_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32),
                          ctypes.c_size_t)
_BAR_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)


class _Collectives(ctypes.Structure):
    _fields_ = [("allgather", _AG_FN), ("allreduce_max_u32", _AR_FN), ("barrier", _BAR_FN),
                ("user", ctypes.c_void_p)]


_lib = None


def lib():
    """The loaded libmapsq.so; raises loudly if the CUDA extension was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"CUDA extension {_LIB_PATH} is missing: run `python build.py` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(_LIB_PATH)
        vp, u64, u32, i32, st = (ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32,
                                 ctypes.c_int32, ctypes.c_int)
        PT, PP = ctypes.POINTER(_Table), ctypes.POINTER(_Pattern)
        sigs = {
            "mapsq_create": (st, [ctypes.POINTER(vp), ctypes.c_int, vp]),
            "mapsq_destroy": (None, [vp]),
            "mapsq_last_error": (ctypes.c_char_p, [vp]),
            "mapsq_version": (ctypes.c_char_p, []),
            "mapsq_table_release": (None, [vp, PT, vp]),
            "mapsq_scan_patterns": (st, [vp, ctypes.POINTER(_Triples), PP, ctypes.c_int, PT, vp]),
            "mapsq_scan_pattern": (st, [vp, ctypes.POINTER(_Triples), PP, PT, vp]),
            "mapsq_join": (st, [vp, PT, PT, PT, vp]),
            "mapsq_plan_join": (st, [PT, PT, ctypes.POINTER(JoinPlan)]),
            "mapsq_plan_join_mode": (st, [PT, PT, ctypes.c_int, ctypes.POINTER(JoinPlan)]),
            "mapsq_query": (st, [vp, ctypes.POINTER(_Triples), PP, ctypes.c_int,
                                 ctypes.POINTER(i32), ctypes.c_int, PT, vp]),
            "mapsq_query_host": (st, [vp, u64, vp, vp, vp, PP, ctypes.c_int, ctypes.POINTER(i32),
                                      ctypes.c_int, ctypes.POINTER(u64), ctypes.POINTER(u32),
                                      ctypes.POINTER(i32), ctypes.POINTER(vp), vp]),
            "mapsq_index_build": (st, [vp, ctypes.POINTER(_Triples), ctypes.POINTER(vp), vp]),
            "mapsq_index_destroy": (None, [vp, vp]),
            "mapsq_index_triples": (st, [vp, ctypes.POINTER(_Triples), ctypes.POINTER(u32)]),
            "mapsq_index_range": (st, [vp, u32, ctypes.POINTER(u64), ctypes.POINTER(u64)]),
            "mapsq_scan_patterns_indexed": (st, [vp, vp, PP, ctypes.c_int, PT, vp]),
            "mapsq_query_indexed": (st, [vp, vp, PP, ctypes.c_int, ctypes.POINTER(i32),
                                         ctypes.c_int, PT, vp]),
            "mapsq_index_to_host": (st, [vp, vp, ctypes.POINTER(vp), vp]),
            "mapsq_host_index_destroy": (None, [vp]),
            "mapsq_query_host_indexed": (st, [vp, vp, PP, ctypes.c_int, ctypes.POINTER(i32),
                                              ctypes.c_int, ctypes.POINTER(u64),
                                              ctypes.POINTER(u32), ctypes.POINTER(i32),
                                              ctypes.POINTER(vp), ctypes.POINTER(u64), vp]),
            "mapsq_query_dist_host_indexed": (st, [vp, vp, PP, ctypes.c_int, ctypes.POINTER(i32),
                                                   ctypes.c_int, ctypes.POINTER(u64),
                                                   ctypes.POINTER(u32), ctypes.POINTER(i32),
                                                   ctypes.POINTER(vp), ctypes.POINTER(u64), vp]),
            "mapsq_map_words": (st, [vp, PT, PT, ctypes.POINTER(JoinPlan), vp, vp]),
            "mapsq_sort_words": (st, [vp, vp, u64, u32, u32, vp]),
            "mapsq_sort_pairs": (st, [vp, vp, vp, u64, u32, u32, vp]),
            "mapsq_reduce_groups": (st, [vp, vp, u64, u64, u32, vp, vp, vp, vp,
                                         ctypes.POINTER(u64), ctypes.POINTER(u64), vp]),
            "mapsq_partition": (st, [vp, PT, ctypes.POINTER(i32), ctypes.c_int, ctypes.c_int, PT,
                                     ctypes.POINTER(u64), vp]),
            "mapsq_table_bounds": (st, [vp, PT, vp]),
            "mapsq_exchange_layout": (st, [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.POINTER(u64), ctypes.POINTER(u64),
                                           ctypes.POINTER(u64), ctypes.POINTER(u64)]),
            "mapsq_dist_unique_id": (st, [ctypes.c_char_p]),
            "mapsq_dist_init": (st, [vp, ctypes.c_char_p, ctypes.c_int, ctypes.c_int]),
            "mapsq_dist_init_host": (st, [vp, ctypes.POINTER(_Collectives), ctypes.c_int,
                                          ctypes.c_int]),
            "mapsq_join_dist": (st, [vp, PT, PT, PT, vp]),
            "mapsq_query_dist": (st, [vp, ctypes.POINTER(_Triples), PP, ctypes.c_int,
                                      ctypes.POINTER(i32), ctypes.c_int, PT, vp]),
            "mapsq_query_dist_indexed": (st, [vp, vp, PP, ctypes.c_int, ctypes.POINTER(i32),
                                              ctypes.c_int, PT, vp]),
            "mapsq_partition_plan": (st, [vp, PT, ctypes.POINTER(i32), ctypes.c_int, ctypes.c_int,
                                          ctypes.POINTER(u64), ctypes.POINTER(vp), vp]),
            "mapsq_partition_scatter": (st, [vp, vp, ctypes.POINTER(u64), ctypes.POINTER(vp), vp]),
            "mapsq_partition_state_free": (None, [vp, vp]),
            "mapsq_ipc_alloc": (st, [vp, ctypes.c_size_t, ctypes.POINTER(vp)]),
            "mapsq_ipc_free": (st, [vp, vp]),
            "mapsq_ipc_export": (st, [vp, vp, ctypes.c_char_p]),
            "mapsq_ipc_open": (st, [vp, ctypes.c_char_p, ctypes.POINTER(vp)]),
            "mapsq_ipc_close": (st, [vp, vp]),
            "mapsq_set_profiling": (st, [vp, ctypes.c_int]),
            "mapsq_set_option": (st, [vp, ctypes.c_int, ctypes.c_int64]),
            "mapsq_stats_reset": (st, [vp]),
            "mapsq_get_stats": (st, [vp, ctypes.POINTER(_Stats)]),
        }
        for name, (res, args) in sigs.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def exported_symbols() -> list:
    """Names of the C ABI functions this binding expects (each must resolve in the .so)."""
    L = lib()
    return [n for n in dir(L) if n.startswith("mapsq_")]


def version() -> str:
    return lib().mapsq_version().decode()


# ------------------------------------------------------------------------------ helpers
def _stream(stream=None):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class _CAI:
    """Zero-copy view of one library-owned device column (keeps the owner alive)."""

    def __init__(self, ptr: int, n: int, owner):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<u4", "data": (ptr, False),
                                         "version": 3, "strides": None}
        self._owner = owner


class _Owner:
    """Holds a library-allocated table and releases it (stream ordered) when collected."""

    def __init__(self, ctx: "Context", t: _Table, stream=None):
        self.ctx, self.t, self.stream = ctx, t, stream

    def release(self):
        if self.t is not None and self.t.owner:
            lib().mapsq_table_release(self.ctx.handle, ctypes.byref(self.t),
                                      self.stream if self.stream is not None else _stream())
        self.t = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class DeviceTable:
    """Partial-match table: ``vars[c]`` is the variable bound by column ``columns[c]``."""

    def __init__(self, vars_, columns, nrows, c_table: _Table, owner=None):
        self.vars = list(vars_)
        # a library result's torch views are built on first use (a caller that only reads nrows,
        # or passes the table on to the next call, never pays for them)
        self._columns = list(columns) if not callable(columns) else None
        self._col_fn = columns if callable(columns) else None
        self.nrows = int(nrows)
        self._c = c_table
        self._owner = owner

    @property
    def columns(self):
        if self._columns is None:
            self._columns = self._col_fn()
        return self._columns

    @columns.setter
    def columns(self, cols):
        self._columns = list(cols)

    @property
    def ncols(self) -> int:
        return len(self.vars)

    @property
    def bounds(self):
        if not (self._c.flags & TABLE_BOUNDS):
            return None
        return [(int(self._c.lo[c]), int(self._c.hi[c])) for c in range(self.ncols)]

    def column(self, var: int):
        return self.columns[self.vars.index(var)]

    def to_numpy(self):
        """Row-major (nrows, ncols) uint32 host copy."""
        import numpy as np
        import torch
        if self.nrows == 0:
            return np.zeros((0, self.ncols), np.uint32)
        cols = [c.view(torch.int32).cpu().numpy().view(np.uint32) for c in self.columns]
        return np.ascontiguousarray(np.stack(cols, 1))

    def release(self):
        if self._owner is not None:
            self._owner.release()
        self.columns = []

    @staticmethod
    def from_torch(vars_, columns, bounds=None) -> "DeviceTable":
        """Borrow caller-owned uint32 device columns (torch.uint32 or int32 tensors)."""
        import torch
        if len(vars_) != len(columns) or not 0 < len(vars_) <= MAX_COLS:
            raise ValueError("one variable per column, 1..16 columns")
        n = int(columns[0].numel())
        t = _Table()
        t.nrows, t.ncols = n, len(vars_)
        for c, (v, col) in enumerate(zip(vars_, columns)):
            if col.numel() != n or not col.is_cuda or col.element_size() != 4:
                raise ValueError("columns must be equal-length 4-byte CUDA tensors")
            if not col.is_contiguous():
                raise ValueError("columns must be contiguous")
            t.var[c] = int(v)
            t.col[c] = col.data_ptr() if n else None
        if bounds is not None:
            t.flags = TABLE_BOUNDS
            for c, (lo, hi) in enumerate(bounds):
                t.lo[c], t.hi[c] = lo, hi
        return DeviceTable(vars_, columns, n, t, owner=None)


def _wrap(ctx: "Context", t: _Table, keep=None, stream=None) -> DeviceTable:
    owner = _Owner(ctx, t, stream)
    owner.keep = keep  # e.g. the Index whose memory a zero-copy view references
    n, w = int(t.nrows), int(t.ncols)
    ptrs = [t.col[c] for c in range(w)]

    def cols():
        import torch
        if n == 0:
            return [torch.empty(0, dtype=torch.uint32, device="cuda") for _ in range(w)]
        return [torch.as_tensor(_CAI(p, n, owner), device="cuda") for p in ptrs]
    return DeviceTable([int(t.var[c]) for c in range(w)], cols, n, t, owner)


def pattern_struct(pattern) -> _Pattern:
    """pattern = ((kind, x), (kind, x), (kind, x)): kind 'v' = variable id, 'c' = constant id."""
    p = _Pattern()
    for j, (kind, x) in enumerate(pattern):
        if kind == "v":
            p.var[j], p.id[j] = int(x), 0
        elif kind == "c":
            p.var[j], p.id[j] = -1, int(x)
        else:
            raise ValueError(f"pattern position kind must be 'v' or 'c', got {kind!r}")
    return p


def _triples(s, p, o) -> _Triples:
    n = int(s.numel())
    if p.numel() != n or o.numel() != n:
        raise ValueError("s, p, o must have equal length")
    for x in (s, p, o):
        if not (x.is_cuda and x.element_size() == 4 and x.is_contiguous()):
            raise ValueError("triples must be contiguous 4-byte CUDA tensors")
    return _Triples(n, s.data_ptr(), p.data_ptr(), o.data_ptr())


class Index:
    """Predicate-range index (mapsq_index_build): the triple table stably partitioned by
    predicate, owned by the library.  Pass it instead of (s, p, o) to scan_patterns / query."""

    def __init__(self, ctx: "Context", handle):
        self.ctx, self.handle = ctx, handle
        T, npreds = _Triples(), ctypes.c_uint32()
        ctx._check(lib().mapsq_index_triples(handle, ctypes.byref(T), ctypes.byref(npreds)))
        self.n, self.npreds, self._T = int(T.n), int(npreds.value), T

    def range(self, p: int):
        b, e = ctypes.c_uint64(), ctypes.c_uint64()
        self.ctx._check(lib().mapsq_index_range(self.handle, int(p), ctypes.byref(b),
                                                ctypes.byref(e)))
        return int(b.value), int(e.value)

    def triples(self):
        """(s, p, o) zero-copy torch views of the permuted table."""
        import torch
        if self.n == 0:
            return tuple(torch.empty(0, dtype=torch.uint32, device="cuda") for _ in range(3))
        return tuple(torch.as_tensor(_CAI(ptr, self.n, self), device="cuda")
                     for ptr in (self._T.s, self._T.p, self._T.o))

    def release(self):
        if self.handle:
            lib().mapsq_index_destroy(self.ctx.handle, self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class HostIndex:
    """Pinned host mirror of an Index (mapsq_index_to_host): pass it to Context.query_host to
    answer a query from host memory, copying only the predicate ranges the query touches."""

    def __init__(self, handle):
        self.handle = handle
        self.last_h2d_bytes = 0

    def release(self):
        if self.handle:
            lib().mapsq_host_index_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class PreparedQuery:
    """A query whose C arguments (patterns, projection, stream, store) are built once; each call
    is one mapsq_query_indexed / mapsq_query call (latency-bound small queries, C1)."""

    def __init__(self, ctx, triples, patterns, proj=None, stream=None):
        self.ctx, self.triples = ctx, triples
        self.k = len(patterns)
        self.pats = (_Pattern * self.k)(*[pattern_struct(p) for p in patterns])
        proj = list(proj or [])
        self.nproj = len(proj)
        self.pr = (ctypes.c_int32 * max(1, len(proj)))(*proj)
        self.stream = _stream(stream)
        if isinstance(triples, Index):
            self.fn, self.src = lib().mapsq_query_indexed, triples.handle
        else:
            self._T = _triples(*triples)
            self.fn, self.src = lib().mapsq_query, ctypes.byref(self._T)

    def __call__(self) -> DeviceTable:
        out = _Table()
        self.ctx._check(self.fn(self.ctx.handle, self.src, self.pats, self.k, self.pr, self.nproj,
                                ctypes.byref(out), self.stream))
        keep = self.triples if isinstance(self.triples, Index) else None
        return _wrap(self.ctx, out, keep=keep, stream=self.stream)


class Context:
    """One libmapsq context on one device (default allocator: cudaMallocAsync pool)."""

    def __init__(self, device: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("mapsq needs a CUDA device (no CPU fallback)")
        self.device = device
        h = ctypes.c_void_p()
        st = lib().mapsq_create(ctypes.byref(h), device, None)
        if st:
            raise MapsqError(st, "mapsq_create failed")
        self.handle = h

    def __del__(self):
        try:
            if self.handle:
                lib().mapsq_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def _check(self, st: int):
        if st:
            raise MapsqError(st, lib().mapsq_last_error(self.handle).decode())

    # ---- partial matching (row a1)
    def index_build(self, triples, stream=None) -> Index:
        """Build the predicate-range index of (s, p, o) (blocking; once per dataset)."""
        T = _triples(*triples)
        h = ctypes.c_void_p()
        self._check(lib().mapsq_index_build(self.handle, ctypes.byref(T), ctypes.byref(h),
                                            _stream(stream)))
        return Index(self, h)

    def scan_patterns(self, triples, patterns, stream=None) -> list:
        """``triples`` = (s, p, o) device tensors, or an Index (range scans / views)."""
        k = len(patterns)
        pats = (_Pattern * k)(*[pattern_struct(p) for p in patterns])
        outs = (_Table * k)()
        if isinstance(triples, Index):
            self._check(lib().mapsq_scan_patterns_indexed(self.handle, triples.handle, pats, k,
                                                          outs, _stream(stream)))
            return [_wrap(self, outs[j], keep=triples) for j in range(k)]
        T = _triples(*triples)
        self._check(lib().mapsq_scan_patterns(self.handle, ctypes.byref(T), pats, k, outs,
                                              _stream(stream)))
        return [_wrap(self, outs[j]) for j in range(k)]

    def scan_pattern(self, triples, pattern, stream=None) -> DeviceTable:
        T = _triples(*triples)
        p = pattern_struct(pattern)
        out = _Table()
        self._check(lib().mapsq_scan_pattern(self.handle, ctypes.byref(T), ctypes.byref(p),
                                             ctypes.byref(out), _stream(stream)))
        return _wrap(self, out)

    # ---- join (rows a2-a6)
    def join(self, tp1: DeviceTable, tp2: DeviceTable, stream=None) -> DeviceTable:
        out = _Table()
        self._check(lib().mapsq_join(self.handle, ctypes.byref(tp1._c), ctypes.byref(tp2._c),
                                     ctypes.byref(out), _stream(stream)))
        return _wrap(self, out)

    # ---- query (row a7)
    def prepare(self, triples, patterns, proj=None, stream=None) -> "PreparedQuery":
        """``query`` with its arguments marshalled once (a prepared statement): calling the
        result runs mapsq_query[_indexed] again on the same store, patterns and stream."""
        return PreparedQuery(self, triples, patterns, proj, stream)

    def query(self, triples, patterns, proj=None, stream=None) -> DeviceTable:
        """``triples`` = (s, p, o) device tensors, or an Index."""
        k = len(patterns)
        pats = (_Pattern * k)(*[pattern_struct(p) for p in patterns])
        proj = list(proj or [])
        pr = (ctypes.c_int32 * max(1, len(proj)))(*proj)
        out = _Table()
        if isinstance(triples, Index):
            self._check(lib().mapsq_query_indexed(self.handle, triples.handle, pats, k, pr,
                                                  len(proj), ctypes.byref(out), _stream(stream)))
            return _wrap(self, out, keep=triples)
        T = _triples(*triples)
        self._check(lib().mapsq_query(self.handle, ctypes.byref(T), pats, k, pr, len(proj),
                                      ctypes.byref(out), _stream(stream)))
        return _wrap(self, out)

    def index_to_host(self, index: Index, stream=None) -> HostIndex:
        """Mirror a device Index into pinned host memory (blocking, once per dataset)."""
        h = ctypes.c_void_p()
        self._check(lib().mapsq_index_to_host(self.handle, index.handle, ctypes.byref(h),
                                              _stream(stream)))
        return HostIndex(h)

    def query_dist_host(self, shard: "HostIndex", patterns, proj=None, stream=None, copy=False):
        """mapsq_query_dist_host_indexed: this rank's result shard, end to end over its
        host-resident store (collective).  Returns (vars, rows) like query_host."""
        return self.query_host(shard, patterns, proj=proj, stream=stream, copy=copy, _dist=True)

    def query_host(self, s, p=None, o=None, patterns=None, proj=None, stream=None, copy=False,
                   _dist=False):
        """End to end over host memory: ``s, p, o`` (numpy, ideally pinned) triples, or a
        HostIndex as the first argument (then only the ranges the query touches are copied;
        ``HostIndex.last_h2d_bytes`` records how many bytes).  Returns (vars, rows) where rows is an
        (nrows, ncols) view of the context's pinned result arena (valid until the next query_host
        on this context) or, with copy=True, an independent array."""
        import numpy as np
        if isinstance(s, HostIndex) and patterns is None:
            patterns, p = p, None
        k = len(patterns)
        pats = (_Pattern * k)(*[pattern_struct(q) for q in patterns])
        proj = list(proj or [])
        pr = (ctypes.c_int32 * max(1, len(proj)))(*proj)
        nrows, ncols = ctypes.c_uint64(), ctypes.c_uint32()
        ovar = (ctypes.c_int32 * MAX_COLS)()
        ocol = (ctypes.c_void_p * MAX_COLS)()
        ptr = lambda a: a.ctypes.data if hasattr(a, "ctypes") else a.data_ptr()  # noqa: E731
        if isinstance(s, HostIndex):
            h2d = ctypes.c_uint64()
            fn = lib().mapsq_query_dist_host_indexed if _dist else lib().mapsq_query_host_indexed
            self._check(fn(self.handle, s.handle, pats, k, pr, len(proj), ctypes.byref(nrows),
                           ctypes.byref(ncols), ovar, ocol, ctypes.byref(h2d), _stream(stream)))
            s.last_h2d_bytes = int(h2d.value)
        else:
            self._check(lib().mapsq_query_host(self.handle, len(s), ptr(s), ptr(p), ptr(o), pats, k,
                                               pr, len(proj), ctypes.byref(nrows),
                                               ctypes.byref(ncols), ovar, ocol, _stream(stream)))
        m, w = int(nrows.value), int(ncols.value)
        vars_ = [int(ovar[c]) for c in range(w)]
        if m == 0 or w == 0:
            return vars_, np.zeros((m, w), np.uint32)
        # columns are consecutive in the arena: one (w, m) block -> transpose view (m, w)
        buf = (ctypes.c_uint32 * (m * w)).from_address(ocol[0])
        cols = np.frombuffer(buf, np.uint32, m * w).reshape(w, m)
        rows = cols.T
        return vars_, (np.ascontiguousarray(rows) if copy else rows)

    # ---- phase entry points (rows a3-a5)
    def map_words(self, tp1, tp2, plan: JoinPlan, words, stream=None):
        self._check(lib().mapsq_map_words(self.handle, ctypes.byref(tp1._c), ctypes.byref(tp2._c),
                                          ctypes.byref(plan), words.data_ptr(), _stream(stream)))

    def sort_words(self, words, bit_lo: int, bit_hi: int, stream=None):
        self._check(lib().mapsq_sort_words(self.handle, words.data_ptr(), words.numel(), bit_lo,
                                           bit_hi, _stream(stream)))

    def sort_pairs(self, keys, vals, bit_lo: int, bit_hi: int, stream=None):
        self._check(lib().mapsq_sort_pairs(self.handle, keys.data_ptr(), vals.data_ptr(),
                                           keys.numel(), bit_lo, bit_hi, _stream(stream)))

    def reduce_groups(self, words, n1: int, n2: int, ib: int, stream=None):
        import torch
        cap = max(1, min(n1, n2))
        dev = words.device
        gs, gp, ge = (torch.empty(cap, dtype=torch.int32, device=dev) for _ in range(3))
        go = torch.empty(cap, dtype=torch.int64, device=dev)
        ng, tot = ctypes.c_uint64(), ctypes.c_uint64()
        self._check(lib().mapsq_reduce_groups(self.handle, words.data_ptr(), n1, n2, ib,
                                              gs.data_ptr(), gp.data_ptr(), ge.data_ptr(),
                                              go.data_ptr(), ctypes.byref(ng), ctypes.byref(tot),
                                              _stream(stream)))
        g = int(ng.value)
        return gs[:g], gp[:g], ge[:g], go[:g], int(tot.value)

    def partition(self, table: DeviceTable, key_vars, nparts: int, stream=None):
        kv = (ctypes.c_int32 * len(key_vars))(*key_vars)
        counts = (ctypes.c_uint64 * nparts)()
        out = _Table()
        self._check(lib().mapsq_partition(self.handle, ctypes.byref(table._c), kv, len(key_vars),
                                          nparts, ctypes.byref(out), counts, _stream(stream)))
        return _wrap(self, out), [int(c) for c in counts]

    def partition_plan(self, table: DeviceTable, key_vars, nparts: int, stream=None):
        """K8 plan: per-destination row counts + an opaque state for partition_scatter."""
        kv = (ctypes.c_int32 * len(key_vars))(*key_vars)
        counts = (ctypes.c_uint64 * nparts)()
        st = ctypes.c_void_p()
        self._check(lib().mapsq_partition_plan(self.handle, ctypes.byref(table._c), kv, len(key_vars),
                                               nparts, counts, ctypes.byref(st), _stream(stream)))
        return st, [int(c) for c in counts]

    def partition_scatter(self, state, dest_row, dest_cols, stream=None):
        """The fused partition + exchange kernel: rows go straight to dest_cols (device or peer
        pointers, destination-major: dest_cols[d * ncols + c]) at dest_row[d] onwards."""
        rows = (ctypes.c_uint64 * len(dest_row))(*dest_row)
        cols = (ctypes.c_void_p * len(dest_cols))(*dest_cols)
        try:
            self._check(lib().mapsq_partition_scatter(self.handle, state, rows, cols, _stream(stream)))
        finally:
            lib().mapsq_partition_state_free(self.handle, state)

    def ipc_alloc(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        self._check(lib().mapsq_ipc_alloc(self.handle, nbytes, ctypes.byref(p)))
        return int(p.value)

    def ipc_free(self, ptr: int):
        self._check(lib().mapsq_ipc_free(self.handle, ctypes.c_void_p(ptr)))

    def ipc_export(self, ptr: int) -> bytes:
        buf = ctypes.create_string_buffer(64)
        self._check(lib().mapsq_ipc_export(self.handle, ctypes.c_void_p(ptr), buf))
        return buf.raw

    def ipc_open(self, handle: bytes) -> int:
        p = ctypes.c_void_p()
        self._check(lib().mapsq_ipc_open(self.handle, handle, ctypes.byref(p)))
        return int(p.value)

    def ipc_close(self, ptr: int):
        self._check(lib().mapsq_ipc_close(self.handle, ctypes.c_void_p(ptr)))

    # ---- distributed join and query (rows b, e): collective calls, one context per rank
    def dist_init(self, group=None):
        """Join this context to an NCCL communicator over the ranks of ``group`` (a
        torch.distributed group): the group's first rank creates the unique id, torch.distributed
        broadcasts it, every rank calls mapsq_dist_init.  Collective; once per context."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [None]
        if rank == 0:
            buf = ctypes.create_string_buffer(DIST_ID_BYTES)
            st = lib().mapsq_dist_unique_id(buf)
            if st:
                raise MapsqError(st, "mapsq_dist_unique_id failed (NCCL not loadable?)")
            obj[0] = buf.raw
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(obj, src=src, group=group)
        self._check(lib().mapsq_dist_init(self.handle, obj[0], rank, world))
        self.dist_rank, self.dist_world = rank, world

    def dist_init_host(self, group=None):
        """Join the ranks of ``group`` with the control plane carried by torch.distributed itself
        (e.g. the gloo backend) instead of NCCL: mapsq_dist_init_host with host-buffer callbacks
        (argument marshalling only; the exchange, arenas and joins are the library's).  This is
        how several rank processes can share one GPU.  Collective; once per context."""
        import numpy as np
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def allgather(_user, send, recv, nbytes):
            try:
                src = torch.from_numpy(np.ctypeslib.as_array(
                    ctypes.cast(send, ctypes.POINTER(ctypes.c_uint8)), shape=(nbytes,)).copy())
                out = torch.empty(world * nbytes, dtype=torch.uint8)
                dist.all_gather_into_tensor(out, src, group=group)
                ctypes.memmove(recv, out.numpy().ctypes.data, world * nbytes)
                return 0
            except Exception:  # noqa: BLE001 (reported to the library as a failed collective)
                return 1

        def allreduce_max(_user, buf, n):
            try:
                arr = np.ctypeslib.as_array(buf, shape=(n,))
                t = torch.from_numpy(arr.astype(np.int64))
                dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
                arr[:] = t.numpy().astype(np.uint32)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        def barrier(_user):
            try:
                dist.barrier(group=group)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        self._coll = _Collectives(_AG_FN(allgather), _AR_FN(allreduce_max), _BAR_FN(barrier), None)
        self._check(lib().mapsq_dist_init_host(self.handle, ctypes.byref(self._coll), rank, world))
        self.dist_rank, self.dist_world = rank, world

    def join_dist(self, tp1: DeviceTable, tp2: DeviceTable, stream=None) -> DeviceTable:
        """This rank's shard of tp1 ⋈ tp2 (inputs: this rank's rows, any distribution)."""
        out = _Table()
        self._check(lib().mapsq_join_dist(self.handle, ctypes.byref(tp1._c), ctypes.byref(tp2._c),
                                          ctypes.byref(out), _stream(stream)))
        return _wrap(self, out)

    def query_dist(self, shard, patterns, proj=None, stream=None) -> DeviceTable:
        """This rank's shard of the query result over this rank's triples ((s, p, o) device
        tensors or an Index of them)."""
        k = len(patterns)
        pats = (_Pattern * k)(*[pattern_struct(p) for p in patterns])
        proj = list(proj or [])
        pr = (ctypes.c_int32 * max(1, len(proj)))(*proj)
        out = _Table()
        if isinstance(shard, Index):
            self._check(lib().mapsq_query_dist_indexed(self.handle, shard.handle, pats, k, pr,
                                                       len(proj), ctypes.byref(out),
                                                       _stream(stream)))
            return _wrap(self, out, keep=shard)
        T = _triples(*shard)
        self._check(lib().mapsq_query_dist(self.handle, ctypes.byref(T), pats, k, pr, len(proj),
                                           ctypes.byref(out), _stream(stream)))
        return _wrap(self, out)

    def table_bounds(self, table: DeviceTable, stream=None):
        self._check(lib().mapsq_table_bounds(self.handle, ctypes.byref(table._c), _stream(stream)))
        return table.bounds

    def set_option(self, option: int, value: int):
        self._check(lib().mapsq_set_option(self.handle, option, value))

    # ---- statistics
    def set_profiling(self, on: bool):
        self._check(lib().mapsq_set_profiling(self.handle, int(bool(on))))

    def stats_reset(self):
        self._check(lib().mapsq_stats_reset(self.handle))

    def stats(self) -> dict:
        st = _Stats()
        self._check(lib().mapsq_get_stats(self.handle, ctypes.byref(st)))
        d = {f: int(getattr(st, f)) for f, _ in _Stats._fields_ if f not in ("kernel", "nkernels")}
        d["kernels"] = {st.kernel[i].name.decode(): dict(launches=int(st.kernel[i].launches),
                                                         ms=float(st.kernel[i].total_ms),
                                                         bytes=int(st.kernel[i].algo_bytes))
                        for i in range(st.nkernels)}
        return d


def device_columns(ptr: int, nrows: int, ncols: int, stride: int, owner=None):
    """Zero-copy uint32 torch views of `ncols` columns of `nrows` at ptr + c * stride * 4."""
    import torch
    if nrows == 0:
        return [torch.empty(0, dtype=torch.uint32, device="cuda") for _ in range(ncols)]
    return [torch.as_tensor(_CAI(ptr + c * stride * 4, nrows, owner), device="cuda")
            for c in range(ncols)]


def exchange_layout(count_matrix, rank: int, ncols: int):
    """mapsq_exchange_layout (host only): (dest_row, recv, need_bytes) per destination rank."""
    world = len(count_matrix)
    flat = (ctypes.c_uint64 * (world * world))(*[int(x) for row in count_matrix for x in row])
    dr, rc, nd = ((ctypes.c_uint64 * world)() for _ in range(3))
    st = lib().mapsq_exchange_layout(world, rank, ncols, flat, dr, rc, nd)
    if st:
        raise MapsqError(st, "mapsq_exchange_layout: bad arguments")
    return list(dr), list(rc), list(nd)


def plan_join(vars1, bounds1, n1, vars2, bounds2, n2, wide_mode=None) -> JoinPlan:
    """Host-only join spec (row a2) from two schemas with column bounds; no GPU needed.
    wide_mode: None = the library default, else WIDE_KEY_RESIDUAL / _KV / _HASH."""
    t1, t2 = _Table(), _Table()
    for t, vs, bs, n in ((t1, vars1, bounds1, n1), (t2, vars2, bounds2, n2)):
        t.nrows, t.ncols, t.flags = n, len(vs), TABLE_BOUNDS
        for c, (v, (lo, hi)) in enumerate(zip(vs, bs)):
            t.var[c], t.lo[c], t.hi[c] = v, lo, hi
            t.col[c] = 16  # never dereferenced by the host-only planner
    plan = JoinPlan()
    if wide_mode is None:
        st = lib().mapsq_plan_join(ctypes.byref(t1), ctypes.byref(t2), ctypes.byref(plan))
    else:
        st = lib().mapsq_plan_join_mode(ctypes.byref(t1), ctypes.byref(t2), int(wide_mode),
                                        ctypes.byref(plan))
    if st:
        raise MapsqError(st, "plan_join")
    return plan
