"""ctypes binding of libtcudb.so (include/tcudb.h) — argument marshalling only.

Every step of the query runs in the library's sm_100a kernels; this module
only converts torch tensors to (pointer, dtype) columns, passes the current
CUDA stream, and wraps the result arrays (allocated through torch's caching
allocator via the ABI's allocator callbacks) as torch tensors. There is no
CPU fallback: a missing library or a non-sm_100 device raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtcudb.so")

TCUDB_OK, TCUDB_E_INVALID, TCUDB_E_UNSUPPORTED, TCUDB_E_PRECISION = 0, -1, -2, -3
TCUDB_E_OVERFLOW, TCUDB_E_NOMEM, TCUDB_E_CUDA, TCUDB_E_COMM = -4, -5, -6, -7
STATUS_NAMES = {0: "OK", -1: "E_INVALID", -2: "E_UNSUPPORTED", -3: "E_PRECISION", -4: "E_OVERFLOW",
                -5: "E_NOMEM", -6: "E_CUDA", -7: "E_COMM"}
I32, I64, F32, F64 = 0, 1, 2, 3
COUNT, SUM, AVG = 0, 1, 2
_AGG = {"count": COUNT, "sum": SUM, "avg": AVG}
FORCE_DENSE, FORCE_SPARSE, GATHER_NONE, UNORDERED, FORCE_WIDE, NO_FP4 = 1, 2, 4, 8, 16, 32
KEY_PARTITIONED, ROW_SHARDED = 64, 128

EXPORTS = sorted(["tcudb_create", "tcudb_join_agg", "tcudb_join_agg_host", "tcudb_chain_join_agg",
                  "tcudb_triangle_count", "tcudb_gemm",
                  "tcudb_minmax", "tcudb_partition", "tcudb_result_free", "tcudb_result_free_host",
                  "tcudb_last_error", "tcudb_launch_count", "tcudb_destroy", "tcudb_shard_agree",
                  "tcudb_shard_bounds", "tcudb_calibration"])
SHARD_DESC_LEN, SHARD_SAMPLES = 11, 1024


class TcudbError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Col(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("type", ctypes.c_int32)]


class TableS(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("key", Col), ("group", Col), ("value", Col)]


class Query(ctypes.Structure):
    _fields_ = [("agg", ctypes.c_int32), ("flags", ctypes.c_uint32)]


class Result(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("g", ctypes.c_void_p), ("h", ctypes.c_void_p), ("agg", ctypes.c_void_p),
                ("g_type", ctypes.c_int32), ("h_type", ctypes.c_int32), ("agg_type", ctypes.c_int32),
                ("on_host", ctypes.c_int32), ("base", ctypes.c_void_p)]


class Stats(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("elem", ctypes.c_int32), ("planes_a", ctypes.c_int32),
                ("planes_b", ctypes.c_int32), ("existence", ctypes.c_int32), ("kchunks", ctypes.c_int32),
                ("key_mode", ctypes.c_int32), ("n_launches", ctypes.c_int32),
                ("G", ctypes.c_int64), ("H", ctypes.c_int64), ("K", ctypes.c_int64), ("K_union", ctypes.c_int64),
                ("join_pairs", ctypes.c_int64), ("n_result", ctypes.c_int64),
                ("density_union", ctypes.c_double), ("gemm_ops", ctypes.c_double),
                ("ms_stats", ctypes.c_float), ("ms_encode", ctypes.c_float), ("ms_fill", ctypes.c_float),
                ("ms_gemm", ctypes.c_float), ("ms_sparse", ctypes.c_float), ("ms_compact", ctypes.c_float),
                ("ms_total", ctypes.c_float), ("spa_mode", ctypes.c_int32), ("spa_max_band", ctypes.c_int64),
                ("fused_compact", ctypes.c_int32), ("ms_kernel", ctypes.c_float), ("kernel_bytes", ctypes.c_double),
                ("ms_comm", ctypes.c_float), ("block_active", ctypes.c_double),
                ("spa_hubs", ctypes.c_int64)]

    def to_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)

_lib = None


def load(build_if_missing: bool = True):
    """Load libtcudb.so (building it with nvcc if absent/stale). Raises if it cannot."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing:
        from . import build as _build
        if _build.stale():
            _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtcudb.so not found at {LIB_PATH}; run paper_2112_07552_b200/build.py")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    lib.tcudb_create.argtypes = [ctypes.POINTER(P), ctypes.c_int, P, ALLOC_FN, FREE_FN, P]
    lib.tcudb_create.restype = ctypes.c_int
    lib.tcudb_join_agg.argtypes = [P, ctypes.POINTER(TableS), ctypes.POINTER(TableS), ctypes.POINTER(Query),
                                   ctypes.POINTER(Result), ctypes.POINTER(Stats), P]
    lib.tcudb_join_agg.restype = ctypes.c_int
    lib.tcudb_join_agg_host.argtypes = lib.tcudb_join_agg.argtypes
    lib.tcudb_join_agg_host.restype = ctypes.c_int
    lib.tcudb_chain_join_agg.argtypes = [P, ctypes.POINTER(TableS), ctypes.POINTER(TableS), ctypes.POINTER(TableS),
                                         ctypes.POINTER(Query), ctypes.POINTER(Result), ctypes.POINTER(Stats), P]
    lib.tcudb_chain_join_agg.restype = ctypes.c_int
    lib.tcudb_triangle_count.argtypes = [P, ctypes.c_int64, P, P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                                         ctypes.POINTER(Stats), P]
    lib.tcudb_triangle_count.restype = ctypes.c_int
    lib.tcudb_gemm.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                               ctypes.c_int64, P, ctypes.c_int64, P, ctypes.c_int64, P, ctypes.c_int64, P]
    lib.tcudb_gemm.restype = ctypes.c_int
    lib.tcudb_minmax.argtypes = [P, P, ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                 ctypes.POINTER(ctypes.c_int64), P]
    lib.tcudb_minmax.restype = ctypes.c_int
    lib.tcudb_partition.argtypes = [P, ctypes.POINTER(TableS), ctypes.POINTER(ctypes.c_int64), ctypes.c_int32,
                                    ctypes.POINTER(TableS), ctypes.POINTER(ctypes.c_int64), P]
    lib.tcudb_partition.restype = ctypes.c_int
    lib.tcudb_result_free.argtypes = [P, ctypes.POINTER(Result)]
    lib.tcudb_result_free_host.argtypes = [P, ctypes.POINTER(Result)]
    lib.tcudb_last_error.argtypes = [P]
    lib.tcudb_last_error.restype = ctypes.c_char_p
    lib.tcudb_launch_count.argtypes = [P]
    lib.tcudb_launch_count.restype = ctypes.c_int64
    lib.tcudb_destroy.argtypes = [P]
    lib.tcudb_calibration.argtypes = [P, ctypes.POINTER(ctypes.c_double)]
    lib.tcudb_calibration.restype = ctypes.c_int32
    I64P = ctypes.POINTER(ctypes.c_int64)
    lib.tcudb_shard_agree.argtypes = [I64P, ctypes.c_int32, I64P]
    lib.tcudb_shard_agree.restype = ctypes.c_int
    lib.tcudb_shard_bounds.argtypes = [I64P, ctypes.c_int32, I64P]
    lib.tcudb_shard_bounds.restype = ctypes.c_int
    _lib = lib
    return lib


def _dtype_code(t):
    import torch
    if t.dtype == torch.int32:
        return I32
    if t.dtype == torch.int64:
        return I64
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"unsupported column dtype {t.dtype}")


def _np_dtype_code(a):
    a = np.asarray(a)
    if a.dtype == np.int32:
        return I32
    if a.dtype == np.int64:
        return I64
    if a.dtype == np.float32:
        return F32
    raise TypeError(f"unsupported column dtype {a.dtype}")


_TYPESTR = {I32: "<i4", I64: "<i8", F32: "<f4", F64: "<f8"}
_TORCH_DT = None


class _Owner:
    """Owns one tcudb_result; frees it through the library when the last view dies."""

    def __init__(self, engine, res):
        self.engine, self.res = engine, res

    def __del__(self):
        try:
            if self.engine._ctx:
                self.engine._lib.tcudb_result_free(self.engine._ctx, ctypes.byref(self.res))
        except Exception:
            pass


class _HostOwner:
    """Owns one host-side tcudb_result (pinned blocks of the context cache)."""

    def __init__(self, engine, res):
        self.engine, self.res = engine, res

    def __del__(self):
        try:
            if self.engine._ctx:
                self.engine._lib.tcudb_result_free_host(self.engine._ctx, ctypes.byref(self.res))
        except Exception:
            pass


class _HostArray:
    def __init__(self, owner, ptr, n, dt):
        self._owner = owner
        self.__array_interface__ = {"shape": (int(n),), "typestr": dt.str, "data": (int(ptr), False),
                                    "version": 3}


class _DevArray:
    def __init__(self, owner, ptr, n, code):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": _TYPESTR[code],
                                         "data": (int(ptr or 0), False), "version": 3, "strides": None,
                                         "stream": None}


def shard_agree(descs):
    """tcudb_shard_agree (host only): descs = P rank descriptors (SHARD_DESC_LEN int64 each)
    -> (status, agreed descriptor)."""
    lib = load()
    d = np.ascontiguousarray(np.asarray(descs, dtype=np.int64).reshape(-1, SHARD_DESC_LEN))
    out = np.zeros(SHARD_DESC_LEN, dtype=np.int64)
    p64 = ctypes.POINTER(ctypes.c_int64)
    st = lib.tcudb_shard_agree(d.ctypes.data_as(p64), d.shape[0], out.ctypes.data_as(p64))
    return int(st), out


def shard_bounds(msgs):
    """tcudb_shard_bounds (host only): msgs = P sample messages (SHARD_SAMPLES + 2 int64
    each: n, S, S values) -> the P-1 range bounds."""
    lib = load()
    m = np.ascontiguousarray(np.asarray(msgs, dtype=np.int64).reshape(-1, SHARD_SAMPLES + 2))
    P = m.shape[0]
    out = np.zeros(max(P - 1, 1), dtype=np.int64)
    p64 = ctypes.POINTER(ctypes.c_int64)
    st = lib.tcudb_shard_bounds(m.ctypes.data_as(p64), P, out.ctypes.data_as(p64))
    if st != TCUDB_OK:
        raise TcudbError(st, "tcudb_shard_bounds")
    return out[:P - 1].tolist()


def shard_sample_msg(g):
    """The sample message one rank contributes (host mirror of collective.cu's strided
    sample: S = min(n, SHARD_SAMPLES) values at stride n // S)."""
    g = np.asarray(g, dtype=np.int64)
    n = len(g)
    S = min(n, SHARD_SAMPLES)
    m = np.zeros(SHARD_SAMPLES + 2, dtype=np.int64)
    m[0], m[1] = n, S
    if S:
        m[2:2 + S] = g[::n // S][:S]
    return m


def nccl_comm_ptr(group, device: int) -> int:
    """The ncclComm_t of a torch.distributed NCCL process group on `device` (created
    eagerly by one tiny collective: ProcessGroupNCCL builds communicators lazily)."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) != "nccl":
        raise ValueError("the collective engine needs an NCCL process group")
    t = torch.zeros(1, device=f"cuda:{device}")
    dist.all_reduce(t, group=group)
    torch.cuda.synchronize(device)
    pg = group if group is not None else dist.group.WORLD
    backend = pg._get_backend(torch.device("cuda", device))
    ptr = int(backend._comm_ptr())
    if not ptr:
        raise RuntimeError("ProcessGroupNCCL has no communicator for this device")
    return ptr


class Engine:
    """One tcudb context on one CUDA device (sm_100a)."""

    def __init__(self, device: int = 0, group=None, comm=None):
        """group: None (single GPU), or a torch.distributed NCCL process group (e.g.
        torch.distributed.group.WORLD) — then join_agg / join_agg_host are collective over
        its ranks (one GPU per rank; see tcudb_create in include/tcudb.h). comm: a raw
        communicator pointer instead of a group (an ncclComm_t, or a communicator of the
        library named by TCUDB_NCCL_LIB)."""
        import torch
        self._torch = torch
        self._lib = load()
        self.device = int(device)
        torch.cuda.init()
        self._alloc_cb = ALLOC_FN(self._alloc)
        self._free_cb = FREE_FN(self._free)
        if comm is not None:
            comm = ctypes.c_void_p(int(comm))
        elif group is not None:
            comm = ctypes.c_void_p(nccl_comm_ptr(group, self.device))
        ctx = ctypes.c_void_p()
        st = self._lib.tcudb_create(ctypes.byref(ctx), self.device, comm, self._alloc_cb, self._free_cb, None)
        if st != TCUDB_OK:
            raise TcudbError(st, "tcudb_create failed (needs an sm_100 GPU; with a group: a usable NCCL communicator)")
        self._ctx = ctx
        self.collective = comm is not None

    # allocator callbacks -> torch caching allocator (torch owns result memory)
    def _alloc(self, nbytes, stream, user):
        try:
            return self._torch.cuda.caching_allocator_alloc(int(nbytes), self.device, int(stream or 0))
        except Exception:
            return None

    def _free(self, ptr, stream, user):
        try:
            self._torch.cuda.caching_allocator_delete(int(ptr))
        except Exception:
            pass

    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.tcudb_destroy(self._ctx)
            self._ctx = None

    def last_error(self):
        return self._lib.tcudb_last_error(self._ctx).decode()

    @property
    def calibration(self) -> dict:
        """Selector constants measured at tcudb_create (tcudb_calibration)."""
        v = (ctypes.c_double * 8)()
        m = self._lib.tcudb_calibration(self._ctx, v)
        keys = ("R_i8", "R_bf16", "R_fp4", "BW", "R_sp", "T_sp0", "ms", "T_d0")
        return dict(zip(keys, list(v)), measured=bool(m), injected=m == 2)

    @property
    def launch_count(self) -> int:
        return int(self._lib.tcudb_launch_count(self._ctx))

    def _check(self, st):
        if st != TCUDB_OK:
            raise TcudbError(st, self.last_error())

    @staticmethod
    def _table_dev(T):
        k, g, v = T["k"], T.get("g"), T.get("v")
        for t in (k, g, v):
            if t is not None and (not t.is_cuda or not t.is_contiguous()):
                raise ValueError("columns must be contiguous CUDA tensors")
        ts = TableS()
        ts.n_rows = k.numel()
        ts.key = Col(k.data_ptr(), _dtype_code(k))
        # absent group column: this side is not grouped (Q3 / Q4 of PAPER.md §3.3)
        ts.group = Col(g.data_ptr(), _dtype_code(g)) if g is not None else Col(None, 0)
        ts.value = Col(v.data_ptr(), _dtype_code(v)) if v is not None else Col(None, 0)
        return ts

    @staticmethod
    def _table_host(T):
        k = np.ascontiguousarray(T["k"])
        g, v = T.get("g"), T.get("v")
        g = None if g is None else np.ascontiguousarray(g)
        v = None if v is None else np.ascontiguousarray(v)
        ts = TableS()
        ts.n_rows = len(k)
        ts.key = Col(k.ctypes.data, _np_dtype_code(k))
        ts.group = Col(g.ctypes.data, _np_dtype_code(g)) if g is not None else Col(None, 0)
        ts.value = Col(v.ctypes.data, _np_dtype_code(v)) if v is not None else Col(None, 0)
        return ts, (k, g, v)

    def _stream(self, stream):
        torch = self._torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    def join_agg(self, A, B, agg="count", flags=0, stream=None, with_stats=False):
        """SELECT A.g, B.h, agg FROM A JOIN B ON A.k = B.k GROUP BY A.g, B.h.

        A, B: dicts of contiguous CUDA tensors {"k", "g", "v" (optional)}.
        Returns {"g", "h", "agg"} CUDA tensors sorted by (g, h) (+ stats dict).
        """
        torch = self._torch
        ta, tb = self._table_dev(A), self._table_dev(B)
        q = Query(_AGG[agg], int(flags))
        res = Result()
        stats = Stats()
        # without stats the call returns while the result write still runs on the stream (tcudb.h)
        st = self._lib.tcudb_join_agg(self._ctx, ctypes.byref(ta), ctypes.byref(tb), ctypes.byref(q),
                                      ctypes.byref(res), ctypes.byref(stats) if with_stats else None,
                                      self._stream(stream))
        self._check(st)
        owner = _Owner(self, res)
        out = {}
        for key, ptr, code in (("g", res.g, res.g_type), ("h", res.h, res.h_type), ("agg", res.agg, res.agg_type)):
            if key != "agg" and (A if key == "g" else B).get("g") is None:
                continue  # ungrouped side: no output column
            if res.n == 0 or not ptr:
                dt = {I32: torch.int32, I64: torch.int64, F32: torch.float32, F64: torch.float64}[code]
                out[key] = torch.empty(0, dtype=dt, device=f"cuda:{self.device}")
            else:
                out[key] = torch.as_tensor(_DevArray(owner, ptr, res.n, code), device=f"cuda:{self.device}")
        return (out, stats.to_dict()) if with_stats else out

    def join_agg_host(self, A, B, agg="count", flags=0, stream=None, with_stats=False):
        """Same query on HOST (numpy) columns: H2D copies, the query, D2H of the
        result tuples into pinned host memory — all inside the C library."""
        ta, keep_a = self._table_host(A)
        tb, keep_b = self._table_host(B)
        q = Query(_AGG[agg], int(flags))
        res = Result()
        stats = Stats()
        st = self._lib.tcudb_join_agg_host(self._ctx, ctypes.byref(ta), ctypes.byref(tb), ctypes.byref(q),
                                           ctypes.byref(res), ctypes.byref(stats), self._stream(stream))
        self._check(st)
        # zero-copy numpy views of the pinned result blocks; the blocks return to the
        # context's pinned cache when the last view is garbage collected
        owner = _HostOwner(self, res)
        out = {}
        for key, ptr, code in (("g", res.g, res.g_type), ("h", res.h, res.h_type), ("agg", res.agg, res.agg_type)):
            if key != "agg" and (A if key == "g" else B).get("g") is None:
                continue  # ungrouped side: no output column
            dt = np.dtype(_TYPESTR[code])
            out[key] = np.zeros(0, dt) if res.n == 0 else np.asarray(_HostArray(owner, ptr, res.n, dt))
        return (out, stats.to_dict()) if with_stats else out

    def chain_join_agg(self, A, B, C, agg="count", flags=0, stream=None, with_stats=False):
        """SELECT A.g, C.h, agg FROM A, B, C WHERE A.k = B.k AND B.g = C.k GROUP BY A.g, C.h
        (B's "g" column is its second join attribute; agg: "count" or integer "sum")."""
        torch = self._torch
        ta, tb, tc = self._table_dev(A), self._table_dev(B), self._table_dev(C)
        q = Query(_AGG[agg], int(flags))
        res = Result()
        stats = Stats()
        st = self._lib.tcudb_chain_join_agg(self._ctx, ctypes.byref(ta), ctypes.byref(tb), ctypes.byref(tc),
                                            ctypes.byref(q), ctypes.byref(res), ctypes.byref(stats),
                                            self._stream(stream))
        self._check(st)
        owner = _Owner(self, res)
        out = {}
        for key, ptr, code in (("g", res.g, res.g_type), ("h", res.h, res.h_type), ("agg", res.agg, res.agg_type)):
            if res.n == 0 or not ptr:
                dt = {I32: torch.int32, I64: torch.int64, F32: torch.float32, F64: torch.float64}[code]
                out[key] = torch.empty(0, dtype=dt, device=f"cuda:{self.device}")
            else:
                out[key] = torch.as_tensor(_DevArray(owner, ptr, res.n, code), device=f"cuda:{self.device}")
        return (out, stats.to_dict()) if with_stats else out

    def triangle_count(self, src, dst, stream=None, with_stats=False):
        """Triangles of the simple undirected graph on an edge list (CUDA int32/int64 tensors)."""
        if src.dtype != dst.dtype or src.numel() != dst.numel():
            raise ValueError("src and dst must have equal dtype and length")
        out = ctypes.c_int64()
        stats = Stats()
        st = self._lib.tcudb_triangle_count(self._ctx, src.numel(), src.data_ptr(), dst.data_ptr(),
                                            _dtype_code(src), ctypes.byref(out), ctypes.byref(stats),
                                            self._stream(stream))
        self._check(st)
        return (int(out.value), stats.to_dict()) if with_stats else int(out.value)

    def minmax(self, col, stream=None):
        """(min, max) of a CUDA int32/int64 column (host ints)."""
        mn, mx = ctypes.c_int64(), ctypes.c_int64()
        self._check(self._lib.tcudb_minmax(self._ctx, col.data_ptr() if col.numel() else None, _dtype_code(col),
                                           col.numel(), ctypes.byref(mn), ctypes.byref(mx), self._stream(stream)))
        return int(mn.value), int(mx.value)

    def partition(self, T, bounds, stream=None):
        """Route a device table's rows into len(bounds)+1 group-key ranges.
        Returns (table grouped by destination, list of rows per destination)."""
        torch = self._torch
        P = len(bounds) + 1
        ts = self._table_dev(T)
        out = {k: torch.empty_like(v) for k, v in T.items() if v is not None}
        to = TableS()
        to.n_rows = T["k"].numel()
        to.key = Col(out["k"].data_ptr(), _dtype_code(out["k"]))
        to.group = Col(out["g"].data_ptr(), _dtype_code(out["g"]))
        to.value = Col(out["v"].data_ptr(), _dtype_code(out["v"])) if "v" in out else Col(None, 0)
        b = (ctypes.c_int64 * max(1, P - 1))(*[int(x) for x in bounds])
        counts = (ctypes.c_int64 * P)()
        self._check(self._lib.tcudb_partition(self._ctx, ctypes.byref(ts), b, P, ctypes.byref(to), counts,
                                              self._stream(stream)))
        return out, [int(c) for c in counts]

    def gemm(self, A, B, a_signed=True, b_signed=True, fp4=False, stream=None):
        """C = A @ B.T on the tcgen05 kernel. A: [M,K], B: [N,K] int8/uint8 (-> int32) or bf16 (-> fp32).
        fp4=True: A, B are uint8 [rows, K/2] of packed e2m1 pairs (kind::mxf4), C int32."""
        torch = self._torch
        M, K = A.shape
        N = B.shape[0]
        elem = 2 if fp4 else (1 if A.dtype == torch.bfloat16 else 0)
        lda, ldb = A.stride(0), B.stride(0)
        if fp4:
            K, lda, ldb = 2 * K, 2 * lda, 2 * ldb
        C = torch.empty((M, N), dtype=torch.float32 if elem == 1 else torch.int32, device=A.device)
        st = self._lib.tcudb_gemm(self._ctx, elem, int(a_signed), int(b_signed), M, N, K, A.data_ptr(), lda,
                                  B.data_ptr(), ldb, C.data_ptr(), C.stride(0), self._stream(stream))
        self._check(st)
        return C

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
