"""CPU oracle for the TCUDB join + group-by hot path — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. The product path
(paper_2112_07552_b200) never imports it and shares no code with it.

Two independent implementations of the same definition:
  * join_agg(A, B, agg)      — liboracle.so: C++17/OpenMP hash join + hash
                               aggregation (oracle.cpp; Fig. 4
                               P:580-598, §3.1, §3.3).
  * nested_loop(A, B, agg)   — pure-Python nested loop for tiny inputs
                               (SPEC.md nested_loop_oracle).
  * triangles(src, dst)      — simple-graph triangle count (§3.2
                               chain exception P:751-756; reading R15).

Result format: dict with numpy arrays "g", "h", "cnt" and, for SUM,
"sum" (int64 or float64) plus "abs" (float64, float SUM only); rows sorted by
(g, h); groups are exactly those with COUNT > 0 (reading R3).
Every function here is pinned in tests/test_oracle.py; none is "parity
unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


class OracleOverflow(ArithmeticError):
    """An integer SUM does not fit int64 (the GPU must report E_OVERFLOW)."""


class _Result(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64),
                ("g", ctypes.POINTER(ctypes.c_int64)),
                ("h", ctypes.POINTER(ctypes.c_int64)),
                ("cnt", ctypes.POINTER(ctypes.c_int64)),
                ("isum", ctypes.POINTER(ctypes.c_int64)),
                ("fsum", ctypes.POINTER(ctypes.c_double)),
                ("fabs_sum", ctypes.POINTER(ctypes.c_double))]


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++ -O2 -fopenmp); no CUDA involved."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared",
                                   _SRC, "-o", tmp])
            os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        lib.oracle_join_agg.argtypes = [ctypes.c_int64, P, P, P, ctypes.c_int,
                                        ctypes.c_int64, P, P, P, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Result)]
        lib.oracle_join_agg.restype = ctypes.c_int
        lib.oracle_free.argtypes = [ctypes.POINTER(_Result)]
        lib.oracle_triangles.argtypes = [ctypes.c_int64, P, P, ctypes.c_int]
        lib.oracle_triangles.restype = ctypes.c_int64
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _vcol(v):
    if v is None:
        return None, 0
    v = np.asarray(v)
    if v.dtype.kind in "iu":
        return np.ascontiguousarray(v, dtype=np.int64), 1
    if v.dtype.kind == "f":
        if v.dtype != np.float32:
            raise TypeError("float values must be float32 (the ABI's float column type)")
        return np.ascontiguousarray(v), 2
    raise TypeError(f"unsupported value dtype {v.dtype}")


def _ungrouped(A, B, out):
    """Drop the output column of an ungrouped side (its group was the constant 0)."""
    if A.get("g") is None:
        out.pop("g")
    if B.get("g") is None:
        out.pop("h")
    return out


def _group_col(T, n):
    g = T.get("g")
    # an absent group column = the side is not grouped: every tuple in one group
    # (GROUP BY B.h only is Q3; no GROUP BY at all is Q4)
    return np.zeros(n, np.int64) if g is None else np.ascontiguousarray(g, dtype=np.int64)


def join_agg(A, B, agg="count", threads: int = 0):
    """SELECT A.g, B.h, agg FROM A JOIN B ON A.k = B.k GROUP BY A.g, B.h.

    agg: "count" -> COUNT(*); "sum" -> SUM(A.v * B.w) (an absent value column
    is the constant 1); "avg" -> AVG(A.v * B.w) = SUM / COUNT as
    "avg" (float64: the int64 SUM or the fp64 SUM divided by the count).
    A table whose "g" is None is not grouped: its output column is omitted.
    Raises OracleOverflow if an integer SUM leaves int64.
    """
    if agg == "avg":
        out = join_agg(A, B, "sum", threads)
        out["avg"] = out["sum"].astype(np.float64) / out["cnt"].astype(np.float64)
        return out
    lib = _load()
    ak = np.ascontiguousarray(A["k"], dtype=np.int64)
    ag = _group_col(A, len(ak))
    bk = np.ascontiguousarray(B["k"], dtype=np.int64)
    bh = _group_col(B, len(bk))
    av, avk = _vcol(A.get("v") if agg == "sum" else None)
    bw, bwk = _vcol(B.get("v") if agg == "sum" else None)
    res = _Result()
    ptr = lambda a: None if a is None else a.ctypes.data
    st = lib.oracle_join_agg(len(ak), ptr(ak), ptr(ag), ptr(av), avk,
                             len(bk), ptr(bk), ptr(bh), ptr(bw), bwk,
                             0 if agg == "count" else 1, int(threads), ctypes.byref(res))
    try:
        if st < 0:
            raise ValueError("oracle_join_agg: invalid arguments")
        n = res.n
        cp = lambda p, dt: np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True) if n else np.zeros(0, dt)
        out = {"g": cp(res.g, np.int64), "h": cp(res.h, np.int64), "cnt": cp(res.cnt, np.int64)}
        if agg == "sum":
            if avk == 2 or bwk == 2:
                out["sum"] = cp(res.fsum, np.float64)
                out["abs"] = cp(res.fabs_sum, np.float64)
            else:
                out["sum"] = cp(res.isum, np.int64)
        if st == 1:
            raise OracleOverflow("integer SUM exceeds int64")
        return _ungrouped(A, B, out)
    finally:
        lib.oracle_free(ctypes.byref(res))


def chain_join_agg(A, B, C, agg="count", threads: int = 0):
    """SELECT A.g, C.h, agg FROM A, B, C WHERE A.k = B.k AND B.g = C.k GROUP BY A.g, C.h.

    PAPER.md §3.2 multi-way joins, in the paper's join order A -> B -> C:
    (1) A ⋈ B, (2) its nonzero() tuples (A.g, B.ID_2, agg) re-encoded as a table,
    (3) that table ⋈ C. agg: "count" or "sum" (SUM(A.v * B.w * C.x), integer values).
    B's "g" column is its second join attribute ID_2."""
    t = join_agg(A, B, agg, threads)
    T = {"k": t["h"], "g": t["g"], "v": t["cnt"] if agg == "count" else t["sum"]}
    C2 = {"k": C["k"], "g": C["g"], "v": C.get("v") if agg == "sum" else None}
    r = join_agg(T, C2, "sum", threads)
    return {"g": r["g"], "h": r["h"], "cnt_triples": r["sum"] if agg == "count" else None,
            "sum": r["sum"], "pairs": r["cnt"]}


def chain_nested_loop(A, B, C, agg="count"):
    """Brute force over all triples (i, j, l) — tiny inputs only."""
    res = {}
    av = A.get("v") if agg == "sum" else None
    bw = B.get("v") if agg == "sum" else None
    cx = C.get("v") if agg == "sum" else None
    for i in range(len(A["k"])):
        for j in range(len(B["k"])):
            if int(A["k"][i]) != int(B["k"][j]):
                continue
            for l in range(len(C["k"])):
                if int(B["g"][j]) != int(C["k"][l]):
                    continue
                key = (int(A["g"][i]), int(C["g"][l]))
                x = 1
                if agg == "sum":
                    x = (int(av[i]) if av is not None else 1) * (int(bw[j]) if bw is not None else 1) * \
                        (int(cx[l]) if cx is not None else 1)
                res[key] = res.get(key, 0) + x
    keys = sorted(res)
    return {"g": np.array([k[0] for k in keys], np.int64), "h": np.array([k[1] for k in keys], np.int64),
            "sum": np.array([res[k] for k in keys], np.int64)}


def triangles(src, dst, threads: int = 0) -> int:
    """Number of triangles of the simple undirected graph on the edge list."""
    lib = _load()
    s = np.ascontiguousarray(src, dtype=np.int64)
    d = np.ascontiguousarray(dst, dtype=np.int64)
    return int(lib.oracle_triangles(len(s), s.ctypes.data, d.ctypes.data, int(threads)))


def nested_loop(A, B, agg="count"):
    """Brute force over all pairs (i, j) — tiny inputs only.

    Exact arithmetic: Python ints for integer values, and for float32 values
    Python floats summed with math.fsum over exact products (fp32*fp32 is exact
    in fp64) — i.e. the correctly rounded sum of the exact products.
    """
    import math
    from fractions import Fraction
    ak, bk = list(map(int, A["k"])), list(map(int, B["k"]))
    ag = list(map(int, A["g"])) if A.get("g") is not None else [0] * len(ak)
    bh = list(map(int, B["g"])) if B.get("g") is not None else [0] * len(bk)
    av = A.get("v") if agg != "count" else None
    bw = B.get("v") if agg != "count" else None
    is_float = (av is not None and np.asarray(av).dtype.kind == "f") or \
               (bw is not None and np.asarray(bw).dtype.kind == "f")
    conv = float if is_float else int
    avl = [conv(x) for x in av] if av is not None else [conv(1)] * len(ak)
    bwl = [conv(x) for x in bw] if bw is not None else [conv(1)] * len(bk)
    groups = {}
    for i in range(len(ak)):
        for j in range(len(bk)):
            if ak[i] == bk[j]:
                groups.setdefault((ag[i], bh[j]), []).append(avl[i] * bwl[j])
    keys = sorted(groups)
    out = {"g": np.array([k[0] for k in keys], dtype=np.int64),
           "h": np.array([k[1] for k in keys], dtype=np.int64),
           "cnt": np.array([len(groups[k]) for k in keys], dtype=np.int64)}
    if agg in ("sum", "avg"):
        if is_float:
            out["sum"] = np.array([math.fsum(groups[k]) for k in keys], dtype=np.float64)
            out["abs"] = np.array([math.fsum(abs(x) for x in groups[k]) for k in keys], dtype=np.float64)
        else:
            sums = [sum(groups[k]) for k in keys]
            if any(s > 2**63 - 1 or s < -2**63 for s in sums):
                raise OracleOverflow("integer SUM exceeds int64")
            out["sum"] = np.array(sums, dtype=np.int64)
    if agg == "avg":
        # the mean of each group's products: exact rational, rounded once (integers);
        # fsum of the exact products / count (floats)
        if is_float:
            out["avg"] = np.array([math.fsum(groups[k]) / len(groups[k]) for k in keys], dtype=np.float64)
        else:
            out["avg"] = np.array([float(Fraction(sum(groups[k]), len(groups[k]))) for k in keys], dtype=np.float64)
    return _ungrouped(A, B, out)
