"""The collective tcudb_join_agg (csrc/collective.cu) at P = 2, 4, 8 ranks on ONE GPU.

NCCL refuses two ranks on one device, so the ranks here are P host threads of this
process, each with its own libtcudb context and CUDA stream, connected by the test
communicator tests/nccl_shim (the NCCL entry points collective.cu resolves, selected
with TCUDB_NCCL_LIB). Everything else is the product path: agreement, balanced range
bounds, tcudb_partition routing, all-to-all-v / allgather-v exchanges, the local
query, the result gather, Q4 partials — against the oracle on the unsharded tables.
"""
import ctypes
import os
import threading

import numpy as np
import pytest

import datagen
from parity_util import compare

pytestmark = pytest.mark.gpu

KEY = {"count": "cnt", "sum": "sum", "avg": "avg"}


@pytest.fixture(scope="module")
def shim():
    from paper_2112_07552_b200 import build
    path = build.build_shim()
    os.environ["TCUDB_NCCL_LIB"] = path  # read by tcudb_create (nccl_attach)
    lib = ctypes.CDLL(path)
    lib.shim_world_create.restype = ctypes.c_void_p
    lib.shim_world_create.argtypes = [ctypes.c_int, ctypes.c_double]
    lib.shim_comm.restype = ctypes.c_void_p
    lib.shim_comm.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.shim_world_destroy.argtypes = [ctypes.c_void_p]
    lib.shim_world_broken.argtypes = [ctypes.c_void_p]
    lib.shim_world_why.argtypes = [ctypes.c_void_p]
    lib.shim_world_why.restype = ctypes.c_char_p
    lib.shim_calls.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.shim_calls.restype = ctypes.c_longlong
    lib.shim_bytes_in.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.shim_bytes_in.restype = ctypes.c_longlong
    yield lib
    os.environ.pop("TCUDB_NCCL_LIB", None)


def run_ranks(shim, P, slices, agg, flags=0, host=False, timeout=120.0):
    """slices[r] = (A_r, B_r) host tables of rank r. Returns (results, errors, calls, bytes)."""
    import torch
    from paper_2112_07552_b200 import Engine, TcudbError
    world = shim.shim_world_create(P, timeout)
    res, err = [None] * P, [None] * P

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                eng = Engine(0, comm=shim.shim_comm(world, r))
                try:
                    A, B = slices[r]
                    if host:
                        out = eng.join_agg_host({k: v for k, v in A.items() if v is not None},
                                                {k: v for k, v in B.items() if v is not None}, agg, flags=flags)
                        res[r] = {k: np.array(v) for k, v in out.items()}
                    else:
                        dev = lambda T: {k: torch.from_numpy(np.ascontiguousarray(v)).cuda()  # noqa: E731
                                         for k, v in T.items() if v is not None}
                        out = eng.join_agg(dev(A), dev(B), agg, flags=flags)
                        res[r] = {k: v.cpu().numpy() for k, v in out.items()}
                        del out
                    s.synchronize()
                except TcudbError as e:
                    err[r] = e
                finally:
                    eng.close()
        except Exception as e:  # noqa: BLE001 - reported by the test
            err[r] = e
    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout + 60)
        assert not t.is_alive(), "rank thread hung"
    calls = [shim.shim_calls(world, r) for r in range(P)]
    nbytes = [shim.shim_bytes_in(world, r) for r in range(P)]
    broken = shim.shim_world_why(world).decode() if shim.shim_world_broken(world) else ""
    shim.shim_world_destroy(world)
    return res, err, calls, nbytes, broken


def contiguous(A, B, P):
    return [(datagen.local_slice(A, P, r), datagen.local_slice(B, P, r)) for r in range(P)]


def variant(A, B, drop):
    if "a" in drop:
        A = dict(A, g=None)
    if "b" in drop:
        B = dict(B, g=None)
    return A, B


def _diff_report(r, out, ref):
    """which (g, h) groups a rank's result has that the oracle lacks (and vice versa)"""
    import json
    got = set(zip(np.asarray(out["g"]).tolist(), np.asarray(out["h"]).tolist())) if "g" in out and "h" in out else set()
    want = set(zip(ref["g"].tolist(), ref["h"].tolist())) if "g" in ref and "h" in ref else set()
    extra, missing = sorted(got - want)[:20], sorted(want - got)[:20]
    dup = len(out["agg"]) - len(got)
    rep = {"rank": r, "n": int(len(out["agg"])), "n_ref": int(len(ref["cnt"])), "duplicates": int(dup),
           "extra": [list(map(int, x)) for x in extra], "missing": [list(map(int, x)) for x in missing]}
    if dup and "g" in out and "h" in out:
        # where the repeated groups sit: (g, h) order breaks at the start of a repeated run
        g, h = np.asarray(out["g"]).astype(np.int64), np.asarray(out["h"]).astype(np.int64)
        brk = np.nonzero((g[1:] < g[:-1]) | ((g[1:] == g[:-1]) & (h[1:] <= h[:-1])))[0]
        rep["order_breaks"] = [[int(i + 1), int(g[i]), int(h[i]), int(g[i + 1]), int(h[i + 1])] for i in brk[:20]]
        rep["n_order_breaks"] = int(len(brk))
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "collective_diff.jsonl"), "a") as f:
        f.write(json.dumps(rep) + "\n")
    return rep


def check_all(res, err, ref, agg, float_vals, broken=""):
    assert all(e is None for e in err), (err, broken)
    for r, out in enumerate(res):
        try:
            compare(out, ref, agg, float_vals=float_vals)
        except AssertionError as e:
            raise AssertionError(f"rank {r}: {e}; {_diff_report(r, out, ref)}") from None


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("name,scale", [("c1", 1.0), ("c1s", 1.0), ("c2", 0.1), ("c3", 1 / 16), ("c5s", 1 / 64)])
def test_collective_configs(shim, oracle_mod, P, name, scale):
    A, B, agg = datagen.make_config(name, scale)
    ref = oracle_mod.join_agg(A, B, agg)
    res, err, calls, nbytes, broken = run_ranks(shim, P, contiguous(A, B, P), agg)
    check_all(res, err, ref, agg, False)
    assert not broken and all(c > 0 for c in calls) and all(b > 0 for b in nbytes)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("name,drop,agg", [("c1s", "", "avg"), ("c1s", "a", "sum"), ("c1s", "b", "avg"),
                                           ("c1s", "ab", "sum"), ("c1s", "ab", "avg"), ("c2", "ab", "count"),
                                           ("c4", "", "sum"), ("c4s", "ab", "avg")])
def test_collective_f2_shapes(shim, oracle_mod, P, name, drop, agg):
    """AVG with both sides grouped, Q3 on either side (route the grouped side), Q4 (partials
    combined exactly) and float SUM, sharded."""
    A, B, _ = datagen.make_config(name, 1 / 1024 if name.startswith("c4") else 1.0)
    A, B = variant(A, B, drop)
    ref = oracle_mod.join_agg(A, B, agg)
    res, err, *_ = run_ranks(shim, P, contiguous(A, B, P), agg)
    if drop == "ab" and name.startswith("c4"):
        # Q4 float partials are added in rank order, not in the one-pass oracle's order
        assert all(e is None for e in err), err
        for out in res:
            assert np.allclose(out["agg"], ref[KEY[agg]], rtol=1e-9, atol=0)
        return
    check_all(res, err, ref, agg, name.startswith("c4"))


@pytest.mark.parametrize("P", [2, 8])
def test_collective_gather_none_shards(shim, oracle_mod, P):
    """TCUDB_GATHER_NONE: each rank keeps its (g, h)-sorted shard; the rank-order
    concatenation is the single-GPU result."""
    from paper_2112_07552_b200 import GATHER_NONE
    A, B, agg = datagen.make_config("c2", 0.1)
    ref = oracle_mod.join_agg(A, B, agg)
    res, err, *_ = run_ranks(shim, P, contiguous(A, B, P), agg, flags=GATHER_NONE)
    assert all(e is None for e in err), err
    cat = {k: np.concatenate([r[k] for r in res]) for k in ("g", "h", "agg")}
    compare(cat, ref, agg)
    sizes = [len(r["agg"]) for r in res]
    assert min(sizes) > 0.5 * max(sizes), sizes  # row-balanced ranges (c2: 1 g value = 1 record)


def test_collective_host_api(shim, oracle_mod):
    A, B, agg = datagen.make_config("c1s")
    ref = oracle_mod.join_agg(A, B, agg)
    res, err, *_ = run_ranks(shim, 4, contiguous(A, B, 4), agg, host=True)
    check_all(res, err, ref, agg, False)


@pytest.mark.parametrize("agg", ["count", "sum", "avg"])
def test_collective_empty_and_skewed_ranks(shim, oracle_mod, agg):
    """Ranks with empty slices (NULL columns: torch's data_ptr of an empty tensor is 0),
    all of A on one rank, and group ranges that own no groups or no joined pairs."""
    A, B, _ = datagen.make_config("c1s")
    P = 8
    n = len(A["k"])
    # A: everything on rank 3; B: ranks 0 and 5 only; 2 distinct g values -> most ranges empty
    A = dict(A, g=np.where(A["g"] > np.median(A["g"]), 7, -7).astype(A["g"].dtype))
    sl = []
    for r in range(P):
        a = {k: (v if r == 3 else v[:0]) if v is not None else None for k, v in A.items()}
        hb = len(B["k"]) // 2
        b = {k: (v[:hb] if r == 0 else v[hb:] if r == 5 else v[:0]) if v is not None else None for k, v in B.items()}
        sl.append((a, b))
    assert n > 0
    ref = oracle_mod.join_agg(A, B, agg)
    res, err, _, _, broken = run_ranks(shim, P, sl, agg)
    check_all(res, err, ref, agg, False, broken)
    # no joined pairs at all on the routed side's owners: disjoint keys
    B2 = dict(B, k=B["k"] + 10 ** 6)
    ref2 = oracle_mod.join_agg(A, B2, agg)
    assert len(ref2["cnt"]) == 0
    res, err, *_ = run_ranks(shim, P, contiguous(A, B2, P), agg)
    assert all(e is None for e in err), err
    assert all(len(r["agg"]) == 0 and set(r) == {"g", "h", "agg"} for r in res)


def test_collective_errors_agreed(shim):
    """One rank's error is every rank's error (no rank left in a collective): a
    non-finite value on one rank (local query), value columns present on one rank only
    (shape disagreement), an int64 Q4 total that only overflows across ranks."""
    from paper_2112_07552_b200._lib import TCUDB_E_INVALID, TCUDB_E_OVERFLOW, TCUDB_E_UNSUPPORTED
    A, B, _ = datagen.make_config("c1s")
    Af = dict(A, v=A["v"].astype(np.float32))
    Bf = dict(B, v=B["v"].astype(np.float32))
    sl = contiguous(Af, Bf, 2)
    bad = dict(sl[1][0], v=sl[1][0]["v"].copy())
    bad["v"][3] = np.nan
    sl[1] = (bad, sl[1][1])
    res, err, _, _, broken = run_ranks(shim, 2, sl, "sum")
    assert not broken
    assert all(e is not None and e.status == TCUDB_E_UNSUPPORTED for e in err), err
    sl = contiguous(A, B, 2)
    sl[0] = (dict(sl[0][0], v=None), sl[0][1])
    res, err, _, _, broken = run_ranks(shim, 2, sl, "sum")
    assert all(e is not None and e.status == TCUDB_E_INVALID for e in err), err
    assert not broken
    # Q4: each rank's partial = 6.25e18 (fits int64, within the per-rank guard); total 1.25e19
    big = 2_500_000_000
    a = {"k": np.array([1], np.int64), "g": None, "v": np.array([big], np.int64)}
    b = {"k": np.array([1], np.int64), "g": None, "v": np.array([big], np.int64)}
    b0 = {"k": b["k"][:0], "g": None, "v": b["v"][:0]}
    res, err, _, _, broken = run_ranks(shim, 2, [(a, b), (a, b0)], "sum")
    assert all(e is not None and e.status == TCUDB_E_OVERFLOW for e in err), err
    assert not broken
    # ... and one rank alone is fine
    res, err, *_ = run_ranks(shim, 2, [(a, b), ({k: (v[:0] if v is not None else None) for k, v in a.items()}, b0)],
                             "sum")
    assert all(e is None for e in err) and all(int(r["agg"][0]) == big * big for r in res)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("name,scale", [("c1", 1.0), ("c1s", 1.0), ("c2", 0.1), ("c3", 1 / 16), ("c5s", 1 / 64)])
def test_collective_key_partitioned(shim, oracle_mod, P, name, scale):
    """§8(f) f4: the key-partitioned path (both sides routed by key hash, partial groups
    merged by g range through a join + group-by) forced with TCUDB_KEY_PARTITIONED."""
    from paper_2112_07552_b200._lib import KEY_PARTITIONED
    A, B, agg = datagen.make_config(name, scale)
    ref = oracle_mod.join_agg(A, B, agg)
    res, err, calls, nbytes, broken = run_ranks(shim, P, contiguous(A, B, P), agg, flags=KEY_PARTITIONED)
    check_all(res, err, ref, agg, False, broken)


def test_collective_key_partitioned_default_and_shards(shim, oracle_mod):
    """c5 at 1/4 scale (B: 4 M rows) takes the key-partitioned path by default; GATHER_NONE
    shards concatenate to the single-GPU result; ROW_SHARDED forces the other path."""
    from paper_2112_07552_b200._lib import GATHER_NONE, ROW_SHARDED
    A, B, agg = datagen.make_config("c5", 1 / 4)
    ref = oracle_mod.join_agg(A, B, agg)
    res, err, *_ = run_ranks(shim, 4, contiguous(A, B, 4), agg, flags=GATHER_NONE)
    assert all(e is None for e in err), err
    cat = {k: np.concatenate([r[k] for r in res]) for k in ("g", "h", "agg")}
    compare(cat, ref, agg)
    res, err, *_ = run_ranks(shim, 2, contiguous(A, B, 2), agg, flags=ROW_SHARDED)
    check_all(res, err, ref, agg, False)
