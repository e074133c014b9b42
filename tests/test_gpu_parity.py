"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Integer results (COUNT, integer SUM) must be bit-exact; float SUM within the
floored 1e-3 relative tolerance of DESIGN.md R9. Every test calls
libtcudb.so through paper_2112_07552_b200.Engine (ctypes -> C ABI).
"""
import os

import numpy as np
import pytest

import datagen
from parity_util import compare, res_np, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture(scope="module")
def engine(torch_mod):
    from paper_2112_07552_b200 import Engine
    e = Engine(0)
    yield e
    e.close()


def run(engine, torch_mod, A, B, agg, flags=0):
    out, st = engine.join_agg(to_dev(A, torch_mod), to_dev(B, torch_mod), agg, flags=flags, with_stats=True)
    return res_np(out), st


# ---------------------------------------------------------------- a6: the GEMM alone
# M % 256 == 0 -> CTA-pair kernel (cta_group::2); M = 128, 1152 -> 1-CTA kernel
@pytest.mark.parametrize("M,N,K", [(128, 256, 128), (256, 512, 384), (512, 768, 1024), (1152, 256, 2048),
                                   (2048, 1024, 640), (4096, 256, 128)])
@pytest.mark.parametrize("sa,sb", [(0, 0), (1, 1), (0, 1), (1, 0)])
def test_gemm_int8_exact(engine, torch_mod, M, N, K, sa, sb):
    torch = torch_mod
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K + 3 * sa + sb)
    def mk(r, signed):
        x = torch.randint(-128 if signed else 0, 128 if signed else 256, (r, K), generator=g, device="cuda",
                          dtype=torch.int32)
        return x.to(torch.int8) if signed else x.to(torch.uint8)
    A, B = mk(M, sa), mk(N, sb)
    C = engine.gemm(A, B, a_signed=sa, b_signed=sb)
    ref = (A.to(torch.float64) @ B.to(torch.float64).T)
    assert torch.equal(C.to(torch.float64), ref)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (384, 512, 1024), (512, 512, 256), (1024, 768, 2048)])
def test_gemm_bf16(engine, torch_mod, M, N, K):
    torch = torch_mod
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, generator=g, device="cuda").to(torch.bfloat16)
    C = engine.gemm(A, B)
    ref = A.to(torch.float64) @ B.to(torch.float64).T
    scale = (A.abs().to(torch.float64) @ B.abs().to(torch.float64).T)
    assert torch.all((C.to(torch.float64) - ref).abs() <= 1e-5 * scale + 1e-6)


# ---------------------------------------------------------------- random tiny instances
@pytest.mark.parametrize("vkind", ["none", "int", "float"])
@pytest.mark.parametrize("flags", [0, 1, 2])  # auto, FORCE_DENSE, FORCE_SPARSE
def test_random_tiny_vs_oracle(engine, torch_mod, oracle_mod, vkind, flags):
    rng = np.random.default_rng(100 + flags)
    agg = "count" if vkind == "none" else "sum"
    for _ in range(60):
        A, B = datagen.random_tiny(rng, n_max=80, vkind=vkind, vmin=-20, vmax=20, allow_empty=True)
        ref = oracle_mod.join_agg(A, B, agg)
        out, _ = run(engine, torch_mod, A, B, agg, flags)
        compare(out, ref, agg, float_vals=(vkind == "float"))


# ---------------------------------------------------------------- §8(f) f2: AVG, Q3, Q4
@pytest.mark.parametrize("vkind", ["none", "int", "float"])
@pytest.mark.parametrize("shape", ["gh", "h_only", "g_only", "none"])
def test_f2_random_tiny_vs_oracle(engine, torch_mod, oracle_mod, vkind, shape):
    """COUNT / SUM / AVG with both sides grouped, one side ungrouped (Q3) or none (Q4)."""
    rng = np.random.default_rng(300 + len(shape) + {"none": 0, "int": 1, "float": 2}[vkind])
    for _ in range(25):
        A, B = datagen.random_tiny(rng, n_max=80, vkind=vkind, vmin=-20, vmax=20, allow_empty=True)
        if shape in ("h_only", "none"):
            A = dict(A, g=None)
        if shape in ("g_only", "none"):
            B = dict(B, g=None)
        for agg in ("count", "sum", "avg"):
            ref = oracle_mod.join_agg(A, B, agg)
            out, st = run(engine, torch_mod, A, B, agg, 0)
            compare(out, ref, agg, float_vals=(vkind == "float"))


@pytest.mark.parametrize("name,scale,shape,agg", [
    ("c2", 0.1, "h_only", "count"), ("c5s", 1 / 64, "h_only", "sum"), ("c5s", 1 / 64, "g_only", "avg"),
    ("c5s", 1 / 64, "none", "sum"), ("c4", 1 / 256, "h_only", "sum"), ("c4", 1 / 256, "none", "avg"),
    ("c5s", 1 / 256, "gh", "avg"), ("c4", 1 / 1024, "gh", "avg"), ("c2", 0.05, "gh", "avg"),
    ("c4s", 1 / 256, "h_only", "sum"), ("c4s", 1 / 1024, "gh", "avg")])
def test_f2_configs_vs_oracle(engine, torch_mod, oracle_mod, name, scale, shape, agg):
    """f2 on the configs' distributions: Q3 / Q4 shapes take the segmented-reduction path
    (stats path 2); two-sided AVG composes the SUM and COUNT queries."""
    A, B, _ = datagen.make_config(name, scale)
    if shape in ("h_only", "none"):
        A = dict(A, g=None)
    if shape in ("g_only", "none"):
        B = dict(B, g=None)
    ref = oracle_mod.join_agg(A, B, agg)
    out, st = run(engine, torch_mod, A, B, agg, 0)
    if shape != "gh":
        assert st["path"] == 2
    compare(out, ref, agg, float_vals=name.startswith("c4"))


def test_wide_count_path_matches(engine, torch_mod, oracle_mod):
    """FORCE_WIDE: int64 scratch + digit-plane guard path for COUNT, and cells > 255
    (a carry out of the packed u8 byte) — both exact."""
    rng = np.random.default_rng(5)
    A = datagen.Table(rng.integers(0, 3, 5000).astype(np.int32), rng.integers(0, 2, 5000).astype(np.int32))
    B = datagen.Table(rng.integers(0, 3, 4000).astype(np.int32), rng.integers(0, 3, 4000).astype(np.int32))
    ref = oracle_mod.join_agg(A, B, "count")
    for flags in (1, 1 | 16):
        out, st = run(engine, torch_mod, A, B, "count", flags)
        compare(out, ref, "count")
        assert st["path"] == 0


def test_int_sum_digit_planes(engine, torch_mod, oracle_mod):
    """Large integer values force multi-plane base-256 decompositions (s8 top digit)."""
    rng = np.random.default_rng(6)
    n = 3000
    for lo, hi in ((-100, 100), (0, 5000), (-(2 ** 20), 2 ** 20), (-(2 ** 23), 2 ** 23)):
        A = datagen.Table(rng.integers(0, 40, n), rng.integers(0, 30, n), rng.integers(lo, hi, n))
        B = datagen.Table(rng.integers(0, 40, n), rng.integers(0, 20, n), rng.integers(lo, hi, n))
        ref = oracle_mod.join_agg(A, B, "sum")
        for flags in (1, 2):
            out, st = run(engine, torch_mod, A, B, "sum", flags)
            compare(out, ref, "sum")


def test_overflow_reported(engine, torch_mod):
    from paper_2112_07552_b200 import TcudbError
    A = datagen.Table(np.zeros(4, np.int64), np.zeros(4, np.int64), np.full(4, 2 ** 62, np.int64))
    B = datagen.Table(np.zeros(1, np.int64), np.zeros(1, np.int64), np.full(1, 2, np.int64))
    with pytest.raises(TcudbError) as ei:
        run(engine, torch_mod, A, B, "sum")
    assert ei.value.status == -4


def test_empty_and_disjoint(engine, torch_mod):
    E = datagen.Table(np.zeros(0, np.int32), np.zeros(0, np.int32))
    A = datagen.Table(np.array([1, 2], np.int32), np.array([0, 0], np.int32))
    B = datagen.Table(np.array([3, 4], np.int32), np.array([0, 0], np.int32))
    for X, Y in ((E, A), (A, E), (A, B)):
        out, _ = run(engine, torch_mod, X, Y, "count")
        assert len(out["g"]) == 0


def test_int64_extreme_keys_hash_path(engine, torch_mod, oracle_mod):
    rng = np.random.default_rng(8)
    pool = np.array([-(2 ** 62), -5, 0, 7, 2 ** 62, 2 ** 61 + 3], dtype=np.int64)
    A = datagen.Table(pool[rng.integers(0, 6, 500)], rng.integers(-(2 ** 40), 2 ** 40, 500) // 2 ** 30 * 2 ** 30)
    B = datagen.Table(pool[rng.integers(0, 6, 400)], rng.integers(0, 7, 400).astype(np.int64) * (2 ** 50))
    ref = oracle_mod.join_agg(A, B, "count")
    for flags in (0, 1, 2):
        out, st = run(engine, torch_mod, A, B, "count", flags)
        compare(out, ref, "count")
        assert st["key_mode"] == 1


def test_zero_sum_groups_kept(engine, torch_mod, oracle_mod):
    A = datagen.Table(np.array([1, 1, 2], np.int32), np.array([0, 0, 1], np.int32), np.array([3, -3, 0], np.int32))
    B = datagen.Table(np.array([1, 2], np.int32), np.array([4, 4], np.int32), np.array([2, 5], np.int32))
    ref = oracle_mod.join_agg(A, B, "sum")
    for flags in (1, 2):
        out, st = run(engine, torch_mod, A, B, "sum", flags)
        compare(out, ref, "sum")
        assert st["existence"] == 1


@pytest.mark.parametrize("case", ["unique_exact", "dups_exact", "unique_inexact"])
@pytest.mark.parametrize("G", [1024, 8576])  # 64 bands in 64 coarse bins; 536 bands, 4 per coarse bin
def test_float_direct_fill_guard_large(engine, torch_mod, oracle_mod, case, G):
    """float SUM with >= 2^20 A tuples: the binned bf16 direct fill (row bands in shared
    memory) must detect a second tuple in a cell and non-bf16 values and hand over to the
    fp32-scratch path; every case matches the oracle (R9 tolerance)."""
    rng = np.random.default_rng({"unique_exact": 11, "dups_exact": 12, "unique_inexact": 13}[case] + G)
    K, n = 2048, 1_200_000
    if case == "dups_exact":
        cell = rng.integers(0, G * K, n)
    else:
        cell = rng.permutation(G * K)[:n]
    if case == "unique_inexact":
        v = rng.standard_normal(n).astype(np.float32)
    else:
        v = (rng.integers(-64, 65, n) / 8).astype(np.float32)
    A = datagen.Table((cell % K).astype(np.int32), (cell // K).astype(np.int32), v)
    nb = 3000
    B = datagen.Table(rng.integers(0, K, nb).astype(np.int32), rng.integers(0, 50, nb).astype(np.int32),
                      (rng.integers(-8, 9, nb) / 4).astype(np.float32))
    ref = oracle_mod.join_agg(A, B, "sum")
    out, st = run(engine, torch_mod, A, B, "sum", 1)
    compare(out, ref, "sum", float_vals=True)
    if case == "unique_exact":
        assert st["elem"] == 1


# SPA schedules: "one" = one persistent pass with look-back (forced even when skewed),
# "auto" = the selector's choice, "two" = count pass + legacy write kernel,
# "0" = C matrix in HBM (no shared-memory SPA)
@pytest.mark.parametrize("spa", ["one", "auto", "two", "0", "hub"])
@pytest.mark.parametrize("case", ["c3", "c5", "c5s", "wide_h", "skew_sum_float", "skew_sum_int", "hot_cell"])
def test_sparse_spa_and_matrix_paths(engine, torch_mod, oracle_mod, monkeypatch, spa, case):
    """The sparse path under every schedule — all exact against the oracle. wide_h has a
    wide H (~30 K groups: one u16 row per band); the skew cases put most updates
    in a few rows (hub: the opt-in hybrid hub-count + one-pass schedule); hot_cell drives
    one (g, h) COUNT past 65,535 (u16 cell overflow -> int32 rerun, from the hybrid schedule
    via the two-pass fallback)."""
    monkeypatch.setenv("TCUDB_SPA_HUB", "1" if spa == "hub" else "0")
    monkeypatch.setenv("TCUDB_NO_SPA", "1" if spa == "0" else "0")
    monkeypatch.setenv("TCUDB_NO_SPA_FUSED", "1" if spa == "two" else "0")
    monkeypatch.setenv("TCUDB_SPA_ONE_PASS", "1" if spa == "one" else "0")
    rng = np.random.default_rng(77)
    if case in ("c3", "c5", "c5s"):
        A, B, agg = datagen.make_config(case, {"c3": 1 / 16, "c5": 1 / 256, "c5s": 1 / 256}[case])
    elif case == "wide_h":
        n = 40000
        A = datagen.Table(rng.integers(0, 5000, n), rng.integers(0, 300, n))
        B = datagen.Table(rng.integers(0, 5000, n), rng.integers(0, 60000, n))
        agg = "count"
    elif case == "hot_cell":
        # key 7 joins 400 A tuples of g=5 with 200 B tuples of h=9: COUNT(5, 9) = 80,000
        n = 20000
        ka = np.concatenate([np.full(400, 7), rng.integers(100, 900000, n)])
        ga = np.concatenate([np.full(400, 5), rng.integers(0, 2000, n)])
        kb = np.concatenate([np.full(200, 7), rng.integers(100, 900000, n)])
        hb = np.concatenate([np.full(200, 9), rng.integers(0, 2000, n)])
        A, B, agg = datagen.Table(ka, ga), datagen.Table(kb, hb), "count"
    else:
        n = 30000
        g = np.where(rng.random(n) < 0.5, 0, rng.integers(0, 3000, n))  # half the tuples in row 0
        k = rng.zipf(1.3, n) % 20000
        A = datagen.Table(k, g, rng.integers(-9, 10, n) if case == "skew_sum_int"
                          else rng.uniform(-2, 2, n).astype(np.float32))
        B = datagen.Table(rng.zipf(1.3, n) % 20000, rng.integers(0, 3000, n),
                          rng.integers(-9, 10, n) if case == "skew_sum_int" else rng.uniform(-2, 2, n).astype(np.float32))
        agg = "sum"
    ref = oracle_mod.join_agg(A, B, agg)
    out, st = run(engine, torch_mod, A, B, agg, 2)
    assert st["path"] == 1
    if spa == "0":
        assert st["spa_mode"] == 0
    elif spa == "two":
        assert st["spa_mode"] in (1, 2)
    elif spa == "one" and case != "hot_cell":  # a band past 65,535 updates: never one-pass COUNT
        assert st["spa_mode"] == 3
    compare(out, ref, agg, float_vals=(case == "skew_sum_float"))


# ---------------------------------------------------------------- configs (reduced + full)
@pytest.mark.parametrize("name,scale", [("c1", 1.0), ("c1s", 1.0), ("c2", 0.1), ("c3", 1 / 16), ("c4", 1 / 1024),
                                        ("c5", 1 / 256), ("c5s", 1 / 256)])
@pytest.mark.parametrize("flags", [0, 1, 2])
def test_configs_small(engine, torch_mod, oracle_mod, name, scale, flags):
    A, B, agg = datagen.make_config(name, scale)
    ref = oracle_mod.join_agg(A, B, agg)
    if name == "c4s" and scale > 1 / 256 and flags == 2:
        pytest.skip("forced sparse on a dense 1024^2 product: 1e9 pairs, no information beyond 1/1024")
    out, st = run(engine, torch_mod, A, B, agg, flags)
    if name == "c4s" and flags != 2:
        assert st["path"] == 0 and st["elem"] == 2  # not bf16-exact: the hi/lo split
    compare(out, ref, agg, float_vals=name.startswith("c4"))


def test_dense_equals_sparse_bitwise(engine, torch_mod):
    A, B, agg = datagen.make_config("c5s", 1 / 512)
    d, _ = run(engine, torch_mod, A, B, agg, 1)
    s, _ = run(engine, torch_mod, A, B, agg, 2)
    for k in ("g", "h", "agg"):
        assert np.array_equal(d[k], s[k])


@pytest.mark.parametrize("path", ["dense", "sparse"])
def test_triangles_textbook_and_random(engine, torch_mod, oracle_mod, monkeypatch, path):
    """a9 on both paths: the masked 2-hop GEMM (dense) and the oriented wedge check
    (tri_sparse.cu) — textbook closed forms and a random multigraph with self-loops."""
    monkeypatch.setenv("TCUDB_TRI_PATH", path)
    torch = torch_mod
    import math
    def tri(edges):
        s, d = (np.array(x, dtype=np.int32) for x in zip(*edges))
        return engine.triangle_count(torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
    for n in (3, 5, 10, 40):
        assert tri([(i, j) for i in range(n) for j in range(i + 1, n)]) == math.comb(n, 3)
    for n in (4, 9):
        rim = [(i, (i + 1) % n) for i in range(n)]
        assert tri(rim) == 0
        assert tri(rim + [(n, i) for i in range(n)]) == n
    rng = np.random.default_rng(3)
    s, d = rng.integers(0, 3000, 40000), rng.integers(0, 3000, 40000)
    got = engine.triangle_count(torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
    assert got == oracle_mod.triangles(s, d)


@pytest.mark.parametrize("path", ["dense", "sparse"])
def test_c3_triangles_reduced(engine, torch_mod, oracle_mod, monkeypatch, path):
    monkeypatch.setenv("TCUDB_TRI_PATH", path)
    torch = torch_mod
    s, d = datagen.c3_graph_edges(scale=12)
    got = engine.triangle_count(torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
    assert got == oracle_mod.triangles(s, d)


def test_c3_triangles_full_sparse(engine, torch_mod, oracle_mod):
    """The full c3 graph (R-MAT scale 16): the default (sparse) path vs the oracle, plus a
    star-heavy graph whose hub exercises the degree orientation."""
    torch = torch_mod
    s, d = datagen.c3_graph_edges()
    got, st = engine.triangle_count(torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda(), with_stats=True)
    assert st["path"] == 1
    assert got == oracle_mod.triangles(s, d)
    rng = np.random.default_rng(4)
    hub = np.zeros(60000, np.int64)
    leaves = rng.integers(1, 20000, 60000)
    ring_a = rng.integers(1, 20000, 100000)
    ring_b = rng.integers(1, 20000, 100000)
    s2 = np.concatenate([hub, ring_a]); d2 = np.concatenate([leaves, ring_b])
    got2 = engine.triangle_count(torch.from_numpy(s2).cuda(), torch.from_numpy(d2).cuda())
    assert got2 == oracle_mod.triangles(s2, d2)


# full-size configs in the launch configuration bench.py times (default flags)
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_configs_full_exact(engine, torch_mod, oracle_mod, name):
    A, B, agg = datagen.make_config(name)
    ref = oracle_mod.join_agg(A, B, agg)
    out, st = run(engine, torch_mod, A, B, agg, 0)
    compare(out, ref, agg)


@pytest.mark.parametrize("name,flags", [("c4", 0), ("c4s", 0), ("c4s", 1)])
def test_c4_full_sampled_and_freivalds(engine, torch_mod, oracle_mod, name, flags):
    """c4 / c4s at full size (8192^3): exact oracle on 64 sampled A rows, compared with the
    floored tolerance, + a Freivalds check y = C x vs A_op (B_op^T x) in fp64 over the
    whole result, bounded by the same tolerance propagated through x:
    |sum_j (C - C^)_ij x_j| <= 1e-3 sum_j (|C_ij| + FLOOR S_abs_ij) |x_j|."""
    from parity_util import FLOAT_RTOL, FLOOR
    A, B, agg = datagen.make_config(name)
    out, st = run(engine, torch_mod, A, B, agg, flags)
    assert st["path"] == 0 and st["elem"] == (2 if name == "c4s" else 1)
    n = 8192
    assert len(out["g"]) == n * n
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(n, 64, replace=False))
    sel = np.isin(A["g"], rows)
    Asub = datagen.Table(A["k"][sel], A["g"][sel], A["v"][sel])
    ref = oracle_mod.join_agg(Asub, B, "sum")
    m = np.isin(out["g"], rows)
    compare({k: v[m] for k, v in out.items()}, ref, "sum", float_vals=True)
    g64, h64 = out["g"].astype(np.int64), out["h"].astype(np.int64)
    x = rng.standard_normal(n)
    Cx = np.zeros(n)
    np.add.at(Cx, g64, out["agg"] * x[h64])
    Cabs = np.zeros(n)
    np.add.at(Cabs, g64, np.abs(out["agg"]) * np.abs(x[h64]))

    def a_bt(xv, absval):                   # (A (B^T xv))_i from the tuples, fp64
        bv = np.abs(B["v"].astype(np.float64)) if absval else B["v"].astype(np.float64)
        av = np.abs(A["v"].astype(np.float64)) if absval else A["v"].astype(np.float64)
        Btx = np.zeros(n)
        np.add.at(Btx, B["k"].astype(np.int64), bv * xv[B["g"].astype(np.int64)])
        r = np.zeros(n)
        np.add.at(r, A["g"].astype(np.int64), av * Btx[A["k"].astype(np.int64)])
        return r
    ABx = a_bt(x, False)
    Sx = a_bt(np.abs(x), True)              # sum_j S_abs_ij |x_j|
    bound = FLOAT_RTOL * (Cabs + FLOOR * Sx)
    assert np.all(np.abs(Cx - ABx) <= bound), float(np.max(np.abs(Cx - ABx) / bound))


# ---------------------------------------------------------------- multi-GPU building blocks (loopback)
def test_minmax_and_partition(engine, torch_mod):
    torch = torch_mod
    rng = np.random.default_rng(4)
    g = rng.integers(-1000, 5000, 100_000).astype(np.int64)
    T = {"k": torch.from_numpy(rng.integers(0, 99, len(g)).astype(np.int32)).cuda(),
         "g": torch.from_numpy(g).cuda(), "v": torch.from_numpy(rng.random(len(g)).astype(np.float32)).cuda()}
    assert engine.minmax(T["g"]) == (int(g.min()), int(g.max()))
    bounds = [0, 1000, 1001, 4000]
    out, counts = engine.partition(T, bounds)
    dest = np.searchsorted(np.array(bounds), g, side="right")
    assert counts == np.bincount(dest, minlength=5).tolist()
    og = out["g"].cpu().numpy()
    off = np.concatenate([[0], np.cumsum(counts)])
    for d in range(5):
        seg = og[off[d]:off[d + 1]]
        assert np.all(np.searchsorted(np.array(bounds), seg, side="right") == d)
    # rows are permuted intact (multiset of (k, g, v) triples preserved)
    trip = lambda T: np.sort(np.stack([T["k"].cpu().numpy().astype(np.float64), T["g"].cpu().numpy(),
                                       T["v"].cpu().numpy().astype(np.float64)], 1), axis=0)
    assert np.array_equal(trip(out), trip(T))


@pytest.mark.parametrize("P", [2, 8])
def test_loopback_row_sharding(engine, torch_mod, P):
    """the P-rank algorithm as P logical shards on one GPU (collectives
    replaced by slicing): concatenated per-range results == the single query. Ranges
    from the library's balanced planning step (tcudb_shard_bounds on a strided sample)."""
    from paper_2112_07552_b200._lib import shard_bounds, shard_sample_msg
    torch = torch_mod
    A, B, agg = datagen.make_config("c2", 0.2)
    dA, dB = to_dev(A, torch), to_dev(B, torch)
    full = res_np(engine.join_agg(dA, dB, agg))
    msgs = [shard_sample_msg(datagen.local_slice(A, P, r)["g"]) for r in range(P)]
    Ap, counts = engine.partition(dA, shard_bounds(msgs))
    assert min(counts) > 0.6 * max(counts), counts  # row-balanced
    off = np.concatenate([[0], np.cumsum(counts)])
    parts = []
    for r in range(P):
        Ar = {k: v[off[r]:off[r + 1]].contiguous() for k, v in Ap.items()}
        parts.append(res_np(engine.join_agg(Ar, dB, agg)))
    for k in ("g", "h", "agg"):
        assert np.array_equal(np.concatenate([p[k] for p in parts]), full[k])


PAIR_SCRIPT = r"""
import torch
from paper_2112_07552_b200 import Engine
e = Engine(0)
g = torch.Generator(device="cuda").manual_seed(7)
for (M, N, K) in [(256, 256, 128), (512, 768, 1024), (2048, 1024, 640)]:
    for sa, sb in [(0, 0), (1, 1), (0, 1)]:
        mk = lambda r, s: (torch.randint(-128, 128, (r, K), generator=g, device="cuda", dtype=torch.int32).to(torch.int8)
                           if s else torch.randint(0, 256, (r, K), generator=g, device="cuda", dtype=torch.int32).to(torch.uint8))
        A, B = mk(M, sa), mk(N, sb)
        C = e.gemm(A, B, a_signed=sa, b_signed=sb)
        assert torch.equal(C.double(), A.double() @ B.double().T), (M, N, K, sa, sb)
    A = torch.randn(M, K, generator=g, device="cuda").bfloat16(); B = torch.randn(N, K, generator=g, device="cuda").bfloat16()
    C = e.gemm(A, B)
    ref = A.double() @ B.double().T
    assert torch.all((C.double() - ref).abs() <= 1e-5 * (A.double().abs() @ B.double().abs().T) + 1e-6)
print("PAIR_OK")
"""


def test_gemm_cta_pair_kernel_exact():
    """The cta_group::2 kernel (TCUDB_GEMM_PAIR=1, read once per process) in a subprocess."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, TCUDB_GEMM_PAIR="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", PAIR_SCRIPT], env=env, cwd=root, capture_output=True, text=True,
                       timeout=300)
    assert "PAIR_OK" in r.stdout, r.stdout + r.stderr


# ---------------------------------------------------------------- e2m1 (fp4) operands, kind::mxf4
E2M1 = {0: 0, 1: 2, 2: 4, 3: 5, 4: 6, 6: 7}   # exact small integers in e2m1 (bias 1)


def _pack_e2m1(vals, torch):
    """uint8 [rows, K/2]: element 2j in the low nibble, 2j+1 in the high nibble."""
    lut = torch.zeros(8, dtype=torch.uint8, device=vals.device)
    for v, c in E2M1.items():
        lut[v] = c
    codes = lut[vals.long()]
    return (codes[:, 0::2] | (codes[:, 1::2] << 4)).contiguous()


@pytest.mark.parametrize("M,N,K,hi", [(128, 240, 256, 1), (256, 480, 1024, 4), (1024, 720, 2048, 6),
                                      (384, 240, 4096, 2)])
def test_gemm_fp4_exact_integers(engine, torch_mod, M, N, K, hi):
    torch = torch_mod
    g = torch.Generator(device="cuda").manual_seed(M + N + K + hi)
    allowed = torch.tensor([v for v in E2M1 if v <= hi], device="cuda")
    A = allowed[torch.randint(0, len(allowed), (M, K), generator=g, device="cuda")]
    B = allowed[torch.randint(0, len(allowed), (N, K), generator=g, device="cuda")]
    C = engine.gemm(_pack_e2m1(A, torch), _pack_e2m1(B, torch), fp4=True)
    assert torch.equal(C.double(), A.double() @ B.double().T)


def test_gemm_fp4_large_sums_exact(engine, torch_mod):
    """All-ones operands: every C = K; partial sums up to 20,480 stay exact in fp32."""
    torch = torch_mod
    K = 20480
    A = torch.ones(128, K, dtype=torch.int32, device="cuda")
    B = torch.ones(240, K, dtype=torch.int32, device="cuda")
    C = engine.gemm(_pack_e2m1(A, torch), _pack_e2m1(B, torch), fp4=True)
    assert torch.all(C == K)


@pytest.mark.parametrize("K,dens", [((1 << 22) - 256, 0.75), ((1 << 24) - 256, 0.9)])
def test_gemm_fp4_large_odd_sums_exact(engine, torch_mod, K, dens):
    """Random 0/1 operands with K up to 2^24: cell sums ~2.4 M and ~13.6 M, half of them
    odd, every MMA step adding a random count into an accumulator far above 2^20. Exact
    iff the kind::mxf4 fp32 accumulation keeps every integer < 2^24 (the e2m1 guard's
    claim, K < 2^24); the reference is a chunked fp64 product (exact below 2^53)."""
    torch = torch_mod
    g = torch.Generator(device="cuda").manual_seed(K)
    A = (torch.rand(128, K, generator=g, device="cuda") < dens).to(torch.uint8)
    B = (torch.rand(240, K, generator=g, device="cuda") < dens).to(torch.uint8)
    pack = lambda X: ((X * 2)[:, 0::2] | ((X * 2)[:, 1::2] << 4)).contiguous()  # noqa: E731
    C = engine.gemm(pack(A), pack(B), fp4=True).long()
    ref = torch.zeros(128, 240, dtype=torch.int64, device="cuda")
    for k0 in range(0, K, 1 << 16):
        ref += (A[:, k0:k0 + (1 << 16)].double() @ B[:, k0:k0 + (1 << 16)].double().T).long()
    assert ref.min().item() > (1 << 21) and (ref % 2).sum().item() > 1000
    assert torch.equal(C, ref)


@pytest.mark.parametrize("name,scale", [("c2", 0.1), ("c3", 1 / 16), ("c5", 1 / 256)])
def test_count_fp4_vs_u8_vs_oracle(engine, torch_mod, oracle_mod, monkeypatch, name, scale):
    """Dense COUNT through e2m1 operands (default), u8 operands (NO_FP4) and the oracle agree."""
    monkeypatch.setenv("TCUDB_FP4_ALWAYS", "1")  # these reduced products are below the e2m1 threshold
    A, B, agg = datagen.make_config(name, scale)
    ref = oracle_mod.join_agg(A, B, agg)
    o4, s4 = run(engine, torch_mod, A, B, agg, 1)
    o8, s8 = run(engine, torch_mod, A, B, agg, 1 | 32)
    # c2 (token sets) and c3 (simple graph) have 0/1 cells -> e2m1; c5's random groups put
    # several tuples in some (g, k) cells -> the fill detects it and falls back to u8
    assert s4["elem"] == (0 if name == "c5" else 3) and s8["elem"] == 0
    compare(o4, ref, agg)
    compare(o8, ref, agg)


@pytest.mark.parametrize("case", ["c2", "c3", "ragged", "many_tiles", "empty_rows"])
def test_fused_compaction_matches(engine, torch_mod, oracle_mod, monkeypatch, case):
    """f1: compaction inside the e2m1 GEMM kernel (TCUDB_FUSED_COMPACT=1) vs the separate
    compaction kernels (default) vs the oracle — bit-identical, (g, h)-ordered.
    ragged: G, H not multiples of the tiles; many_tiles: > 148 M-blocks x N-tiles with
    int64 group values; empty_rows: most A groups join nothing."""
    rng = np.random.default_rng(11)
    if case in ("c2", "c3"):
        A, B, agg = datagen.make_config(case, {"c2": 0.25, "c3": 1 / 8}[case])
    elif case == "ragged":
        def side(n_rec, vocab):
            rec = np.repeat(np.arange(n_rec), 7)
            tok = np.concatenate([rng.choice(vocab, 7, replace=False) for _ in range(n_rec)])
            return tok, rec
        ka, ga = side(1333, 700)
        kb, hb = side(977, 700)
        A, B, agg = datagen.Table(ka, ga * 3 + 5), datagen.Table(kb, hb - 400), "count"
    elif case == "many_tiles":
        def side(n_rec, vocab, L):
            rec = np.repeat(np.arange(n_rec), L)
            tok = np.concatenate([rng.choice(vocab, L, replace=False) for _ in range(n_rec)])
            return tok, rec
        ka, ga = side(9000, 4000, 5)
        kb, hb = side(6000, 4000, 5)
        A = datagen.Table(ka.astype(np.int64), (ga.astype(np.int64) << 33) + 1)
        B = datagen.Table(kb.astype(np.int64), hb.astype(np.int64) * 7 - (1 << 40))
        agg = "count"
    else:
        ka = rng.choice(50000, 30000, replace=False)
        ga = rng.integers(0, 20000, 30000)
        kb = np.concatenate([ka[:300], rng.integers(60000, 90000, 5000)])
        hb = rng.integers(0, 3000, len(kb))
        A, B, agg = datagen.Table(ka, ga), datagen.Table(kb, hb), "count"
    ref = oracle_mod.join_agg(A, B, agg)
    monkeypatch.setenv("TCUDB_FP4_ALWAYS", "1")
    monkeypatch.setenv("TCUDB_FUSED_COMPACT", "1")
    of, sf = run(engine, torch_mod, A, B, agg, 1)
    assert sf["elem"] == 3 and sf["fused_compact"] == 1
    compare(of, ref, agg)
    monkeypatch.setenv("TCUDB_FUSED_COMPACT", "0")
    ou, su = run(engine, torch_mod, A, B, agg, 1)
    assert su["fused_compact"] == 0
    for k in ("g", "h", "agg"):
        assert np.array_equal(of[k], ou[k])


@pytest.mark.parametrize("case", ["c5_64", "c5_16", "zipf", "int32_keys", "few_groups", "disjoint"])
def test_hash_partitioned_count(engine, torch_mod, oracle_mod, monkeypatch, case):
    """Hash-partitioned sparse COUNT (hashpart.cu; the default for c5-sized inputs) forced
    on smaller inputs, and the general path, both exact against the oracle. zipf: skewed
    keys (the plan may fall back when a partition outgrows shared memory)."""
    rng = np.random.default_rng(55)
    if case.startswith("c5"):
        A, B, agg = datagen.make_config("c5", {"c5_64": 1 / 64, "c5_16": 1 / 16}[case])
    elif case == "zipf":
        n = 300000
        A = datagen.Table(rng.zipf(1.2, n).astype(np.int64) * 7919 + (1 << 40), rng.integers(0, 500, n))
        B = datagen.Table(rng.zipf(1.2, n).astype(np.int64) * 7919 + (1 << 40), rng.integers(0, 700, n))
        agg = "count"
    elif case == "int32_keys":
        n = 200000
        A = datagen.Table(rng.integers(-2**31, 2**31 - 1, n).astype(np.int32) // 64, rng.integers(0, 3000, n))
        B = datagen.Table(rng.integers(-2**31, 2**31 - 1, n).astype(np.int32) // 64, rng.integers(0, 2000, n))
        agg = "count"
    elif case == "few_groups":
        n = 250000
        keys = rng.integers(0, 2**62, 60000)
        A = datagen.Table(rng.choice(keys, n), rng.integers(0, 3, n) * 1000003)
        B = datagen.Table(rng.choice(keys, n), rng.integers(0, 5, n) - 7)
        agg = "count"
    else:
        n = 100000
        A = datagen.Table(rng.integers(0, 2**40, n), rng.integers(0, 100, n))
        B = datagen.Table(rng.integers(2**41, 2**42, n), rng.integers(0, 100, n))
        agg = "count"
    ref = oracle_mod.join_agg(A, B, agg)
    monkeypatch.setenv("TCUDB_FORCE_HASHPART", "1")
    out, st = run(engine, torch_mod, A, B, agg, 0)
    compare(out, ref, agg)
    if case in ("c5_64", "c5_16"):  # (elsewhere the selector may prefer the dense path)
        assert st["spa_mode"] == 4
    if st["spa_mode"] == 4:  # the exact join size measured by the expand (c5_16: sampled count)
        assert st["join_pairs"] == int(ref["cnt"].sum())
    monkeypatch.setenv("TCUDB_FORCE_HASHPART", "0")
    monkeypatch.setenv("TCUDB_NO_HASHPART", "1")
    out2, st2 = run(engine, torch_mod, A, B, agg, 0)
    assert st2["spa_mode"] != 4
    compare(out2, ref, agg)


# ---------------------------------------------------------------- §8(f) f3: chain joins
def _chain_run(engine, torch_mod, A, B, C, agg, flags=0):
    out = engine.chain_join_agg(to_dev(A, torch_mod), to_dev(B, torch_mod), to_dev(C, torch_mod), agg, flags=flags)
    return res_np(out)


# flags: default (COUNT takes the chain exception when small), FORCE_DENSE (the matrix
# chain mat(A)·mat(B)^T·mat(C)^T), FORCE_SPARSE (the table route through nonzero())
@pytest.mark.parametrize("flags", [0, 1, 2])
def test_chain_join_tiny_vs_triple_loop(engine, torch_mod, oracle_mod, flags):
    rng = np.random.default_rng(32)
    for _ in range(40):
        A, B = datagen.random_tiny(rng, n_max=40, k_max=8, g_max=4, vkind="int", vmin=-4, vmax=4, allow_empty=False)
        C, _ = datagen.random_tiny(rng, n_max=40, k_max=8, g_max=4, vkind="int", vmin=-4, vmax=4, allow_empty=False)
        B = dict(B, g=rng.choice(np.concatenate([C["k"], [999]]), len(B["k"])))
        for agg in ("count", "sum"):
            got = _chain_run(engine, torch_mod, A, B, C, agg, flags)
            ref = oracle_mod.chain_nested_loop(A, B, C, agg)
            assert np.array_equal(got["g"].astype(np.int64), ref["g"])
            assert np.array_equal(got["h"].astype(np.int64), ref["h"])
            assert np.array_equal(got["agg"], ref["sum"])


@pytest.mark.parametrize("flags", [0, 1, 2])
def test_chain_three_hop_graphs(engine, torch_mod, oracle_mod, flags):
    """3-hop path counts (A -> B -> C over the edge table): K_9 closed form and the c3
    graph at 1/16 scale vs the oracle's join-order evaluation, on the chain exception
    (matrix chain, default / FORCE_DENSE) and the table route (FORCE_SPARSE)."""
    n = 9
    src, dst = (np.array(x) for x in zip(*[(i, j) for i in range(n) for j in range(n) if i != j]))
    E1, E2 = datagen.Table(dst, src), datagen.Table(src, dst)
    r = _chain_run(engine, torch_mod, E1, E2, E2, "count", flags)
    assert len(r["g"]) == n * n
    for g, h, c in zip(r["g"], r["h"], r["agg"]):
        assert c == ((n - 1) * (n - 2) if g == h else n * n - 3 * n + 3)
    A, B, _ = datagen.make_config("c3", 1 / 16)
    C = {"k": B["k"], "g": B["g"], "v": None}
    B2 = {"k": B["k"], "g": B["g"], "v": None}
    got = _chain_run(engine, torch_mod, A, B2, C, "count", flags)
    ref = oracle_mod.chain_join_agg(A, B2, C, "count")
    assert np.array_equal(got["g"].astype(np.int64), ref["g"]) and np.array_equal(got["h"].astype(np.int64), ref["h"])
    assert np.array_equal(got["agg"], ref["sum"])


NATIVE_SCRIPT = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
import datagen, oracle
from paper_2112_07552_b200 import Engine, GATHER_NONE, TcudbError
from datagen import local_slice
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
e = Engine(0, group=dist.group.WORLD)
assert e.collective
ws, rk = dist.get_world_size(), dist.get_rank()
KEY = {"count": "cnt", "sum": "sum", "avg": "avg"}
def check(out, ref, agg, tag):
    for c in ("g", "h"):
        assert (c in out) == (c in ref), (tag, c)
        if c in ref:
            assert np.array_equal(np.asarray(out[c].cpu() if hasattr(out[c], "cpu") else out[c]), ref[c]), (tag, c)
    got = np.asarray(out["agg"].cpu() if hasattr(out["agg"], "cpu") else out["agg"])
    want = ref[KEY[agg]]
    ok = np.allclose(got, want, rtol=1e-12, atol=0) if want.dtype == np.float64 else np.array_equal(got, want)
    assert ok, tag
for name, scale, drop, ag, flags in (("c1", 1.0, "", None, 0), ("c2", 0.1, "", None, 0), ("c1s", 1.0, "", None, 0),
                                     ("c1s", 1.0, "", "avg", 0), ("c1s", 1.0, "b", "sum", 0),
                                     ("c1s", 1.0, "a", "avg", 0), ("c1s", 1.0, "ab", "sum", 0),
                                     ("c1s", 1.0, "ab", "avg", 0), ("c2", 0.1, "ab", "count", 0),
                                     ("c1", 1.0, "", None, GATHER_NONE)):
    A, B, agg = datagen.make_config(name, scale)
    agg = ag or agg
    if "a" in drop: A = dict(A, g=None)
    if "b" in drop: B = dict(B, g=None)
    sA, sB = local_slice(A, ws, rk), local_slice(B, ws, rk)
    dev = lambda T: {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in T.items() if v is not None}
    out, st = e.join_agg(dev(sA), dev(sB), agg, flags=flags, with_stats=True)
    assert st["ms_comm"] >= 0
    ref = oracle.join_agg(A, B, agg)
    check(out, ref, agg, (name, drop, agg, flags))
    # collective host API: host slices in, the full result out
    hout = e.join_agg_host({k: v for k, v in sA.items() if v is not None},
                           {k: v for k, v in sB.items() if v is not None}, agg, flags=flags)
    check(hout, ref, agg, ("host", name, drop, agg))
# empty inputs on the collective path: empty result, no exchange errors
A, B, _ = datagen.make_config("c1")
Z = {k: v[:0] for k, v in A.items() if v is not None}
for agg in ("count", "sum", "avg"):
    for TA, TB in ((Z, B), (A, Z)):
        out = e.join_agg(dev(TA), dev(TB), agg)
        assert all(len(v) == 0 for v in out.values()), agg
    out = e.join_agg(dev(dict(Z, g=None)), dev(dict(B, g=None)), agg)
    assert len(out["agg"]) == 0, agg
# chain joins are single-GPU only on a collective context
try:
    e.chain_join_agg(dev(A), dev(B), dev(B), "count")
    raise SystemExit("chain on a collective context should fail")
except TcudbError:
    pass
dist.destroy_process_group()
print("NATIVE_OK")
"""


def test_native_collective_single_rank(tmp_path):
    """The collective tcudb_join_agg (collective.cu: NCCL resolved by dlopen, torch's
    communicator) on a 1-rank NCCL group: routing, all-to-all-v, allgather-v, Q3/Q4
    allreduces, GATHER_NONE and the host API, against the oracle."""
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "native_check.py"
    script.write_text(NATIVE_SCRIPT)
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)],
                       cwd=root, capture_output=True, text=True, timeout=600)
    assert "NATIVE_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def test_bench_collective_single_rank():
    """bench.py --force-shard under torchrun: the collective library call on a 1-rank
    NCCL group (real NCCL; the P > 1 exchanges run in test_collective_shim.py)."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--force-shard",
                        "--config", "c1", "--also", "", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                        "--e2e-steps", "1"],
                       cwd=root, capture_output=True, text=True, timeout=600)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert line, r.stdout[-3000:] + r.stderr[-3000:]
    d = json.loads(line[-1])
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and "row-shard" in d["config"]["parallelism"]


# ---------------------------------------------------------------- randomized sweep over the plans
# (plus the seeds of the 300-seed sweep that exposed the two-way split's residual: groups of a
# few float products missing the 1e-5 S_abs floor by up to 2x; fixed by the three-way split)
@pytest.mark.parametrize("seed", sorted(set(range(int(os.environ.get("TCUDB_FUZZ_SEEDS", "6"))))
                                        | {101, 108, 192, 215, 221, 235, 250}))
def test_fuzz_all_plans(engine, torch_mod, oracle_mod, monkeypatch, seed):
    """Random shapes (sizes, key/group spans and dtypes, skew, value kinds) through every
    plan the selector can take — auto, FORCE_DENSE, FORCE_SPARSE, the one-pass band kernel,
    the hash-partitioned path — and the f2 shapes; all against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    for it in range(6):
        n_a, n_b = int(rng.integers(1, 60000)), int(rng.integers(1, 60000))
        kspan = int(rng.choice([50, 3000, 10 ** 6, 2 ** 40]))
        zipf = rng.random() < 0.3
        def keys(n):
            k = (rng.zipf(1.3, n) % kspan) if zipf else rng.integers(0, kspan, n)
            return (k * int(rng.choice([1, 7919])) - kspan // 3).astype(rng.choice([np.int32, np.int64]) if kspan < 2 ** 30 else np.int64)
        G, H = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
        vk = rng.choice(["none", "int", "float"])
        def vals(n):
            if vk == "none":
                return None
            if vk == "int":
                return rng.integers(-30, 31, n).astype(rng.choice([np.int32, np.int64]))
            return rng.uniform(-4, 4, n).astype(np.float32)
        A = datagen.Table(keys(n_a), rng.integers(0, G, n_a) * 3 - 100, vals(n_a))
        B = datagen.Table(keys(n_b), rng.integers(0, H, n_b) - 7, vals(n_b))
        agg = "count" if vk == "none" else rng.choice(["sum", "avg"])
        ref = oracle_mod.join_agg(A, B, agg)
        for flags, env in ((0, {}), (1, {}), (2, {}), (2, {"TCUDB_SPA_ONE_PASS": "1"}),
                           (0, {"TCUDB_FORCE_HASHPART": "1"})):
            for k_, v_ in env.items():
                monkeypatch.setenv(k_, v_)
            out, st = run(engine, torch_mod, A, B, agg, flags)
            compare(out, ref, agg, float_vals=(vk == "float"))
            for k_ in env:
                monkeypatch.delenv(k_)
        # f2 shapes on the same tables
        for shape in ("h_only", "none"):
            A2 = dict(A, g=None)
            B2 = B if shape == "h_only" else dict(B, g=None)
            ref2 = oracle_mod.join_agg(A2, B2, agg)
            out2, _ = run(engine, torch_mod, A2, B2, agg, 0)
            compare(out2, ref2, agg, float_vals=(vk == "float"))


def test_u8_count_long_k_and_wide_retry(engine, torch_mod, oracle_mod):
    """Dense COUNT with K > 32 K keys (the u8 fill is checked before the GEMM and the int32
    accumulation is chunked) and, separately, a cell past 255 caught by the optimistic u8
    check (rerun on the int64 wide path)."""
    rng = np.random.default_rng(8)
    K = 40000
    ka = np.concatenate([np.arange(K), rng.integers(0, K, 30000)])
    A = datagen.Table(ka, rng.integers(0, 200, len(ka)))
    B = datagen.Table(rng.integers(0, K, 50000), rng.integers(0, 300, 50000))
    ref = oracle_mod.join_agg(A, B, "count")
    out, st = run(engine, torch_mod, A, B, "count", 1)
    assert st["path"] == 0 and st["elem"] == 0
    compare(out, ref, "count")
    # 300 copies of one (g, k) cell: the optimistic u8 fill overflows and the query reruns wide
    A2 = datagen.Table(np.concatenate([np.full(300, 5), rng.integers(0, 100, 2000)]),
                       np.concatenate([np.full(300, 1), rng.integers(0, 50, 2000)]))
    B2 = datagen.Table(rng.integers(0, 100, 3000), rng.integers(0, 60, 3000))
    ref2 = oracle_mod.join_agg(A2, B2, "count")
    out2, st2 = run(engine, torch_mod, A2, B2, "count", 1)
    compare(out2, ref2, "count")


@pytest.mark.parametrize("case", ["c5s_64", "c5s_16", "one_side_values", "negative_cancel"])
def test_hash_partitioned_int_sum(engine, torch_mod, oracle_mod, monkeypatch, case):
    """Integer SUM on the hash-partitioned path (value payload through both radix passes, a
    wrapping int64 plane plus a COUNT plane for existence) vs the oracle and vs the general
    path; SUM = 0 groups are kept (R3)."""
    rng = np.random.default_rng(66)
    if case.startswith("c5s"):
        A, B, _ = datagen.make_config("c5s", {"c5s_64": 1 / 64, "c5s_16": 1 / 16}[case])
    elif case == "one_side_values":
        n = 200000
        A = datagen.Table(rng.integers(0, 2 ** 45, n), rng.integers(0, 400, n), rng.integers(-1000, 1000, n))
        B = datagen.Table(A["k"][rng.integers(0, n, n)], rng.integers(0, 300, n))
    else:
        n = 150000
        keys = rng.integers(0, 2 ** 50, 40000)
        A = datagen.Table(rng.choice(keys, n), rng.integers(0, 50, n), rng.choice([-1, 1], n).astype(np.int32))
        B = datagen.Table(rng.choice(keys, n), rng.integers(0, 50, n), rng.choice([-2, 2], n).astype(np.int32))
    ref = oracle_mod.join_agg(A, B, "sum")
    monkeypatch.setenv("TCUDB_FORCE_HASHPART", "1")
    out, st = run(engine, torch_mod, A, B, "sum", 0)
    compare(out, ref, "sum")
    if case.startswith("c5s"):
        assert st["spa_mode"] == 4
    monkeypatch.setenv("TCUDB_FORCE_HASHPART", "0")
    monkeypatch.setenv("TCUDB_NO_HASHPART", "1")
    out2, _ = run(engine, torch_mod, A, B, "sum", 0)
    for k in ("g", "h", "agg"):
        assert np.array_equal(out[k], out2[k])


def test_abi_error_statuses(engine, torch_mod):
    """Argument errors come back as status codes (never partial results): exclusive FORCE
    flags -> E_INVALID; float keys, mixed int/float values, float chain values ->
    E_UNSUPPORTED; and the context stays usable afterwards."""
    torch = torch_mod
    from paper_2112_07552_b200._lib import TcudbError
    k = torch.arange(10, device="cuda", dtype=torch.int32)
    A = {"k": k, "g": k}
    with pytest.raises(TcudbError) as ei:
        engine.join_agg(A, A, "count", flags=1 | 2)
    assert ei.value.status == -1
    with pytest.raises(TcudbError) as ei:
        engine.join_agg({"k": k.float(), "g": k}, A, "count")
    assert ei.value.status == -2
    with pytest.raises(TcudbError) as ei:
        engine.join_agg(dict(A, v=k.float()), dict(A, v=k), "sum")
    assert ei.value.status == -2
    with pytest.raises(TcudbError) as ei:
        engine.chain_join_agg(dict(A, v=k.float()), A, A, "sum")
    assert ei.value.status == -2
    out = engine.join_agg(A, A, "count")
    assert out["agg"].sum().item() == 10


# ---------------------------------------------------------------- ranged bf16 fill (a5)
@pytest.mark.parametrize("passes", [None, "1", "3"])
@pytest.mark.parametrize("case", ["unique", "dup_nonzero", "dup_zero_after", "zero_values"])
def test_bf16_range_fill_duplicates(engine, torch_mod, oracle_mod, monkeypatch, passes, case):
    """The row-range direct fill trusts #nonzero cells == #nonzero-valued tuples: a duplicate
    (row, k) cell that loses a nonzero value must send the guard to the fp32-scratch path,
    zero-valued duplicates may not change a cell, so either way the result is the oracle's."""
    if passes is not None:
        monkeypatch.setenv("TCUDB_FILL_PASSES", passes)
    rng = np.random.default_rng(11)
    n = 96
    cells = rng.permutation(n * n)
    ag, ak = (cells // n).astype(np.int32), (cells % n).astype(np.int32)
    av = datagen._bf16_representable(rng.uniform(2.0 ** -8, 1.0, n * n).astype(np.float32))
    if case == "dup_nonzero":      # a second tuple in cell (ag[0], ak[0]) with another value
        ag, ak, av = np.append(ag, ag[0]), np.append(ak, ak[0]), np.append(av, np.float32(0.5))
    elif case == "dup_zero_after":  # ... with value 0, stored after the nonzero one
        ag, ak, av = np.append(ag, ag[0]), np.append(ak, ak[0]), np.append(av, np.float32(0.0))
    elif case == "zero_values":
        av[::7] = 0.0
    cells_b = rng.permutation(n * n)
    bk, bh = (cells_b // n).astype(np.int32), (cells_b % n).astype(np.int32)
    bw = datagen._bf16_representable(rng.uniform(2.0 ** -8, 1.0, n * n).astype(np.float32))
    A, B = datagen.Table(ak, ag, av), datagen.Table(bk, bh, bw)
    out, st = run(engine, torch_mod, A, B, "sum", flags=1)  # FORCE_DENSE: the fill under test
    assert st["path"] == 0
    compare(out, oracle_mod.join_agg(A, B, "sum"), "sum", float_vals=True)


def test_selector_calibration_measured(engine):
    """tcudb_create measured the selector's constants (A19) on this device: rates in the
    B200's range (the clamps allow 1/4..4x of the defaults; these bounds are tighter)."""
    c = engine.calibration
    assert c["measured"], c
    assert 1.0e15 < c["R_i8"] < 5.0e15 and 0.5e15 < c["R_bf16"] < 2.5e15 and 2.0e15 < c["R_fp4"] < 1.0e16, c
    assert 3.0e12 < c["BW"] < 9.0e12, c
    assert 1.25e10 <= c["R_sp"] <= 2.0e11 and 10e-6 <= c["T_sp0"] <= 400e-6, c
    assert 10e-6 <= c["T_d0"] <= 2e-3, c


@pytest.mark.parametrize("mode", ["tiled", "range", "binned"])
@pytest.mark.parametrize("case", ["unique", "dup_nonzero", "dup_zero_after", "zero_values", "inexact",
                                  "inexact_dup"])
def test_bf16_fill_modes_large(engine, torch_mod, oracle_mod, monkeypatch, mode, case):
    """The bf16 direct fills on >= 2^20 tuples (the tiled fill's size): 1024 x 1024 cells in
    shuffled order, ragged G (1000 rows), a duplicate cell (nonzero / zero second value),
    zero values, a non-bf16-exact value (-> fp32 scratch path). All equal the oracle."""
    monkeypatch.setenv("TCUDB_FILL_MODE", mode)
    rng = np.random.default_rng(12)
    n, m = 1000, 1088
    cells = rng.permutation(n * m)
    ag, ak = (cells // m).astype(np.int32), (cells % m).astype(np.int32)
    av = datagen._bf16_representable(rng.uniform(2.0 ** -8, 1.0, n * m).astype(np.float32))
    if case == "dup_nonzero":
        ag, ak, av = np.append(ag, ag[5]), np.append(ak, ak[5]), np.append(av, np.float32(0.5))
    elif case == "dup_zero_after":
        ag, ak, av = np.append(ag, ag[5]), np.append(ak, ak[5]), np.append(av, np.float32(0.0))
    elif case == "zero_values":
        av[::7] = 0.0
    elif case == "inexact":          # -> the tiled hi/lo split fill (unique cells)
        av[123] = np.float32(0.1)
    elif case == "inexact_dup":      # -> split fill sees the duplicate -> fp32 scratch path
        av[123] = np.float32(0.1)
        ag, ak, av = np.append(ag, ag[5]), np.append(ak, ak[5]), np.append(av, np.float32(0.3))
    bk = np.tile(np.arange(m, dtype=np.int32), 3)
    bh = np.repeat(np.arange(3, dtype=np.int32), m)
    bw = datagen._bf16_representable(rng.uniform(2.0 ** -8, 1.0, 3 * m).astype(np.float32))
    A, B = datagen.Table(ak, ag, av), datagen.Table(bk, bh, bw)
    out, st = run(engine, torch_mod, A, B, "sum", flags=1)
    assert st["path"] == 0
    compare(out, oracle_mod.join_agg(A, B, "sum"), "sum", float_vals=True)


@pytest.mark.parametrize("mode", ["atomic", "histscan"])
@pytest.mark.parametrize("name", ["c5", "c5s"])
def test_hash_partition_pass_modes(engine, torch_mod, oracle_mod, monkeypatch, mode, name):
    """Both partitioning schemes of the hash-partitioned path (one histogram + atomic run
    reservation, default; per-pass histogram + scan) against the oracle at 1/16 scale
    (1 M tuples per side: two radix passes, 1,024 partitions, the sampled selector)."""
    if mode == "histscan":
        monkeypatch.setenv("TCUDB_HASHPART_HISTSCAN", "1")
    monkeypatch.setenv("TCUDB_FORCE_HASHPART", "1")
    A, B, agg = datagen.make_config(name, 1 / 16)
    ref = oracle_mod.join_agg(A, B, agg)
    out, st = run(engine, torch_mod, A, B, agg, 0)
    assert st["spa_mode"] == 4
    compare(out, ref, agg)


# ---------------------------------------------------------------- a2 + a5 fused (fill_direct.cu)
@pytest.mark.parametrize("case", ["dense_exact", "holes", "signed_exact", "signed_split", "dup", "dup_split",
                                  "one_side_value", "ragged_kp", "shifted_keys", "negative_groups"])
@pytest.mark.parametrize("flags", [0, 1])
def test_fused_direct_fill(engine, torch_mod, oracle_mod, monkeypatch, case, flags):
    """Deferred per-tuple codes (the c4 class, TCUDB_LAZY_CODES=1 lifts the size threshold):
    the counting pass marks the direct dictionaries and counts per key, the fused fill looks
    the codes up itself (key_mode 2) — bf16 cells, the hi/lo split for non-bf16 values, the
    e2m1 existence pattern from the tiles' occupancy bits for signed values. Keys present on
    one side only (∩ domain), group values with gaps, duplicate cells (-> the codes are
    materialized and the scratch path runs), an absent value column, a K that is not a power
    of two. Auto flags may pick the sparse path (codes materialized). All equal the oracle."""
    monkeypatch.setenv("TCUDB_LAZY_CODES", "1")
    rng = np.random.default_rng(["dense_exact", "holes", "signed_exact", "signed_split", "dup", "dup_split",
                                 "one_side_value", "ragged_kp", "shifted_keys", "negative_groups"].index(case) + 40)
    G, K = 600, (1000 if case == "ragged_kp" else 1024)
    cells = rng.permutation(G * K)
    ag, ak = (cells // K).astype(np.int32), (cells % K).astype(np.int32)
    exact = datagen._bf16_representable(rng.uniform(2.0 ** -8, 1.0, G * K).astype(np.float32))
    av = exact
    if case == "holes":       # groups 3g + 7, keys only on even codes + 100 (B covers a shifted range)
        keep = ak % 2 == 0
        ag, ak, av = 3 * ag[keep] + 7, ak[keep] + 100, av[keep]
    elif case == "signed_exact":
        av = (rng.integers(-16, 17, G * K) / 8).astype(np.float32)
    elif case in ("signed_split", "dup_split"):
        av = rng.standard_normal(G * K).astype(np.float32)
    if case in ("dup", "dup_split"):
        ag, ak, av = np.append(ag, ag[7]), np.append(ak, ak[7]), np.append(av, av[3])
    H = 40
    bk = np.tile(np.arange(K, dtype=np.int32), H)
    bh = np.repeat(np.arange(H, dtype=np.int32) * 5, K).astype(np.int32)
    if case == "holes":
        bk = bk + 150
    bw = datagen._bf16_representable(rng.uniform(2.0 ** -8, 1.0, H * K).astype(np.float32))
    if case in ("signed_exact", "signed_split"):
        bw = -bw
    if case == "shifted_keys":
        ak, bk = ak + 50_000, bk + 50_000
    elif case == "negative_groups":
        ag, bh = ag - 5_000, bh - 70_000
    perm = rng.permutation(len(bk))
    A = datagen.Table(ak.astype(np.int32), ag.astype(np.int32), av)
    B = datagen.Table(bk[perm].astype(np.int32), bh[perm], None if case == "one_side_value" else bw[perm])
    ref = oracle_mod.join_agg(A, B, "sum")
    out, st = run(engine, torch_mod, A, B, "sum", flags)
    compare(out, ref, "sum", float_vals=True)
    if flags == 1:
        assert st["path"] == 0
        assert st["key_mode"] == (0 if case.startswith("dup") else 2), st["key_mode"]
        if case in ("signed_split",):
            assert st["elem"] == 2 and st["existence"] == 1


@pytest.mark.parametrize("case", ["complete", "rare_value_a", "rare_value_b"])
def test_hash_partitioned_sampled_group_dictionary(engine, torch_mod, oracle_mod, monkeypatch, case):
    """Small group domains over >= 2^22 tuples are built from a strided sample (every
    n/2^18-th value); every tuple is looked up afterwards and a value the sample missed sends
    the query to the general path. A value that occurs once, off the sample grid, on either
    side: the result still equals the oracle (and the hash-partitioned plan is not taken)."""
    rng = np.random.default_rng(77)
    n = 1 << 22
    pool_a, pool_b = datagen._pool(rng, 1500), datagen._pool(rng, 900)
    ga = pool_a[rng.integers(0, len(pool_a), n)]
    hb = pool_b[rng.integers(0, len(pool_b), n)]
    ka = datagen.scramble(rng.integers(0, 1 << 21, n, dtype=np.int64).astype(np.uint64))
    kb = datagen.scramble(rng.integers(0, 1 << 21, n, dtype=np.int64).astype(np.uint64))
    rare = np.int32(123456789)
    assert rare not in pool_a and rare not in pool_b
    if case == "rare_value_a":
        ga[12345] = rare   # 12345 is not a multiple of the sample step (16)
        kb[7] = ka[12345]  # ... and it joins
    elif case == "rare_value_b":
        hb[54321] = rare
        ka[9] = kb[54321]
    A, B = datagen.Table(ka, ga), datagen.Table(kb, hb)
    ref = oracle_mod.join_agg(A, B, "count")
    monkeypatch.setenv("TCUDB_FORCE_HASHPART", "1")
    out, st = run(engine, torch_mod, A, B, "count", 0)
    compare(out, ref, "count")
    if case == "complete":
        assert st["spa_mode"] == 4
    else:
        assert st["spa_mode"] != 4


# ---------------------------------------------------------------- asynchronous return
# Without stats tcudb_join_agg returns while the result write still runs on the stream
# (tcudb.h); the next query's scratch (the context's bump region) waits for the previous
# query's event. Results must be right when read in stream order, across streams once the
# reader's stream waits on the writer's, and for back-to-back queries on different streams.
@pytest.mark.parametrize("name,scale", [("c1", 1.0), ("c1s", 1.0), ("c2", 0.2), ("c3", 1 / 16), ("c4", 1 / 1024),
                                        ("c5", 1 / 64), ("c5s", 1 / 256)])
def test_no_stats_async_return(engine, torch_mod, oracle_mod, name, scale):
    A, B, agg = datagen.make_config(name, scale)
    ref = oracle_mod.join_agg(A, B, agg)
    out = engine.join_agg(to_dev(A, torch_mod), to_dev(B, torch_mod), agg)  # no stats: no final sync
    compare(res_np(out), ref, agg, float_vals=name.startswith("c4"))


def test_no_stats_back_to_back_streams(engine, torch_mod, oracle_mod):
    torch = torch_mod
    cases = [datagen.make_config("c2", 0.3), datagen.make_config("c1", 1.0), datagen.make_config("c5", 1 / 64),
             datagen.make_config("c1s", 1.0)]
    refs = [oracle_mod.join_agg(A, B, agg) for A, B, agg in cases]
    dev = [(to_dev(A, torch), to_dev(B, torch), agg) for A, B, agg in cases]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for rep in range(3):
        outs = []
        for i, (dA, dB, agg) in enumerate(dev):  # alternate streams, no host sync in between
            s = streams[i % 2]
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                outs.append(engine.join_agg(dA, dB, agg, stream=s))
        # read every result on the default stream after it waits on both writers
        cur = torch.cuda.current_stream()
        for s in streams:
            cur.wait_stream(s)
        for out, ref, (_, _, agg) in zip(outs, refs, dev):
            compare(res_np(out), ref, agg)
