"""Pins for the CPU oracle (runs with -m "not gpu").

The oracle (oracle/oracle.cpp, hash join + hash aggregation) and the
pure-Python nested loop are each pinned to things other than themselves:
  * worked examples printed in SPEC.md / PAPER.md (tests/golden/*.json);
  * closed forms: COUNT total = sum_k cntA(k)*cntB(k) (follows PAPER.md §3.1
    P:683-685); SUM total = sum_k SA(k)*SB(k) (Q4); the Q3 marginal
    sum_g SUM(g,h) from an independent 1-D aggregation;
  * special cases reducing to a library routine: per-group COUNT/SUM equals
    numpy's integer matmul of the dense (g x k)/(h x k) cell matrices
    (adjacency form) on small inputs;
  * textbook graph counts for triangles (K_n, C_n, W_n, Petersen, K_{3,3},
    friendship graphs) and 2-hop counts (K_n, directed path, star);
  * invariants: permutation invariance, A (+) A doubles, swapping A/B transposes.
A plausible mistake (a dropped term, a wrong sign/index, transposed operands,
dropping zero-SUM groups, wrapping on overflow) fails at least one of these.
"""
import glob
import itertools
import json
import math
import os

import numpy as np
import pytest

import datagen

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "spec_*.json")))


def _table(d):
    v = None if d["v"] is None else np.array(d["v"], dtype=np.int64)
    return datagen.Table(np.array(d["k"], dtype=np.int64), np.array(d["g"], dtype=np.int64), v)


def _triples(res, agg):
    col = res["cnt"] if agg == "count" else res["sum"]
    return [[int(a), int(b), int(c)] for a, b, c in zip(res["g"], res["h"], col)]


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_golden_examples(oracle_mod, path):
    fx = json.load(open(path))
    A, B = _table(fx["A"]), _table(fx["B"])
    assert fx["cite"]
    assert _triples(oracle_mod.join_agg(A, B, fx["agg"]), fx["agg"]) == fx["expect"]
    assert _triples(oracle_mod.nested_loop(A, B, fx["agg"]), fx["agg"]) == fx["expect"]


def _same(r1, r2, agg, float_tol=None):
    assert np.array_equal(r1["g"], r2["g"])
    assert np.array_equal(r1["h"], r2["h"])
    assert np.array_equal(r1["cnt"], r2["cnt"])
    if agg == "sum":
        if float_tol is None:
            assert np.array_equal(r1["sum"], r2["sum"])
        else:
            err = np.abs(r1["sum"] - r2["sum"])
            assert np.all(err <= float_tol * np.maximum(r2["abs"], 1e-300))
            assert np.allclose(r1["abs"], r2["abs"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("vkind", ["none", "int", "float"])
def test_hash_oracle_equals_nested_loop(oracle_mod, vkind):
    rng = np.random.default_rng(2112)
    agg = "count" if vkind == "none" else "sum"
    for _ in range(300):
        A, B = datagen.random_tiny(rng, vkind=vkind, vmin=-9, vmax=9)
        _same(oracle_mod.join_agg(A, B, agg), oracle_mod.nested_loop(A, B, agg), agg,
              float_tol=1e-12 if vkind == "float" else None)


def _cells(T, kdict, gdict, use_value):
    """Dense |gdict| x |kdict| cell matrix (python ints) of a table."""
    M = np.zeros((len(gdict), len(kdict)), dtype=object)
    gi = {x: i for i, x in enumerate(gdict)}
    ki = {x: i for i, x in enumerate(kdict)}
    vals = T["v"] if use_value and T["v"] is not None else [1] * len(T["k"])
    for k, g, v in zip(T["k"], T["g"], vals):
        M[gi[int(g)], ki[int(k)]] += int(v)
    return M


@pytest.mark.parametrize("agg", ["count", "sum"])
def test_per_group_equals_dense_matmul(oracle_mod, agg):
    """Adjacency form: C = A_op . B_op^T over the union
    key domain; entry (g,h) is the aggregate, existence = pattern product > 0."""
    rng = np.random.default_rng(7)
    for _ in range(40):
        A, B = datagen.random_tiny(rng, n_max=80, vkind="int" if agg == "sum" else "none")
        kd = sorted(set(map(int, A["k"])) | set(map(int, B["k"])))
        gd, hd = sorted(set(map(int, A["g"]))), sorted(set(map(int, B["g"])))
        C = _cells(A, kd, gd, agg == "sum").dot(_cells(B, kd, hd, agg == "sum").T) if gd and hd and kd else None
        P = _cells(A, kd, gd, False).dot(_cells(B, kd, hd, False).T) if gd and hd and kd else None
        res = oracle_mod.join_agg(A, B, agg)
        expect = []
        if C is not None:
            for i, g in enumerate(gd):
                for j, h in enumerate(hd):
                    if P[i, j] > 0:
                        expect.append([g, h, int(C[i, j] if agg == "sum" else P[i, j])])
        assert _triples(res, agg) == expect


def _key_counts(T):
    u, c = np.unique(np.asarray(T["k"], dtype=np.int64), return_counts=True)
    return dict(zip(u.tolist(), c.tolist()))


@pytest.mark.parametrize("cfg", ["c1", "c1s", "random"])
def test_count_total_closed_form(oracle_mod, cfg):
    """sum_(g,h) COUNT = sum_k cntA(k)*cntB(k) (north star)."""
    if cfg == "random":
        rng = np.random.default_rng(11)
        A = datagen.Table(rng.integers(0, 300, 20000), rng.integers(0, 50, 20000))
        B = datagen.Table(rng.integers(0, 300, 15000), rng.integers(0, 70, 15000))
    else:
        A, B, _ = datagen.make_config(cfg)
    res = oracle_mod.join_agg(A, B, "count")
    ca, cb = _key_counts(A), _key_counts(B)
    J = sum(ca[k] * cb.get(k, 0) for k in ca)
    assert int(res["cnt"].sum()) == J
    assert np.all(res["cnt"] >= 1)


def test_sum_total_q4_and_marginal_q3(oracle_mod):
    """Q4: sum of all SUMs = sum_k SA(k)*SB(k). Q3: for every h,
    sum_g SUM(g,h) = sum_{b: b.h=h} w_b * SA(b.k)."""
    rng = np.random.default_rng(5)
    A = datagen.Table(rng.integers(0, 500, 30000), rng.integers(0, 40, 30000), rng.integers(-100, 101, 30000))
    B = datagen.Table(rng.integers(0, 500, 25000), rng.integers(0, 60, 25000), rng.integers(-100, 101, 25000))
    res = oracle_mod.join_agg(A, B, "sum")
    SA, SB = {}, {}
    for k, v in zip(A["k"].tolist(), A["v"].tolist()):
        SA[k] = SA.get(k, 0) + v
    for k, w in zip(B["k"].tolist(), B["v"].tolist()):
        SB[k] = SB.get(k, 0) + w
    assert int(res["sum"].sum()) == sum(SA[k] * SB.get(k, 0) for k in SA)
    per_h = {}
    for k, h, w in zip(B["k"].tolist(), B["g"].tolist(), B["v"].tolist()):
        per_h[h] = per_h.get(h, 0) + w * SA.get(k, 0)
    got = {}
    for h, s in zip(res["h"].tolist(), res["sum"].tolist()):
        got[h] = got.get(h, 0) + s
    for h, s in per_h.items():
        assert got.get(h, 0) == s


def test_float_sum_all_ones_and_tolerance(oracle_mod):
    """All-ones float tables: every SUM equals its COUNT exactly ({0,1}
    inputs give MAPE 0); random floats agree with math.fsum brute force."""
    rng = np.random.default_rng(3)
    A = datagen.Table(rng.integers(0, 30, 3000), rng.integers(0, 20, 3000), np.ones(3000, np.float32))
    B = datagen.Table(rng.integers(0, 30, 2000), rng.integers(0, 20, 2000), np.ones(2000, np.float32))
    res = oracle_mod.join_agg(A, B, "sum")
    assert np.array_equal(res["sum"], res["cnt"].astype(np.float64))
    assert np.array_equal(res["abs"], res["cnt"].astype(np.float64))


def test_zero_sum_groups_and_signs(oracle_mod):
    rng = np.random.default_rng(17)
    zero_groups = 0
    for _ in range(200):
        A, B = datagen.random_tiny(rng, vkind="int", vmin=-2, vmax=2)
        r = oracle_mod.join_agg(A, B, "sum")
        zero_groups += int(np.sum(r["sum"] == 0))
        assert np.all(r["cnt"] >= 1)
    assert zero_groups > 0   # the generator does exercise COUNT>0, SUM=0 groups


def test_overflow_is_reported_not_wrapped(oracle_mod):
    big = 2**62
    A = datagen.Table(np.zeros(4, np.int64), np.zeros(4, np.int64), np.full(4, big, np.int64))
    B = datagen.Table(np.zeros(1, np.int64), np.zeros(1, np.int64), np.full(1, 2, np.int64))
    with pytest.raises(oracle_mod.OracleOverflow):
        oracle_mod.join_agg(A, B, "sum")
    with pytest.raises(oracle_mod.OracleOverflow):
        oracle_mod.nested_loop(A, B, "sum")
    # the intermediate product leaves int64 but the sum returns into range
    A2 = datagen.Table(np.zeros(2, np.int64), np.zeros(2, np.int64), np.array([big, -big], np.int64))
    B2 = datagen.Table(np.zeros(1, np.int64), np.zeros(1, np.int64), np.array([4], np.int64))
    assert oracle_mod.join_agg(A2, B2, "sum")["sum"].tolist() == [0]


def test_invariants_permutation_duplication_swap(oracle_mod):
    rng = np.random.default_rng(23)
    n = 4000
    A = datagen.Table(rng.integers(0, 200, n), rng.integers(0, 30, n), rng.integers(-50, 51, n))
    B = datagen.Table(rng.integers(0, 200, n), rng.integers(0, 40, n), rng.integers(-50, 51, n))
    base = oracle_mod.join_agg(A, B, "sum")
    p = rng.permutation(n)
    Ap = datagen.Table(A["k"][p], A["g"][p], A["v"][p])
    _same(oracle_mod.join_agg(Ap, B, "sum"), base, "sum")
    AA = datagen.Table(np.concatenate([A["k"]] * 2), np.concatenate([A["g"]] * 2), np.concatenate([A["v"]] * 2))
    dbl = oracle_mod.join_agg(AA, B, "sum")
    assert np.array_equal(dbl["cnt"], 2 * base["cnt"]) and np.array_equal(dbl["sum"], 2 * base["sum"])
    sw = oracle_mod.join_agg(B, A, "sum")
    o = np.lexsort((sw["g"], sw["h"]))
    assert np.array_equal(sw["h"][o], base["g"]) and np.array_equal(sw["g"][o], base["h"])
    assert np.array_equal(sw["sum"][o], base["sum"]) and np.array_equal(sw["cnt"][o], base["cnt"])


# ------------------------------------------------------------------ graph pins
def _complete(n):
    return [(i, j) for i in range(n) for j in range(n) if i != j]


def _cycle(n):
    return [(i, (i + 1) % n) for i in range(n)]


def _wheel(n):      # hub n, rim 0..n-1
    return _cycle(n) + [(n, i) for i in range(n)]


def _petersen():
    outer = [(i, (i + 1) % 5) for i in range(5)]
    spokes = [(i, i + 5) for i in range(5)]
    inner = [(5 + i, 5 + (i + 2) % 5) for i in range(5)]
    return outer + spokes + inner


def _friendship(k):  # k triangles sharing vertex 0
    e = []
    for t in range(k):
        a, b = 1 + 2 * t, 2 + 2 * t
        e += [(0, a), (0, b), (a, b)]
    return e


def _tri(oracle_mod, edges):
    s, d = zip(*edges)
    return oracle_mod.triangles(np.array(s), np.array(d))


def test_triangle_textbook_counts(oracle_mod):
    for n in range(3, 11):
        assert _tri(oracle_mod, _complete(n)) == math.comb(n, 3)
    assert _tri(oracle_mod, _complete(4)) == 4 and _tri(oracle_mod, _complete(10)) == 120
    assert _tri(oracle_mod, _cycle(3)) == 1
    for n in range(4, 12):
        assert _tri(oracle_mod, _cycle(n)) == 0
        assert _tri(oracle_mod, _wheel(n)) == n
    assert _tri(oracle_mod, _petersen()) == 0
    assert _tri(oracle_mod, [(a, b) for a in range(3) for b in range(3, 6)]) == 0   # K_{3,3}
    for k in range(1, 7):
        assert _tri(oracle_mod, _friendship(k)) == k
    # self-loops, duplicates and reversed copies do not change a simple-graph count
    e = _wheel(6)
    assert _tri(oracle_mod, e + [(b, a) for a, b in e] + [(1, 1), (2, 2)] + e[:3]) == 6


def test_triangles_brute_force_and_trace(oracle_mod):
    rng = np.random.default_rng(9)
    for _ in range(20):
        n = int(rng.integers(4, 25))
        m = int(rng.integers(0, n * 3))
        s, d = rng.integers(0, n, m), rng.integers(0, n, m)
        adj = np.zeros((n, n), dtype=np.int64)
        for a, b in zip(s, d):
            if a != b:
                adj[a, b] = adj[b, a] = 1
        brute = sum(1 for i, j, k in itertools.combinations(range(n), 3) if adj[i, j] and adj[j, k] and adj[i, k])
        assert oracle_mod.triangles(s, d) == brute
        assert np.trace(adj @ adj @ adj) == 6 * brute


def _two_hop(oracle_mod, edges):
    s, d = (np.array(x) for x in zip(*edges))
    A, B = datagen.c3_two_hop(s, d)
    return oracle_mod.join_agg(A, B, "count")


def test_two_hop_closed_forms(oracle_mod):
    for n in (3, 4, 6, 9):       # K_n: (J-I)^2 -> diag n-1, off-diag n-2
        r = _two_hop(oracle_mod, _complete(n))
        diag = r["g"] == r["h"]
        assert np.all(r["cnt"][diag] == n - 1) and np.all(r["cnt"][~diag] == n - 2)
        assert len(r["g"]) == (n * n if n > 2 else n)
    for n in (3, 5, 10):         # directed path 0->1->...->n-1
        r = _two_hop(oracle_mod, [(i, i + 1) for i in range(n - 1)])
        assert len(r["g"]) == n - 2 and np.all(r["cnt"] == 1) and np.all(r["h"] - r["g"] == 2)
    r = _two_hop(oracle_mod, [(0, i) for i in range(1, 8)])    # star center -> leaves
    assert len(r["g"]) == 0


def test_generators_shapes():
    """Generator sanity (sizes / distributions, not the method): c1 tables."""
    A, B = datagen.c1_join_smoke()
    assert len(A["k"]) == len(B["k"]) == 1000
    assert len(np.unique(np.concatenate([A["k"], B["k"]]))) <= 64
    assert len(np.unique(A["g"])) == 32 and len(np.unique(B["g"])) == 32
    s, d = datagen.c3_graph_edges(scale=10, edge_factor=8)
    assert np.all(s != d) and len(np.unique(np.stack([s, d], 1), axis=0)) == len(s)
    k = datagen.scramble(np.arange(10, dtype=np.uint64))
    assert len(np.unique(k)) == 10 and k.dtype == np.int64


# ---------------------------------------------------------------- §8(f) f2: AVG, Q3, Q4
def _drop_g(T):
    return {"k": T["k"], "g": None, "v": T["v"]}


@pytest.mark.parametrize("vkind", ["none", "int", "float"])
@pytest.mark.parametrize("shape", ["gh", "h_only", "g_only", "none"])
def test_avg_and_ungrouped_vs_nested_loop(oracle_mod, vkind, shape):
    """AVG (= SUM / COUNT) and ungrouped sides (Q3 P:785-823, Q4 P:842-850):
    the hash oracle equals the pure-Python nested loop (exact rational mean for
    integers, math.fsum of exact products for floats) on random tiny instances."""
    rng = np.random.default_rng({"none": 1, "int": 2, "float": 3}[vkind] * 10 + len(shape))
    for _ in range(120):
        A, B = datagen.random_tiny(rng, vkind=vkind)
        if shape in ("h_only", "none"):
            A = _drop_g(A)
        if shape in ("g_only", "none"):
            B = _drop_g(B)
        for agg in ("count", "sum", "avg"):
            got = oracle_mod.join_agg(A, B, agg)
            ref = oracle_mod.nested_loop(A, B, agg)
            assert set(got) == set(ref)
            for col in ("g", "h", "cnt"):
                if col in ref:
                    assert np.array_equal(got[col], ref[col])
            if agg != "count":
                if vkind == "float":
                    assert np.allclose(got["sum"], ref["sum"], rtol=1e-12, atol=1e-9)
                else:
                    assert np.array_equal(got["sum"], ref["sum"])
            if agg == "avg":
                if vkind == "float":
                    assert np.allclose(got["avg"], ref["avg"], rtol=1e-12, atol=1e-9)
                else:
                    assert np.array_equal(got["avg"], ref["avg"])


def test_q3_q4_spec_examples_ungrouped(oracle_mod):
    """SPEC S:514 (Q3: GROUP BY B.Val only -> g1: 30) and S:515 (Q4: no GROUP BY -> 6)
    with the constant group columns of the golden fixtures replaced by absent ones."""
    A = {"k": np.array([1, 2]), "g": None, "v": np.array([10, 20])}
    B = {"k": np.array([1, 2]), "g": np.array([1, 1]), "v": None}
    r = oracle_mod.join_agg(A, B, "sum")
    assert "g" not in r and r["h"].tolist() == [1] and r["sum"].tolist() == [30]
    A = {"k": np.array([7]), "g": None, "v": np.array([2])}
    B = {"k": np.array([7]), "g": None, "v": np.array([3])}
    r = oracle_mod.join_agg(A, B, "sum")
    assert "g" not in r and "h" not in r and r["sum"].tolist() == [6] and r["cnt"].tolist() == [1]
    assert oracle_mod.join_agg(A, B, "avg")["avg"].tolist() == [6.0]


def test_ungrouped_closed_forms(oracle_mod):
    """Q3 with A ungrouped: SUM(h) = sum_{b.h=h} w_b * SA(b.k) and COUNT(h) =
    sum_{b.h=h} cntA(b.k); Q4: SUM = sum_k SA(k) * SB(k), COUNT = J — computed here
    with independent per-key dictionaries (the 1^{1xn} x mat(A) reduction)."""
    rng = np.random.default_rng(21)
    A = datagen.Table(rng.integers(0, 400, 20000), None, rng.integers(-50, 51, 20000))
    B = datagen.Table(rng.integers(0, 400, 15000), rng.integers(0, 90, 15000), rng.integers(-50, 51, 15000))
    SA, CA = {}, {}
    for k, v in zip(A["k"].tolist(), A["v"].tolist()):
        SA[k] = SA.get(k, 0) + v
        CA[k] = CA.get(k, 0) + 1
    per_h, cnt_h = {}, {}
    for k, h, w in zip(B["k"].tolist(), B["g"].tolist(), B["v"].tolist()):
        if k in CA:
            per_h[h] = per_h.get(h, 0) + w * SA[k]
            cnt_h[h] = cnt_h.get(h, 0) + CA[k]
    r = oracle_mod.join_agg(A, B, "sum")
    assert r["h"].tolist() == sorted(per_h)
    assert r["sum"].tolist() == [per_h[h] for h in sorted(per_h)]
    assert r["cnt"].tolist() == [cnt_h[h] for h in sorted(per_h)]
    SB = {}
    for k, w in zip(B["k"].tolist(), B["v"].tolist()):
        SB[k] = SB.get(k, 0) + w
    q4 = oracle_mod.join_agg(A, _drop_g(B), "sum")
    assert q4["sum"].tolist() == [sum(SA[k] * SB.get(k, 0) for k in SA)]


# ---------------------------------------------------------------- §8(f) f3: chain joins
def test_chain_join_vs_triple_loop(oracle_mod):
    """The chain oracle (join order A -> B -> C with the nonzero() re-encoding)
    equals a brute-force loop over all triples (COUNT and integer SUM, duplicates,
    negatives, empty and disjoint inputs)."""
    rng = np.random.default_rng(31)
    for _ in range(150):
        A, B = datagen.random_tiny(rng, n_max=24, k_max=8, g_max=4, vkind="int", vmin=-4, vmax=4)
        C, _ = datagen.random_tiny(rng, n_max=24, k_max=8, g_max=4, vkind="int", vmin=-4, vmax=4)
        # B's second attribute joins C's key: draw it from C's key values (and some misses)
        B = dict(B, g=rng.choice(np.concatenate([C["k"], [999]]), len(B["k"])) if len(C["k"]) else B["g"])
        for agg in ("count", "sum"):
            got = oracle_mod.chain_join_agg(A, B, C, agg)
            ref = oracle_mod.chain_nested_loop(A, B, C, agg)
            assert np.array_equal(got["g"], ref["g"]) and np.array_equal(got["h"], ref["h"])
            assert np.array_equal(got["sum"], ref["sum"])


def test_chain_three_hop_complete_graph(oracle_mod):
    """3-hop walks on K_n: A^3 = (n^2 - 3n + 3) off the diagonal, (n-1)(n-2) on it
    (A = J - I, A^2 = (n-2)A + (n-1)I)."""
    n = 9
    src, dst = zip(*[(i, j) for i in range(n) for j in range(n) if i != j])
    src, dst = np.array(src), np.array(dst)
    E1 = datagen.Table(dst, src)   # A: k = dst (the walk's next vertex), g = src
    E2 = datagen.Table(src, dst)   # B: k = src, ID_2 = dst
    E3 = datagen.Table(src, dst)   # C: k = src, h = dst
    r = oracle_mod.chain_join_agg(E1, E2, E3, "count")
    for g, h, c in zip(r["g"], r["h"], r["sum"]):
        assert c == ((n - 1) * (n - 2) if g == h else n * n - 3 * n + 3)
    assert len(r["g"]) == n * n
