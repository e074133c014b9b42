"""Seeded synthetic input generators for the five BASELINE.json configs.

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NO arithmetic of the method (no join, no aggregation, no encoding):
it only draws the input tables with the shapes, sizes and value distributions
stated in SURVEY.md §8(d) (recipe restated in DESIGN.md "Input recipe").

A table is a dict of numpy arrays: {"k": keys, "g": groups, "v": values or None}.
Both sides of a query use the same dict layout (B's group column is its "h").
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "Table", "c1_join_smoke", "c2_entity_matching", "c3_graph_edges", "c3_two_hop",
    "c4_matrix", "c5_low_density", "random_tiny", "make_config", "CONFIGS",
    "symmetrize_simple",
]


def Table(k, g, v=None):
    """Column-store table {"k", "g", "v"}; g None = the side is not grouped."""
    k = np.ascontiguousarray(k)
    if g is not None:
        g = np.ascontiguousarray(g)
        assert len(k) == len(g)
    if v is not None:
        v = np.ascontiguousarray(v)
        assert len(v) == len(k)
    return {"k": k, "g": g, "v": v}


def _pool(rng, n, dtype=np.int32):
    """n distinct random values of dtype (drawn without replacement)."""
    info = np.iinfo(dtype)
    out = np.unique(rng.integers(info.min, info.max, size=n * 2 + 16, dtype=np.int64))
    while len(out) < n:
        out = np.unique(np.concatenate([out, rng.integers(info.min, info.max, size=n, dtype=np.int64)]))
    out = rng.permutation(out)[:n]
    return out.astype(dtype)


# --------------------------------------------------------------------------- c1
def c1_join_smoke(agg="count", seed=1, n=1000, n_keys=64, n_groups=32):
    """Config 1: two 1,000-row tables, k uniform over 64 distinct random int32
    values, A.g / B.h over 32 random int32 values each.
    SUM variant: v, w ~ U{-100..100} int32."""
    rng = np.random.default_rng(seed)
    keys = _pool(rng, n_keys)
    ga = _pool(rng, n_groups)
    hb = _pool(rng, n_groups)
    A = Table(keys[rng.integers(0, n_keys, n)], ga[rng.integers(0, n_groups, n)],
              rng.integers(-100, 101, n).astype(np.int32) if agg == "sum" else None)
    B = Table(keys[rng.integers(0, n_keys, n)], hb[rng.integers(0, n_groups, n)],
              rng.integers(-100, 101, n).astype(np.int32) if agg == "sum" else None)
    return A, B


# --------------------------------------------------------------------------- c2
def _zipf_sampler(vocab, s, rng):
    w = 1.0 / np.arange(1, vocab + 1, dtype=np.float64) ** s
    cdf = np.cumsum(w)
    cdf /= cdf[-1]

    def draw(size):
        return np.minimum(np.searchsorted(cdf, rng.random(size), side="right"), vocab - 1)
    return draw


def _token_bags(rng, n_records, vocab, lmin, lmax, s):
    draw = _zipf_sampler(vocab, s, rng)
    lens = rng.integers(lmin, lmax + 1, n_records)
    rids, toks = [], []
    for r in range(n_records):
        L = int(lens[r])
        got = np.empty(0, dtype=np.int64)
        while len(got) < L:  # tokens are distinct within a record (token SETS)
            cand = draw(2 * L)
            got = np.concatenate([got, cand])
            _, first = np.unique(got, return_index=True)
            got = got[np.sort(first)]
        rids.append(np.full(L, r, dtype=np.int32))
        toks.append(got[:L].astype(np.int32))
    return np.concatenate(rids), np.concatenate(toks)


def c2_entity_matching(n_records=10_000, vocab=32_768, lmin=10, lmax=30, s=1.0, seeds=(2, 3)):
    """Config 2: token-bag entity matching. Records of L~U{10..30} distinct
    tokens, Zipf(s=1) over a 32,768 vocabulary (inverse CDF). Tables are
    (rid, tok); k = tok, g = A.rid, h = B.rid; COUNT(*) = shared tokens."""
    ra, ta = _token_bags(np.random.default_rng(seeds[0]), n_records, vocab, lmin, lmax, s)
    rb, tb = _token_bags(np.random.default_rng(seeds[1]), n_records, vocab, lmin, lmax, s)
    return Table(ta, ra), Table(tb, rb)


def c2_blocked(n_records=10_000, n_blocks=100, block_vocab=400, lmin=100, lmax=200, seeds=(21, 22)):
    """Blocked entity matching (the paper's EM blocking, as a block-structured
    input for the §8(f) f4 block-sparse path; not one of BASELINE's five configs): records
    numbered block by block (a table sorted by its blocking key), n_blocks blocks, each
    record a set of L ~ U{lmin..lmax} distinct tokens drawn uniformly from its block's own
    vocabulary of block_vocab tokens; token ids are a random permutation of the whole
    vocabulary (so the block structure is invisible in key order). k = tok, g / h = rid,
    COUNT(*) = shared tokens; pairs only inside blocks."""
    V = n_blocks * block_vocab
    perm = np.random.default_rng(seeds[0] * 7 + 1).permutation(V).astype(np.int32)

    def side(seed):
        rng = np.random.default_rng(seed)
        lens = rng.integers(lmin, lmax + 1, n_records)
        block = (np.arange(n_records) * n_blocks) // n_records
        order = np.argsort(rng.random((n_records, block_vocab)), axis=1)[:, :lmax]
        keep = np.arange(lmax)[None, :] < lens[:, None]
        local = order[keep]
        rid = np.repeat(np.arange(n_records, dtype=np.int32), lens)
        tok = perm[np.repeat(block, lens) * block_vocab + local]
        return Table(tok.astype(np.int32), rid)
    return side(seeds[0]), side(seeds[1])


# --------------------------------------------------------------------------- c3
def c3_graph_edges(scale=16, edge_factor=16, abcd=(0.57, 0.19, 0.19, 0.05), seed=4):
    """R-MAT edge list (Chakrabarti et al.): scale 16 (65,536 ids), edge factor
    16, (a,b,c,d) = (0.57,0.19,0.19,0.05); random vertex-id permutation;
    self-loops and duplicate directed edges dropped. Returns (src, dst) int32."""
    rng = np.random.default_rng(seed)
    n_edges = edge_factor << scale
    a, b, c, _ = abcd
    src = np.zeros(n_edges, dtype=np.int64)
    dst = np.zeros(n_edges, dtype=np.int64)
    for bit in range(scale):
        r = rng.random(n_edges)
        s_bit = r >= a + b                   # quadrants c, d -> src bit set
        d_bit = ((r >= a) & (r < a + b)) | (r >= a + b + c)  # quadrants b, d -> dst bit set
        src |= s_bit.astype(np.int64) << bit
        dst |= d_bit.astype(np.int64) << bit
    perm = rng.permutation(1 << scale)
    src, dst = perm[src], perm[dst]
    keep = src != dst
    e = np.unique(np.stack([src[keep], dst[keep]], 1), axis=0)
    e = e[rng.permutation(len(e))]
    return e[:, 0].astype(np.int32), e[:, 1].astype(np.int32)


def c3_two_hop(src, dst):
    """2-hop path count as a self-join: A = B = E; A.k = dst, A.g = src;
    B.k = src, B.h = dst; COUNT(*) per (src, dst2)."""
    return Table(dst, src), Table(src, dst)


def symmetrize_simple(src, dst):
    """Simple undirected graph stored in both directions (no self-loops, no
    duplicates) — the reading of SURVEY §8(c) #15 for triangle counting."""
    s = np.asarray(src, dtype=np.int64)
    d = np.asarray(dst, dtype=np.int64)
    keep = s != d
    s, d = s[keep], d[keep]
    lo, hi = np.minimum(s, d), np.maximum(s, d)
    und = np.unique(np.stack([lo, hi], 1), axis=0)
    both = np.concatenate([und, und[:, ::-1]], 0)
    return both[:, 0].astype(np.int32), both[:, 1].astype(np.int32)


# --------------------------------------------------------------------------- c4
def _bf16_representable(x):
    """Round fp32 values to the nearest bf16-representable fp32 (input shaping)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32)


def c4_matrix(n=8192, seed=5, signed=False):
    """Config 4: SQL matmul. A(i,k,v) holds every (i,k) in [0,n)^2 in shuffled
    row order; B(k,j,w) likewise. Values bf16-representable from U[2^-8, 1)
    stored as fp32 (variant c4s: signed N(0,1), not bf16-exact).
    As join tables: A.k = k, A.g = i, A.v = v; B.k = k, B.g(h) = j, B.v = w."""
    rng = np.random.default_rng(seed)

    def one():
        cells = rng.permutation(n * n).astype(np.int64)
        row = (cells // n).astype(np.int32)
        col = (cells % n).astype(np.int32)
        if signed:
            val = rng.standard_normal(n * n, dtype=np.float32)
        else:
            val = _bf16_representable(rng.uniform(2.0 ** -8, 1.0, n * n).astype(np.float32))
        return row, col, val
    ai, ak, av = one()          # A rows are (i, k, v)
    bk, bj, bw = one()          # B rows are (k, j, w)
    return Table(ak, ai, av), Table(bk, bj, bw)


# --------------------------------------------------------------------------- c5
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def scramble(x):
    """scramble(x) = x * 0x9E3779B97F4A7C15 mod 2^64, viewed as int64."""
    with np.errstate(over="ignore"):
        return (np.asarray(x, dtype=np.uint64) * _GOLDEN).view(np.int64)


def c5_low_density(n=1 << 24, key_domain=1 << 22, n_groups=4096, agg="count", seed=6):
    """Config 5: 2^24-row tables, k = scramble(U{0..2^22-1}) int64, g/h uniform
    over 4,096 random int32 values, v/w ~ U{-100..100} int32 (SUM variant)."""
    rng = np.random.default_rng(seed)
    ga = _pool(rng, n_groups)
    hb = _pool(rng, n_groups)
    ka = scramble(rng.integers(0, key_domain, n, dtype=np.int64).astype(np.uint64))
    kb = scramble(rng.integers(0, key_domain, n, dtype=np.int64).astype(np.uint64))
    A = Table(ka, ga[rng.integers(0, n_groups, n)],
              rng.integers(-100, 101, n).astype(np.int32) if agg == "sum" else None)
    B = Table(kb, hb[rng.integers(0, n_groups, n)],
              rng.integers(-100, 101, n).astype(np.int32) if agg == "sum" else None)
    return A, B


# --------------------------------------------------------------------------- tiny
def random_tiny(rng, n_max=64, k_max=16, g_max=8, vkind="none", vmin=-5, vmax=5,
                key_dtype=np.int64, allow_empty=True):
    """Random tiny instance for nested-loop cross-checks: duplicates, negatives,
    empty and disjoint key sets all occur with non-trivial probability."""
    lo = 0 if allow_empty else 1
    na, nb = int(rng.integers(lo, n_max + 1)), int(rng.integers(lo, n_max + 1))
    nk = int(rng.integers(1, k_max + 1))
    off = int(rng.integers(-3, 3)) * nk if rng.random() < 0.2 else 0  # sometimes disjoint-ish
    ka = rng.integers(0, nk, na) * 7 - 11
    kb = rng.integers(0, nk, nb) * 7 - 11 + off * 7
    ga = rng.integers(-g_max, g_max, na) * 3
    hb = rng.integers(-g_max, g_max, nb) * 5

    def vals(m):
        if vkind == "none":
            return None
        if vkind == "int":
            return rng.integers(vmin, vmax + 1, m).astype(np.int64)
        if vkind == "float":
            return rng.uniform(vmin, vmax, m).astype(np.float32)
        raise ValueError(vkind)
    return (Table(ka.astype(key_dtype), ga.astype(np.int64), vals(na)),
            Table(kb.astype(key_dtype), hb.astype(np.int64), vals(nb)))


# --------------------------------------------------------------------------- placement
def local_slice(T, ws, rank):
    """Contiguous 1/ws slice of a host table (numpy columns): rank r's starting data in
    the multi-GPU runs."""
    n = len(T["k"])
    lo, hi = n * rank // ws, n * (rank + 1) // ws
    return {k: (None if v is None else np.ascontiguousarray(v[lo:hi])) for k, v in T.items()}


# --------------------------------------------------------------------------- registry
CONFIGS = {
    "c1": "COUNT(*) natural join of two 1,000-row int tables on 64 distinct keys, 32x32 groups",
    "c1s": "c1 with SUM(A.v*B.w), v,w ~ U{-100..100}",
    "c2": "entity matching: 10k x 10k token-bag records, vocab 32k, shared-token COUNT",
    "c2b": "blocked entity matching (f4 block-sparse input): 100 blocks x 100 records, 400-token block vocabularies",
    "c3": "graph query: 2-hop path count on R-MAT scale-16 edge table (self-join + group-by)",
    "c4": "matrix analytics: SQL matmul of two 8192x8192 (row,col,val) tables, SUM bf16",
    "c4s": "c4 with signed fp32 N(0,1) values (not bf16-exact: the guard's hi/lo split)",
    "c5": "low-density join: 16M x 16M tuples over 4M-key domain, COUNT",
    "c5s": "c5 with SUM(A.v*B.w), v,w ~ U{-100..100}",
}


def make_config(name, scale=1.0):
    """Return (A, B, agg) for a named config. `scale` < 1 shrinks c4/c5 for
    parity tests (same distribution, fewer rows)."""
    if name == "c1":
        A, B = c1_join_smoke("count"); return A, B, "count"
    if name == "c1s":
        A, B = c1_join_smoke("sum"); return A, B, "sum"
    if name == "c2":
        n = max(16, int(10_000 * scale))
        A, B = c2_entity_matching(n_records=n); return A, B, "count"
    if name == "c2b":
        n = max(100, int(10_000 * scale))
        A, B = c2_blocked(n_records=n, n_blocks=max(1, n // 100)); return A, B, "count"
    if name == "c3":
        sc = 16 if scale >= 1.0 else max(6, int(round(16 + np.log2(scale))))
        s, d = c3_graph_edges(scale=sc)
        A, B = c3_two_hop(s, d); return A, B, "count"
    if name in ("c4", "c4s"):
        n = 8192 if scale >= 1.0 else max(16, int(8192 * np.sqrt(scale)))
        A, B = c4_matrix(n=n, signed=name == "c4s"); return A, B, "sum"
    if name in ("c5", "c5s"):
        n = int((1 << 24) * scale)
        kd = max(16, int((1 << 22) * scale))
        agg = "sum" if name == "c5s" else "count"
        A, B = c5_low_density(n=n, key_domain=kd, agg=agg); return A, B, agg
    raise KeyError(name)
