"""§8(f) f4: the block-sparse tensor-core path (csrc/blocksparse.cu + gemm_tc.cu's
K-block skipping), the B200 form of the paper's TCU-SpMM zero-tile skipping
(§4.2.4). Forced on every dense plan (e2m1 / u8 COUNT, digit-plane
int SUM, existence pattern planes, bf16 direct and hi/lo split, K chunks) it must give
the oracle's result; on block-structured input (c2b) the selector takes it by itself.
"""
import numpy as np
import pytest

import datagen
from parity_util import compare, res_np, to_dev

pytestmark = pytest.mark.gpu

FORCE_DENSE, FORCE_WIDE, NO_FP4 = 1, 16, 32


@pytest.fixture(scope="module")
def engine():
    import torch
    assert torch.cuda.is_available()
    from paper_2112_07552_b200 import Engine
    e = Engine(0)
    yield e
    e.close()


def run(engine, A, B, agg, flags):
    import torch
    out, st = engine.join_agg(to_dev(A, torch), to_dev(B, torch), agg, flags=flags, with_stats=True)
    return res_np(out), st


@pytest.mark.parametrize("name,scale,flags", [
    ("c1", 1.0, FORCE_DENSE), ("c1", 1.0, FORCE_DENSE | NO_FP4), ("c1s", 1.0, FORCE_DENSE),
    ("c1s", 1.0, FORCE_DENSE | FORCE_WIDE), ("c2", 0.1, FORCE_DENSE), ("c2", 0.1, FORCE_DENSE | NO_FP4),
    ("c3", 1 / 16, FORCE_DENSE), ("c4", 1 / 1024, FORCE_DENSE), ("c4s", 1 / 1024, FORCE_DENSE),
    ("c5s", 1 / 512, FORCE_DENSE), ("c2b", 0.05, FORCE_DENSE), ("c2b", 0.05, FORCE_DENSE | NO_FP4)])
def test_block_sparse_forced_matches_oracle(engine, oracle_mod, monkeypatch, name, scale, flags):
    monkeypatch.setenv("TCUDB_BLOCK_SPARSE", "1")
    monkeypatch.setenv("TCUDB_FP4_ALWAYS", "1")  # e2m1 also on small products
    A, B, agg = datagen.make_config(name, scale)
    ref = oracle_mod.join_agg(A, B, agg)
    out, st = run(engine, A, B, agg, flags)
    assert st["path"] == 0 and 0 < st["block_active"] <= 1.0
    compare(out, ref, agg, float_vals=name.startswith("c4"))


def test_block_sparse_skips_on_blocked_input(engine, oracle_mod, monkeypatch):
    """c2b (blocked entity matching, token ids randomly permuted): the key reordering
    recovers the blocks, the selector takes the dense path with a small active share, and
    the result is the oracle's; with the analysis off the plain dense / sparse result is
    the same."""
    A, B, agg = datagen.make_config("c2b")
    ref = oracle_mod.join_agg(A, B, agg)
    out, st = run(engine, A, B, agg, 0)
    assert st["path"] == 0 and 0 < st["block_active"] < 0.1, st["block_active"]
    compare(out, ref, agg)
    monkeypatch.setenv("TCUDB_BLOCK_SPARSE", "0")
    out2, st2 = run(engine, A, B, agg, 0)
    assert st2["block_active"] == 0
    compare(out2, ref, agg)


def test_block_sparse_empty_tiles_and_chunks(engine, oracle_mod, monkeypatch):
    """Block-diagonal COUNT with multi-byte cells (u8 counts > 1 -> digit planes when
    forced wide) and a K longer than one int32 chunk would allow for 255 x 255 cells:
    whole tiles have no active K-block (zeros written without an accumulator)."""
    monkeypatch.setenv("TCUDB_BLOCK_SPARSE", "1")
    rng = np.random.default_rng(3)
    nb, per, kv = 6, 300, 700           # 6 blocks of 300 groups, 700 private keys each
    g = np.repeat(np.arange(nb * per), 40)
    blk = g // per
    k = blk * kv + rng.integers(0, kv, len(g))
    v = rng.integers(-3, 4, len(g))
    A = datagen.Table(k.astype(np.int64), g.astype(np.int32), v.astype(np.int32))
    h = np.repeat(np.arange(nb * per), 40)
    kb = (h // per) * kv + rng.integers(0, kv, len(h))
    B = datagen.Table(kb.astype(np.int64), h.astype(np.int32), rng.integers(-3, 4, len(h)).astype(np.int32))
    for agg, flags in (("count", FORCE_DENSE), ("sum", FORCE_DENSE), ("sum", FORCE_DENSE | FORCE_WIDE)):
        ref = oracle_mod.join_agg(A, B, agg)
        out, st = run(engine, A, B, agg, flags)
        assert st["path"] == 0 and st["block_active"] < 0.5
        compare(out, ref, agg)
