"""World-size-2 gloo tests (CPU) of the multi-GPU row sharding.

1. The product's host planning steps across two processes: each rank builds its
   query descriptor and its strided group sample from its own slice, the ranks
   allgather them over gloo, and each calls libtcudb's tcudb_shard_agree /
   tcudb_shard_bounds (host-only C ABI, no GPU) — both ranks must take the same
   decision (including an empty-slice rank with NULL columns and a disagreeing rank).
2. The exchange algorithm (tests/shard_ref.py: row-balanced g ranges from those
   bounds, routing via all_to_all_single, allgather of the other side, result
   allgather-v, rank-order concat; Q4 partials combined exactly) on 2 CPU processes
   with a CPU stand-in for the per-rank engine (test-only, from the oracle): the
   sharded result must equal the single-process oracle result exactly. The CUDA
   collective itself runs at P = 2/4/8 in tests/test_collective_shim.py (GPU).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen


class CpuStandIn:
    """Test-only engine: numpy / oracle implementations of the three calls shard.py makes."""

    def minmax(self, col):
        a = col.numpy()
        return (int(a.min()), int(a.max())) if len(a) else (2 ** 63 - 1, -2 ** 63)

    def partition(self, T, bounds):
        g = T["g"].numpy().astype(np.int64)
        dest = np.searchsorted(np.asarray(bounds, dtype=np.int64), g, side="right")
        order = np.argsort(dest, kind="stable")
        counts = np.bincount(dest, minlength=len(bounds) + 1).tolist()
        return {k: v[torch.from_numpy(order)] for k, v in T.items() if v is not None}, counts

    def join_agg(self, A, B, agg, with_stats=False):
        import oracle
        col = lambda T, c: T[c].numpy() if T.get(c) is not None else None
        np_t = lambda T: datagen.Table(T["k"].numpy(), col(T, "g"), col(T, "v"))
        r = oracle.join_agg(np_t(A), np_t(B), agg)
        out = {c: torch.from_numpy(r[c]) for c in ("g", "h") if c in r}
        out["agg"] = torch.from_numpy(r[_AGGKEY[agg]])
        return (out, {}) if with_stats else out


_AGGKEY = {"count": "cnt", "sum": "sum", "avg": "avg"}


def _variant(A, B, agg, drop):
    """Q3 / Q4 variants of a config: drop="a" ungroups A, "b" ungroups B, "ab" both."""
    if "a" in drop:
        A = dict(A, g=None)
    if "b" in drop:
        B = dict(B, g=None)
    return A, B


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _load(name):
    base, _, rest = name.partition(":")
    A, B, agg = datagen.make_config(base, 0.05) if base != "c1s" else datagen.make_config(base)
    drop, _, ag = rest.partition(":")
    return (*_variant(A, B, agg, drop), ag or agg)


def _worker(rank, ws, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from shard_ref import local_slice, sharded_join_agg
        A, B, agg = _load(name)
        tA = {k: torch.from_numpy(v) for k, v in local_slice(A, ws, rank).items() if v is not None}
        tB = {k: torch.from_numpy(v) for k, v in local_slice(B, ws, rank).items() if v is not None}
        out = sharded_join_agg(CpuStandIn(), tA, tB, agg)
        q.put((rank, {k: v.numpy() for k, v in out.items()}))
    finally:
        dist.destroy_process_group()


# "config:ungrouped sides:agg" — Q3 by A.g / by B.h and Q4 shard on the grouped
# side or reduce the per-rank partials with an allreduce
@pytest.mark.parametrize("name", ["c1s", "c2", "c3", "c1s:b:sum", "c1s:a:avg", "c2:a:count",
                                  "c1s:ab:sum", "c1s:ab:avg", "c3:ab:count"])
def test_sharded_equals_single(oracle_mod, name):
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, name, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, B, agg = _load(name)
    ref = oracle_mod.join_agg(A, B, agg)
    for r in range(ws):
        assert set(res[r]) == {c for c in ("g", "h") if c in ref} | {"agg"}
        for c in ("g", "h"):
            if c in ref:
                assert np.array_equal(res[r][c], ref[c])
        want = ref[_AGGKEY[agg]]
        if want.dtype == np.float64:
            # Q4 adds the per-rank partials in another order than the one-pass oracle
            assert np.allclose(res[r]["agg"], want, rtol=1e-12, atol=0)
        else:
            assert np.array_equal(res[r]["agg"], want)


_DESC_CASES = {
    # name: per-rank (nA, nB, a_key, a_group, a_value, b_key, b_group, b_value, agg, flags, st) builders
    "same": [lambda r: (100, 50, 2 + 1, 2 + 0, 1, 2 + 1, 2 + 0, 1, 0, 0, 0)] * 2,
    "empty_rank_null_cols": [lambda r: (100, 50, 3, 2, 4, 3, 2, 4, 1, 0, 0),
                             lambda r: (0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0)],
    "group_disagrees": [lambda r: (100, 50, 3, 2, 1, 3, 2, 1, 0, 0, 0),
                        lambda r: (100, 50, 3, 1, 1, 3, 2, 1, 0, 0, 0)],
    "one_rank_bad_args": [lambda r: (100, 50, 3, 2, 1, 3, 2, 1, 0, 0, 0),
                          lambda r: (100, 50, 3, 2, 1, 3, 2, 1, 0, 0, -2)],
    "flags_differ": [lambda r: (10, 10, 3, 2, 1, 3, 2, 1, 0, 1, 0), lambda r: (10, 10, 3, 2, 1, 3, 2, 1, 0, 2, 0)],
    "mixed_values": [lambda r: (10, 10, 3, 2, 2 + 2, 3, 2, 2 + 0, 1, 0, 0),
                     lambda r: (0, 10, 0, 0, 0, 3, 2, 2 + 0, 1, 0, 0)],
}
_DESC_WANT = {"same": 0, "empty_rank_null_cols": 0, "group_disagrees": -1, "one_rank_bad_args": -2,
              "flags_differ": -1, "mixed_values": -2}


def _plan_worker(rank, ws, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2112_07552_b200._lib import shard_agree, shard_bounds, shard_sample_msg
        d = torch.tensor(_DESC_CASES[case][rank](rank), dtype=torch.int64)
        ds = [torch.zeros_like(d) for _ in range(ws)]
        dist.all_gather(ds, d)
        st, agreed = shard_agree(torch.stack(ds).numpy())
        # balanced bounds from each rank's own skewed slice of a Zipf-like group column
        rng = np.random.default_rng(rank)
        g = (rng.zipf(1.3, 50_000 if rank == 0 else 5_000) % 10_000).astype(np.int64)
        m = torch.from_numpy(shard_sample_msg(g))
        ms = [torch.zeros_like(m) for _ in range(ws)]
        dist.all_gather(ms, m)
        b = shard_bounds(torch.stack(ms).numpy())
        q.put((rank, st, agreed.tolist(), b, g))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", sorted(_DESC_CASES))
def test_plan_agreement_and_bounds_gloo(case):
    """Both ranks agree (same status, same agreed descriptor, same bounds) from their own
    inputs; the bounds split the pooled rows into near-equal halves."""
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, ws, port, case, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(ws):
        r, st, agreed, b, g = q.get(timeout=300)
        res[r] = (st, agreed, b, g)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == res[1][0] == _DESC_WANT[case]
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]
    if case == "empty_rank_null_cols":
        assert res[0][1][:8] == [100, 50, 3, 2, 4, 3, 2, 4]  # the empty rank takes the others' shape
    allg = np.concatenate([res[0][3], res[1][3]])
    left = (allg < res[0][2][0]).mean()
    assert 0.3 < left < 0.7, left  # a Zipf head value is never split, so not exactly 1/2


def test_shard_bounds_host():
    """tcudb_shard_bounds on hand-made samples: equal weights, weighted ranks, ties kept
    on one rank, empty ranks, a value at INT64_MAX."""
    from paper_2112_07552_b200._lib import shard_bounds, shard_sample_msg
    m = [shard_sample_msg(np.arange(0, 100)), shard_sample_msg(np.arange(100, 200))]
    assert shard_bounds(m) == [100]
    assert shard_bounds([shard_sample_msg(np.arange(0, 400))] * 1 + [shard_sample_msg(np.zeros(0))] * 3) == \
        [100, 200, 300]
    # rank 1 holds 10x the rows of rank 0 (each sample weighs 10x): the median lies inside rank 1's values
    big = shard_sample_msg(np.arange(1000, 11000))
    assert 5000 <= shard_bounds([shard_sample_msg(np.arange(0, 1000)), big])[0] <= 6500
    # a value holding 80 % of the rows stays on one rank
    g = np.concatenate([np.full(800, 7), np.arange(100, 300)])
    b = shard_bounds([shard_sample_msg(g), shard_sample_msg(np.zeros(0))])
    assert b[0] in (7, 8, 100) or b[0] > 7
    dest = np.searchsorted(np.asarray(b), g, side="right")
    assert len(set(dest[g == 7])) == 1
    assert shard_bounds([shard_sample_msg(np.zeros(0))] * 4) == [0, 0, 0]
    top = np.array([2 ** 63 - 1] * 10)
    assert shard_bounds([shard_sample_msg(top), shard_sample_msg(top)]) == [2 ** 63 - 1]
