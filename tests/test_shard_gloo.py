"""World-size-2 gloo test (CPU) of the multi-GPU row-sharding driver.

The exchange logic of paper_2112_07552_b200/shard.py (g-range bounds, A routing
via all_to_all_single, B allgather, result allgather-v, rank-order concat) is
run on 2 CPU processes; the per-rank compute is a CPU stand-in built from the
oracle (test-only), so the sharded result must equal the single-process oracle
result exactly. The CUDA partition kernel itself is covered by a GPU test.
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
        np_t = lambda T: datagen.Table(T["k"].numpy(), T["g"].numpy(), T["v"].numpy() if "v" in T else None)
        r = oracle.join_agg(np_t(A), np_t(B), agg)
        out = {"g": torch.from_numpy(r["g"]), "h": torch.from_numpy(r["h"]),
               "agg": torch.from_numpy(r["cnt"] if agg == "count" else r["sum"])}
        return (out, {}) if with_stats else out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2112_07552_b200.shard import local_slice, sharded_join_agg
        A, B, agg = datagen.make_config(name, 0.05) if name != "c1s" else datagen.make_config(name)
        tA = {k: torch.from_numpy(v) for k, v in local_slice(A, ws, rank).items() if v is not None}
        tB = {k: torch.from_numpy(v) for k, v in local_slice(B, ws, rank).items() if v is not None}
        out = sharded_join_agg(CpuStandIn(), tA, tB, agg)
        q.put((rank, {k: v.numpy() for k, v in out.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1s", "c2", "c3"])
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
    A, B, agg = datagen.make_config(name, 0.05) if name != "c1s" else datagen.make_config(name)
    ref = oracle_mod.join_agg(A, B, agg)
    for r in range(ws):
        assert np.array_equal(res[r]["g"], ref["g"])
        assert np.array_equal(res[r]["h"], ref["h"])
        assert np.array_equal(res[r]["agg"], ref["cnt"] if agg == "count" else ref["sum"])


def test_range_bounds():
    from paper_2112_07552_b200.shard import range_bounds
    assert range_bounds(0, 99, 4) == [25, 50, 75]
    assert range_bounds(-(2 ** 63), 2 ** 63 - 1, 2) == [0]
    b = range_bounds(5, 5, 8)
    assert len(b) == 7 and all(x >= 5 for x in b)
