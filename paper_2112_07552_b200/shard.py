"""Multi-GPU row sharding of the join + group-by (north star):
output rows are sharded by ranges of A's group key; B is broadcast (allgather)
over NVLink; result tuples are allgathered. One process per GPU, NCCL through
torch.distributed (the plumbing); routing and the local query run in
libtcudb.so kernels (tcudb_minmax, tcudb_partition, tcudb_join_agg).

Steps per query on every rank r of P (each rank starts with a 1/P slice of A
and of B in its HBM):
  1. global min/max of A.g (allreduce) -> P equal-width g ranges;
  2. route A by g range: tcudb_partition + all_to_all_single (sizes first);
  3. allgather B (sizes first, padded);
  4. local query on (A_r, B) -> tuples whose g lies in rank r's range;
  5. allgather-v of the result tuples in rank order. Since ranges are ascending
     in rank and each rank's output is (g, h)-sorted, the concatenation is the
     globally (g, h)-sorted result — identical to the single-GPU result.
"""
from __future__ import annotations

import numpy as np


def local_slice(T, ws, rank):
    """Contiguous 1/ws slice of a host table (numpy columns)."""
    n = len(T["k"])
    lo, hi = n * rank // ws, n * (rank + 1) // ws
    return {k: (None if v is None else np.ascontiguousarray(v[lo:hi])) for k, v in T.items()}


def range_bounds(gmin: int, gmax: int, P: int):
    """P-1 ascending bounds splitting [gmin, gmax] into P equal-width ranges."""
    if gmin > gmax:
        return [0] * (P - 1)
    span = gmax - gmin + 1
    return [gmin + (span * i) // P for i in range(1, P)]


def _all_gather_var(t, dist, group=None):
    """Concatenate 1-D tensors of different lengths from all ranks, in rank order."""
    import torch
    ws = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(ws)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes) if sizes else 0
    pad = torch.zeros(m, dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t
    bufs = [torch.empty(m, dtype=t.dtype, device=t.device) for _ in range(ws)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)])


def sharded_join_agg(eng, A, B, agg="count", with_stats=False, group=None):
    """Collective version of Engine.join_agg: A, B are this rank's slices (dicts
    of device tensors); returns the full result on every rank."""
    import torch
    import torch.distributed as dist
    if A.get("g") is None or B.get("g") is None:
        # the row shards are A.g ranges: an ungrouped side (Q3 / Q4) would need a cross-rank
        # reduction of partial groups, which this sharding does not do
        raise NotImplementedError("sharded_join_agg needs both group columns (Q3/Q4 run on one GPU)")
    ws = dist.get_world_size(group)
    dev = A["k"].device
    # 1. global A.g range (every group (g, h) lives on exactly one rank, so COUNT, SUM
    #    and AVG are all complete locally)
    mn, mx = eng.minmax(A["g"])
    t = torch.tensor([mn, mx], dtype=torch.int64, device=dev)
    lo, hi = t[:1].clone(), t[1:].clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    bounds = range_bounds(int(lo.item()), int(hi.item()), ws)
    # 2. route A by g range
    Ap, counts = eng.partition(A, bounds)
    send = torch.tensor(counts, dtype=torch.int64, device=dev)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    rc = [int(x) for x in recv.tolist()]
    Ar = {}
    for col, v in Ap.items():
        o = torch.empty(sum(rc), dtype=v.dtype, device=dev)
        dist.all_to_all_single(o, v, output_split_sizes=rc, input_split_sizes=counts, group=group)
        Ar[col] = o
    # 3. B everywhere
    Bf = {col: _all_gather_var(v, dist, group) for col, v in B.items() if v is not None}
    # 4. local query on this rank's g range
    out = eng.join_agg(Ar, Bf, agg, with_stats=with_stats)
    res, st = (out if with_stats else (out, None))
    # 5. allgather-v of the result tuples (rank order = ascending g ranges)
    full = {col: _all_gather_var(v, dist, group) for col, v in res.items()}
    return (full, st) if with_stats else full
