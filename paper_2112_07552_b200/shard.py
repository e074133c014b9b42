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

Aggregates with one group column (Q3) shard the same way on the grouped side:
GROUP BY A.g routes A by g range (as above); GROUP BY B.h routes B by h range and
allgathers A. Without GROUP BY (Q4) every rank joins its own A slice with the
allgathered B and the one partial aggregate per rank is combined with an allreduce
(SUM of COUNT, SUM of SUM; AVG = the reduced SUM / the reduced COUNT).
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


def _route(eng, T, bounds, dist, group):
    """Send every tuple of T to the rank owning its "g" range (all-to-all-v)."""
    import torch
    dev = T["k"].device
    Tp, counts = eng.partition(T, bounds)
    send = torch.tensor(counts, dtype=torch.int64, device=dev)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    rc = [int(x) for x in recv.tolist()]
    out = {}
    for col, v in Tp.items():
        o = torch.empty(sum(rc), dtype=v.dtype, device=dev)
        dist.all_to_all_single(o, v, output_split_sizes=rc, input_split_sizes=counts, group=group)
        out[col] = o
    return out


def _global_bounds(eng, col, dist, group):
    """P equal-width ranges of a column's global [min, max] (allreduce of tcudb_minmax)."""
    import torch
    mn, mx = eng.minmax(col)
    t = torch.tensor([mn, mx], dtype=torch.int64, device=col.device)
    lo, hi = t[:1].clone(), t[1:].clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return range_bounds(int(lo.item()), int(hi.item()), dist.get_world_size(group))


def _one(res, dtype, dev):
    """The (at most one) local Q4 aggregate as a 1-element tensor (0 when empty)."""
    import torch
    a = res["agg"]
    return a[:1].to(dtype) if a.numel() else torch.zeros(1, dtype=dtype, device=dev)


def _sharded_q4(eng, A, B, agg, with_stats, group):
    import torch
    import torch.distributed as dist
    dev = A["k"].device
    Bf = {col: _all_gather_var(v, dist, group) for col, v in B.items() if v is not None}
    st = None
    if agg == "avg":
        rc = eng.join_agg(A, Bf, "count")
        out = eng.join_agg(A, Bf, "sum", with_stats=with_stats)
    else:
        out = eng.join_agg(A, Bf, agg, with_stats=with_stats)
        rc = None
    rs, st = (out if with_stats else (out, None))
    n = torch.tensor([rs["agg"].numel()], dtype=torch.int64, device=dev)
    dist.all_reduce(n, group=group)
    s = _one(rs, rs["agg"].dtype, dev)
    dist.all_reduce(s, group=group)
    if agg == "avg":
        c = _one(rc, torch.int64, dev)
        dist.all_reduce(c, group=group)
        s = s.to(torch.float64) / c.clamp(min=1).to(torch.float64)
    full = {"agg": s if int(n.item()) > 0 else s[:0]}
    return (full, st) if with_stats else full


def sharded_join_agg(eng, A, B, agg="count", with_stats=False, group=None):
    """Collective version of Engine.join_agg: A, B are this rank's slices (dicts
    of device tensors); returns the full result on every rank."""
    import torch.distributed as dist
    ga, gb = A.get("g") is not None, B.get("g") is not None
    if not ga and not gb:
        return _sharded_q4(eng, A, B, agg, with_stats, group)
    # the grouped side is routed by group range: every output group lives on exactly one
    # rank, so COUNT, SUM and AVG are all complete locally
    R, O = (A, B) if ga else (B, A)
    bounds = _global_bounds(eng, R["g"], dist, group)
    Rr = _route(eng, R, bounds, dist, group)
    Of = {col: _all_gather_var(v, dist, group) for col, v in O.items() if v is not None}
    Ar, Bf = (Rr, Of) if ga else (Of, Rr)
    out = eng.join_agg(Ar, Bf, agg, with_stats=with_stats)
    res, st = (out if with_stats else (out, None))
    # allgather-v of the result tuples (rank order = ascending group ranges)
    full = {col: _all_gather_var(v, dist, group) for col, v in res.items()}
    return (full, st) if with_stats else full
