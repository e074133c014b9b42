"""TEST INFRASTRUCTURE — a torch.distributed reference driver of the §8(e) row sharding.

The product's multi-GPU path is the collective tcudb_join_agg inside libtcudb
(csrc/collective.cu, NCCL). This module writes the same exchange algorithm over
torch.distributed collectives so that it can run on CPU processes with the gloo
backend (tests/test_shard_gloo.py), with a CPU stand-in for the per-rank engine;
the range bounds come from the product's own host planning step
(tcudb_shard_bounds over allgathered samples, as collective.cu computes them).

Steps per query on every rank r of P (each rank starts with a 1/P slice of A
and of B):
  1. strided sample of A.g per rank (allgather) -> P row-balanced g ranges;
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


from datagen import local_slice  # noqa: F401  (re-exported for the tests)


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
    """Row-balanced ranges: every rank's strided sample of the column is allgathered and
    the product's host planning step (tcudb_shard_bounds) picks the weighted quantiles."""
    import torch
    from paper_2112_07552_b200._lib import shard_bounds, shard_sample_msg
    m = torch.from_numpy(shard_sample_msg(col.cpu().numpy())).to(col.device)
    ms = [torch.zeros_like(m) for _ in range(dist.get_world_size(group))]
    dist.all_gather(ms, m, group=group)
    return shard_bounds(torch.stack(ms).cpu().numpy())


def _one(res, dtype, dev):
    """The (at most one) local Q4 aggregate as a 1-element tensor (0 when empty)."""
    import torch
    a = res["agg"].to(dev)
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
    # partials allgathered and combined exactly in rank order (integer SUM in Python ints:
    # a total beyond int64 raises, as the library's E_OVERFLOW)
    part = torch.stack([torch.tensor(rs["agg"].numel(), dtype=torch.float64),
                        _one(rs, torch.float64, "cpu")[0] if rs["agg"].dtype == torch.float64 else torch.tensor(0.0),
                        torch.tensor(0.0)])
    ints = torch.tensor([int(_one(rs, torch.int64, "cpu")[0]) if rs["agg"].dtype != torch.float64 else 0,
                         int(_one(rc, torch.int64, "cpu")[0]) if rc is not None else 0], dtype=torch.int64)
    ws = dist.get_world_size(group)
    pl = [torch.zeros_like(part) for _ in range(ws)]
    il = [torch.zeros_like(ints) for _ in range(ws)]
    dist.all_gather(pl, part, group=group)
    dist.all_gather(il, ints, group=group)
    n = sum(int(p[0]) for p in pl)
    if rs["agg"].dtype == torch.float64:
        tot = 0.0
        for p in pl:
            tot += float(p[1])
        s = torch.tensor([tot], dtype=torch.float64)
    else:
        tot = sum(int(i[0]) for i in il)
        if not -2 ** 63 <= tot < 2 ** 63:
            raise OverflowError("int64 overflow of the Q4 total")
        s = torch.tensor([tot], dtype=torch.int64)
    if agg == "avg":
        c = sum(int(i[1]) for i in il)
        s = s.to(torch.float64) / max(c, 1)
    full = {"agg": s if n > 0 else s[:0]}
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
