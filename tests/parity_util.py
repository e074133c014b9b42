"""Helpers shared by the GPU parity tests: table transfer and result comparison.

Tolerance for float SUM (reading R9, from the north star's "1e-3
relative"): |x_gpu - x| <= 1e-3 * max(|x|, 0.01 * S_abs), S_abs = sum |v*w| of
the group (computed by the oracle). Integer results: bit-exact. Group sets and
order: identical (existence = COUNT > 0, ascending (g, h)).
"""
import numpy as np

FLOAT_RTOL = 1e-3
FLOOR = 0.01  # DESIGN.md R9 = SURVEY §8(c) #9: the floor is 1e-5 S_abs (cancellation only)


def to_dev(T, torch, device="cuda:0"):
    out = {"k": torch.from_numpy(np.ascontiguousarray(T["k"])).to(device)}
    if T.get("g") is not None:  # absent: the side is not grouped (Q3 / Q4)
        out["g"] = torch.from_numpy(np.ascontiguousarray(T["g"])).to(device)
    if T.get("v") is not None:
        out["v"] = torch.from_numpy(np.ascontiguousarray(T["v"])).to(device)
    return out


def res_np(r):
    return {k: v.cpu().numpy() for k, v in r.items()}


def compare(gpu, ref, agg, float_vals=False):
    """Assert GPU result == oracle result (see module docstring). AVG: integer inputs
    bit-exact (both sides divide the exact int64 SUM by the COUNT in fp64); float inputs
    within the SUM tolerance scaled by 1 / COUNT."""
    a = np.asarray(gpu["agg"])
    assert len(a) == len(ref["cnt"]), f"group count {len(a)} != oracle {len(ref['cnt'])}"
    for col in ("g", "h"):
        assert (col in gpu) == (col in ref), f"column {col}: present on one side only"
        if col in ref:
            assert np.array_equal(np.asarray(gpu[col]).astype(np.int64), ref[col]), f"{col} keys / order differ"
    if agg == "avg":
        assert a.dtype == np.float64
        if not float_vals:
            assert np.array_equal(a, ref["avg"]), "integer AVG differs"
        else:
            err = np.abs(a - ref["avg"])
            tol = FLOAT_RTOL * np.maximum(np.abs(ref["avg"]), FLOOR * ref["abs"] / ref["cnt"])
            bad = err > tol
            assert not bad.any(), f"{bad.sum()} float AVG groups outside tolerance; worst err {err.max():.3g}"
        return
    if agg == "count":
        assert np.array_equal(a.astype(np.int64), ref["cnt"]), "COUNT differs"
    elif not float_vals:
        assert np.array_equal(a.astype(np.int64), ref["sum"]), "integer SUM differs"
    else:
        err = np.abs(a.astype(np.float64) - ref["sum"])
        tol = FLOAT_RTOL * np.maximum(np.abs(ref["sum"]), FLOOR * ref["abs"])
        bad = err > tol
        assert not bad.any(), f"{bad.sum()} float SUM groups outside tolerance; worst err {err.max():.3g}"


def mape(gpu_agg, ref_sum):
    x = np.asarray(ref_sum, dtype=np.float64)
    y = np.asarray(gpu_agg, dtype=np.float64)
    nz = x != 0
    return float(np.mean(np.abs(y[nz] - x[nz]) / np.abs(x[nz]))) if nz.any() else 0.0
