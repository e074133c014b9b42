"""Helpers shared by the GPU parity tests: table transfer and result comparison.

Tolerance for float SUM (reading R9, from the north star's "1e-3
relative"): |x_gpu - x| <= 1e-3 * max(|x|, 0.01 * S_abs), S_abs = sum |v*w| of
the group (computed by the oracle). Integer results: bit-exact. Group sets and
order: identical (existence = COUNT > 0, ascending (g, h)).
"""
import numpy as np

FLOAT_RTOL = 1e-3
FLOOR = 0.01


def to_dev(T, torch, device="cuda:0"):
    out = {"k": torch.from_numpy(np.ascontiguousarray(T["k"])).to(device),
           "g": torch.from_numpy(np.ascontiguousarray(T["g"])).to(device)}
    if T.get("v") is not None:
        out["v"] = torch.from_numpy(np.ascontiguousarray(T["v"])).to(device)
    return out


def res_np(r):
    return {k: v.cpu().numpy() for k, v in r.items()}


def compare(gpu, ref, agg, float_vals=False):
    """Assert GPU result == oracle result (see module docstring)."""
    g, h, a = np.asarray(gpu["g"]), np.asarray(gpu["h"]), np.asarray(gpu["agg"])
    assert len(g) == len(ref["g"]), f"group count {len(g)} != oracle {len(ref['g'])}"
    assert np.array_equal(g.astype(np.int64), ref["g"]), "g keys / order differ"
    assert np.array_equal(h.astype(np.int64), ref["h"]), "h keys / order differ"
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
