"""§8(f) f4: dense-vs-sparse selector calibration on B200 (Fig. 9(a)).

Fixed G = H groups of L tuples each (n = G·L per side), join keys uniform over K distinct
values; density of mat(A) = n / (G·K). For each K: query time with FORCE_DENSE (a5+a6),
FORCE_SPARSE (a7) and the selector's own choice (median of 5 after 2 warm-ups), COUNT and
integer SUM. Prints one JSON line per point."""
import json, statistics, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2112_07552_b200 import Engine

e = Engine(0)
G = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
L = int(sys.argv[2]) if len(sys.argv) > 2 else 16
rng = np.random.default_rng(9)


def timed(A, B, agg, flags):
    for _ in range(2):
        e.join_agg(A, B, agg, flags=flags)
    ts, st = [], None
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        out, st = e.join_agg(A, B, agg, flags=flags, with_stats=True)
        torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
        del out
    return statistics.median(ts), st


n = G * L
for K in [64, 256, 1024, 4096, 16384, 65536, 262144, 1048576]:
    for agg in ("count", "sum"):
        ka = rng.integers(0, K, n); kb = rng.integers(0, K, n)
        ga = np.repeat(np.arange(G), L); hb = np.repeat(np.arange(G), L)
        A = {"k": torch.from_numpy(ka).cuda(), "g": torch.from_numpy(ga).cuda()}
        B = {"k": torch.from_numpy(kb).cuda(), "g": torch.from_numpy(hb).cuda()}
        if agg == "sum":
            A["v"] = torch.from_numpy(rng.integers(-50, 51, n)).cuda()
            B["v"] = torch.from_numpy(rng.integers(-50, 51, n)).cuda()
        td, sd = timed(A, B, agg, 1)
        ts_, ss = timed(A, B, agg, 2)
        ta, sa = timed(A, B, agg, 0)
        faster = "dense" if td <= ts_ else "sparse"
        chosen = "dense" if sa["path"] == 0 else ("sparse" if sa["path"] == 1 else "reduce")
        print(json.dumps({"G": G, "L": L, "K": K, "agg": agg, "density_pct": 100.0 * n / (G * K),
                          "join_pairs": sa["join_pairs"], "ms_dense": round(td, 4), "ms_sparse": round(ts_, 4),
                          "ms_auto": round(ta, 4), "faster": faster, "selector": chosen,
                          "regret": round(ta / min(td, ts_), 3)}), flush=True)
