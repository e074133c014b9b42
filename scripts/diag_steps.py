"""Per-step stage times for one config (variance diagnosis)."""
import sys, json, time, numpy as np, torch
sys.path.insert(0, '.')
import datagen
from paper_2112_07552_b200 import Engine
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A, B, agg = datagen.make_config(cfg)
e = Engine(0)
dev = lambda T: {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in T.items() if v is not None}
dA, dB = dev(A), dev(B)
for i in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out, st = e.join_agg(dA, dB, agg, flags=flags, with_stats=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    del out
    print(cfg, i, f"wall {1e3*(t1-t0):.2f} ms", {k: round(st[k], 3) for k in ("ms_stats","ms_encode","ms_fill","ms_gemm","ms_sparse","ms_compact","ms_total")}, "path", st["path"], "elem", st["elem"], flush=True)
