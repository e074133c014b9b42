"""Host-side overhead of small queries: Python wall per call vs device span, and the library's
per-stage host / device clocks (TCUDB_HOST_TRACE=1). usage: python scripts/host_trace.py c1"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
from paper_2112_07552_b200 import Engine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
A, B, agg = datagen.make_config(cfg)
dev = lambda T: {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in T.items() if v is not None}
dA, dB = dev(A), dev(B)
eng = Engine(0)
for _ in range(5):
    eng.join_agg(dA, dB, agg)
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N):
    out = eng.join_agg(dA, dB, agg)
    del out
torch.cuda.synchronize()
print(f"{cfg}: python wall per call (no stats) {1e3 * (time.perf_counter() - t0) / N:.3f} ms")
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(N):
    out = eng.join_agg(dA, dB, agg)
    del out
ev1.record()
torch.cuda.synchronize()
print(f"{cfg}: device span per call {ev0.elapsed_time(ev1) / N:.3f} ms")
t0 = time.perf_counter()
for _ in range(N):
    eng._table_dev(dA), eng._table_dev(dB)
print(f"python marshalling per call {1e3 * (time.perf_counter() - t0) / N:.4f} ms")
os.environ["TCUDB_HOST_TRACE"] = "1"
out, st = eng.join_agg(dA, dB, agg, with_stats=True)
torch.cuda.synchronize()
print({k: v for k, v in st.items() if k.startswith("ms_")}, "launches", st.get("n_launches"))
