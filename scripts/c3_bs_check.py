"""c3: does the selector run the block-sparse analysis? (launch counts and time, default vs
TCUDB_BLOCK_SPARSE=0, same process: the env is read per query)"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
from paper_2112_07552_b200 import Engine  # noqa: E402

A, B, agg = datagen.make_config(sys.argv[1] if len(sys.argv) > 1 else "c3")
dev = lambda T: {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in T.items() if v is not None}
dA, dB = dev(A), dev(B)
eng = Engine(0)
for env in ("", "0"):
    if env:
        os.environ["TCUDB_BLOCK_SPARSE"] = env
    for _ in range(3):
        out, st = eng.join_agg(dA, dB, agg, with_stats=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        out = eng.join_agg(dA, dB, agg)
    torch.cuda.synchronize()
    print(f"TCUDB_BLOCK_SPARSE={env or 'default'}: launches {st['n_launches']}, path {st['path']}, "
          f"block_active {st['block_active']:.3f}, {1e3 * (time.perf_counter() - t0) / 10:.3f} ms/query")
