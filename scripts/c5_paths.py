import sys, time, numpy as np, torch, os
sys.path.insert(0, '.')
import datagen
from paper_2112_07552_b200 import Engine
e = Engine(0)
for cfg in ("c5s", "c5"):
    A, B, agg = datagen.make_config(cfg)
    dev = lambda T: {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in T.items() if v is not None}
    dA, dB = dev(A), dev(B)
    for hp in ("1", "0"):
        os.environ["TCUDB_NO_HASHPART"] = "0" if hp == "1" else "1"
        for i in range(4):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            out, st = e.join_agg(dA, dB, agg, with_stats=True)
            torch.cuda.synchronize(); t1 = time.perf_counter()
            del out
        print(cfg, "hashpart" if hp == "1" else "general", f"{1e3*(t1-t0):.2f} ms spa_mode={st['spa_mode']}",
              {k: round(st[k], 3) for k in ("ms_encode", "ms_sparse", "ms_compact")}, "kernel ms", round(st["ms_kernel"], 3), flush=True)
