import os, sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import datagen, oracle
from paper_2112_07552_b200 import Engine
from parity_util import to_dev, res_np
e = Engine(0)
seed = 4
rng = np.random.default_rng(1000 + seed)
for it in range(6):
    n_a, n_b = int(rng.integers(1, 60000)), int(rng.integers(1, 60000))
    kspan = int(rng.choice([50, 3000, 10 ** 6, 2 ** 40]))
    zipf = rng.random() < 0.3
    def keys(n):
        k = (rng.zipf(1.3, n) % kspan) if zipf else rng.integers(0, kspan, n)
        return (k * int(rng.choice([1, 7919])) - kspan // 3).astype(rng.choice([np.int32, np.int64]) if kspan < 2 ** 30 else np.int64)
    G, H = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
    vk = rng.choice(["none", "int", "float"])
    def vals(n):
        if vk == "none": return None
        if vk == "int": return rng.integers(-30, 31, n).astype(rng.choice([np.int32, np.int64]))
        return rng.uniform(-4, 4, n).astype(np.float32)
    A = datagen.Table(keys(n_a), rng.integers(0, G, n_a) * 3 - 100, vals(n_a))
    B = datagen.Table(keys(n_b), rng.integers(0, H, n_b) - 7, vals(n_b))
    agg = "count" if vk == "none" else rng.choice(["sum", "avg"])
    if vk != "float":
        for shape in ("h_only", "none"): pass
        continue
    ref = oracle.join_agg(A, B, "sum")
    for flags, env in ((0, {}), (1, {}), (2, {}), (2, {"TCUDB_SPA_ONE_PASS": "1"}), (0, {"TCUDB_FORCE_HASHPART": "1"})):
        os.environ.update(env)
        out, st = e.join_agg(to_dev(A, torch), to_dev(B, torch), "sum", flags=flags, with_stats=True)
        for k_ in env: del os.environ[k_]
        o = res_np(out)
        err = np.abs(o["agg"] - ref["sum"])
        ratio = err / np.maximum(ref["abs"], 1e-30)
        rel = err / np.maximum(np.abs(ref["sum"]), 0.01 * ref["abs"])
        print(it, "n", n_a, n_b, "kspan", kspan, "G,H", G, H, "flags", flags, env, "path", st["path"], "elem", st["elem"],
              "K", st["K"], "max err/S_abs %.2e" % ratio.max(), "max tol-ratio %.3f" % (rel.max() / 1e-3))
