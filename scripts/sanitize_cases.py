"""Small inputs over every plan, for compute-sanitizer (memcheck / racecheck / synccheck).

usage: compute-sanitizer --tool <tool> python scripts/sanitize_cases.py [quick]
Covers: c1 / c1s (COUNT, SUM, AVG, Q3, Q4) on the selector's path and forced dense /
sparse, the wide (int64 scratch) path, e2m1 forced on small products, the band-SPA
schedules (one pass, count + write), the hash-partitioned path, float SUM (bf16 direct,
hi/lo split; the fused direct fill), sampled group dictionaries, random tiny instances, triangles (both paths), the chain join and the
a6 GEMM kinds. Every result is checked against the oracle (test infrastructure).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import datagen  # noqa: E402
import oracle  # noqa: E402
from parity_util import compare  # noqa: E402
from paper_2112_07552_b200 import Engine  # noqa: E402

quick = "quick" in sys.argv
eng = Engine(0)
dev = lambda T: {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in T.items() if v is not None}  # noqa
host = lambda out: {k: v.cpu().numpy() for k, v in out.items()}  # noqa
n_checks = 0


def check(A, B, agg, flags=0, env=None, float_vals=False):
    global n_checks
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        out = host(eng.join_agg(dev(A), dev(B), agg, flags=flags))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    compare(out, oracle.join_agg(A, B, agg), agg, float_vals=float_vals)
    n_checks += 1


for name in ("c1", "c1s"):
    A, B, agg = datagen.make_config(name)
    for flags in (0, 1, 2, 16, 32):
        check(A, B, agg, flags)
    check(A, B, agg, 1, {"TCUDB_FP4_ALWAYS": "1"})
    for spa in ("TCUDB_SPA_ONE_PASS",):
        check(A, B, agg, 2, {spa: "1"})
    check(A, B, agg, 2, {"TCUDB_NO_SPA_FUSED": "1"})
    check(A, B, agg, 2, {"TCUDB_NO_SPA": "1"})
A, B, _ = datagen.make_config("c1s")
for shape, (a, b) in {"q3": (dict(A, g=None), B), "q4": (dict(A, g=None), dict(B, g=None)), "avg": (A, B)}.items():
    check(a, b, "avg" if shape == "avg" else "sum")
A, B, agg = datagen.make_config("c5s", 1 / 1024)
check(A, B, agg, 0, {"TCUDB_FORCE_HASHPART": "1"})
check(A, B, "count", 0, {"TCUDB_FORCE_HASHPART": "1"})
A, B, agg = datagen.make_config("c4s", 1 / 4096)
check(A, B, agg, 0, float_vals=True)
check(A, B, agg, 2, float_vals=True)
A, B, agg = datagen.make_config("c4", 1 / 4096)
check(A, B, agg, 0, float_vals=True)
# a2 + a5 fused (deferred codes, fill_direct.cu): bf16 cells, hi/lo split + e2m1 pattern
check(A, B, agg, 1, {"TCUDB_LAZY_CODES": "1"}, float_vals=True)
A, B, agg = datagen.make_config("c4s", 1 / 4096)
check(A, B, agg, 1, {"TCUDB_LAZY_CODES": "1"}, float_vals=True)
# sampled group dictionaries + shared-memory code lookup (hash-partitioned path, 2^22 tuples)
A, B, agg = datagen.make_config("c5", 1 / 4)
check(A, B, agg, 0, {"TCUDB_FORCE_HASHPART": "1"})
rng = np.random.default_rng(7)
for i in range(6 if quick else 24):
    vk = ("none", "int", "float")[i % 3]
    A, B = datagen.random_tiny(rng, vkind=vk)
    agg = "count" if vk == "none" else "sum"
    check(A, B, agg, (0, 1, 2)[(i // 3) % 3], float_vals=vk == "float")
for path in ("dense", "sparse"):
    os.environ["TCUDB_TRI_PATH"] = path
    s10, d10 = (torch.tensor(x, device="cuda") for x in zip(*[(i, j) for i in range(10) for j in range(i + 1, 10)]))
    assert eng.triangle_count(s10, d10) == 120
os.environ.pop("TCUDB_TRI_PATH", None)
n = 6
src, dst = (np.array(x) for x in zip(*[(i, j) for i in range(n) for j in range(n) if i != j]))
r = host(eng.chain_join_agg(dev({"k": dst, "g": src}), dev({"k": src, "g": dst}), dev({"k": src, "g": dst})))
assert len(r["agg"]) == n * n
g = torch.Generator(device="cuda").manual_seed(1)
Ai = torch.randint(-128, 128, (128, 256), generator=g, device="cuda", dtype=torch.int32).to(torch.int8)
Bi = torch.randint(-128, 128, (256, 256), generator=g, device="cuda", dtype=torch.int32).to(torch.int8)
assert torch.equal(eng.gemm(Ai, Bi).double(), Ai.double() @ Bi.double().T)
torch.cuda.synchronize()
print(f"SANITIZE_CASES_OK {n_checks} checked queries, {eng.launch_count} kernel launches")
eng.close()
