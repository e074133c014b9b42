"""A/B of the 1-CTA and CTA-pair tcgen05 GEMM kernels on a c2-shaped product (kernel time, CUDA events)."""
import os, sys, torch
sys.path.insert(0, ".")
from paper_2112_07552_b200 import Engine
e = Engine(0)
M, N, K = 10240, 10240, 18688
for kind in sys.argv[1:] or ["i8", "fp4", "bf16"]:
    if kind == "i8":
        A = torch.randint(0, 2, (M, K), dtype=torch.uint8, device="cuda"); B = torch.randint(0, 2, (N, K), dtype=torch.uint8, device="cuda")
        f = lambda: e.gemm(A, B, False, False); flops = 2.0 * M * N * K
    elif kind == "bf16":
        A = torch.rand(M, K // 2, device="cuda").bfloat16(); B = torch.rand(N, K // 2, device="cuda").bfloat16()
        f = lambda: e.gemm(A, B); flops = 2.0 * M * N * (K // 2)
    else:
        A = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device="cuda") & 0x22
        B = torch.randint(0, 256, (10080, K // 2), dtype=torch.uint8, device="cuda") & 0x22
        f = lambda: e.gemm(A, B, fp4=True); flops = 2.0 * M * 10080 * K
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): f()
    t.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(t) / 10
    print(kind, "pair" if os.environ.get("TCUDB_GEMM_PAIR") == "1" else "1cta", f"{ms:.3f} ms", f"{flops / ms / 1e9:.0f} TFLOP/s", flush=True)
