"""Probe: int8 (torch._int_mm) and bf16 matmul throughput, host cores, GPU info.
Context numbers only (cuBLASLt yardstick for the int8 roofline denominator)."""
import os, json, time, subprocess, torch
dev = torch.device("cuda:0")
out = {"gpu": torch.cuda.get_device_name(0), "host_cores": len(os.sched_getaffinity(0))}
try:
    out["lscpu_model"] = [l for l in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines() if "Model name" in l]
except Exception as e:
    out["lscpu_model"] = str(e)
props = torch.cuda.get_device_properties(0)
out["sm_count"] = props.multi_processor_count
out["total_mem_gb"] = props.total_memory / 1e9
out["l2_bytes"] = getattr(props, "L2_cache_size", None)
def bench(fn, iters=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(iters):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best
for n in (8192, 16384):
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
    ms = bench(lambda: torch._int_mm(a, b.t()))
    out[f"int8_intmm_{n}_tops"] = 2 * n**3 / ms / 1e9
    x = torch.randn(n, n, dtype=torch.bfloat16, device=dev); y = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    ms = bench(lambda: x @ y.t())
    out[f"bf16_{n}_tflops"] = 2 * n**3 / ms / 1e9
# sustained int8 for ~3 s
n = 8192
a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
torch.cuda.synchronize(); t0 = time.time(); cnt = 0
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True); s.record()
while time.time() - t0 < 3.0:
    for _ in range(20): torch._int_mm(a, b.t())
    cnt += 20
    torch.cuda.synchronize()
e.record(); torch.cuda.synchronize()
out["int8_intmm_8192_sustained_tops"] = 2 * n**3 * cnt / s.elapsed_time(e) / 1e9
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_peaks.json", "w"), indent=1)
