"""bench.py — the driver's benchmark contract for the TCUDB join + group-by hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--also c1,c3,c4,c5]
                    [--impl reference]

One "step" = one whole query (all §8(a) rows: statistics, dictionaries,
selector, fill, tcgen05 GEMM or sparse expand, compaction) over the config's
synthetic tables, inputs already resident in HBM. Headline workload: c2
(BASELINE.json configs[1], entity matching, the int8-class GEMM the metric's
"% of int8 tensor peak" names). The other configs (c1, c3, c4, c5 by default)
are measured in the same run and reported under "configs" with the same keys
(query ms, tuples/s, query-level roofline, dominant-kernel roofline,
cpu_baseline, e2e). L2 is flushed (a 256 MiB write) between timed steps,
outside the timed events.

Metric: input tuples/s = (n_A + n_B) * steps / device time (max over ranks);
query ms = ms_per_step. Rank 0 prints ONE JSON line. Under torchrun (N > 1)
every query is the collective tcudb_join_agg (row-sharded over NCCL inside
libtcudb); a failure of the collective fails the run (no fallback).
--impl reference times the CPU oracle (oracle/, the only other implementation
of the method) on the host cores on the headline workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
PAPER_CONTEXT = ("paper: up to 288x over YDB (GPU query engine) on RTX 3090 + i7-7700K, fp16 WMMA/cuBLAS, "
                 "EM blocking on iTunes-Amazon Price (P:37, P:1494-1501, P:2041-2043)")

WORKLOADS = {
    "c1": "c1: COUNT(*) join of two 1,000-row tables, 64 keys, 32x32 groups",
    "c2": "c2: entity matching, 10k x 10k token-bag records, vocab 32k (Zipf s=1), shared-token COUNT(*)",
    "c3": "c3: 2-hop path COUNT(*) on an R-MAT scale-16 edge table (self-join + group-by)",
    "c4": "c4: SQL matmul of two 8192x8192 (row,col,val) tables, SUM(A.v*B.w), bf16-exact values",
    "c4s": "c4s: c4 with signed fp32 N(0,1) values (not bf16-exact: hi/lo split)",
    "c5": "c5: low-density COUNT(*) join, 2^24 x 2^24 tuples over a 2^22 scrambled int64 key domain",
    "c5s": "c5s: c5 with SUM(A.v*B.w), v,w ~ U{-100..100}",
    "c1s": "c1s: c1 with SUM(A.v*B.w), v,w ~ U{-100..100}",
    "c2b": ("c2b: blocked entity matching (not a BASELINE config; the f4 block-sparse path's input): "
            "100 blocks x 100 records per side, L ~ U{100..200} tokens from a 400-token block vocabulary"),
}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        if os.environ.get("TCUDB_BENCH_NO_CLOCKS") == "1":  # diagnosis: no sampler process
            return self
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        try:
            rows = [l.strip().split(", ") for l in open(self.f.name) if l.strip()]
        except Exception:
            rows = []
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_tables(config):
    import datagen
    A, B, agg = datagen.make_config(config)
    return A, B, agg


def gemm_traffic_from_profiles(config, elem):
    """DRAM bytes per GEMM launch from the committed ncu capture of this kernel variant."""
    p = os.path.join(ROOT, "profiles", f"gemm_traffic_{config}.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if d.get("elem", 0) == elem:
            return d.get("dram_bytes_per_launch")
    return None


def sparse_traffic_from_profiles(config, spa_mode):
    """DRAM bytes per sparse-kernel launch from the committed ncu capture (same schedule only)."""
    p = os.path.join(ROOT, "profiles", f"kernel_traffic_{config}.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if d.get("spa_mode") == spa_mode:
            return d.get("dram_bytes_per_launch")
    return None


# ---------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    A, B, agg = load_tables(args.config)
    n_tuples = len(A["k"]) + len(B["k"])
    cores = len(os.sched_getaffinity(0))
    sample, A_s, frac = bounded_sample(args.config, A)
    oracle.build()  # the checker (test infrastructure) compiled, not the product
    for _ in range(args.warmup):
        oracle.join_agg(A_s, B, agg, threads=cores)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.join_agg(A_s, B, agg, threads=cores)
        ts.append(time.perf_counter() - t0)
    step_s = statistics.mean(ts)
    # tuples/s of the full workload, extrapolated linearly in the joined pairs when sampled
    value = n_tuples / (step_s / frac)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s / frac * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": {"workload": WORKLOADS[args.config], "n_A": len(A["k"]),
                                           "n_B": len(B["k"]), "parallelism": "host cores"},
            "cpu_baseline": {"value": value, "unit": "tuples/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "context": PAPER_CONTEXT}
    print(json.dumps(line))
    return 0


def bounded_sample(config, A, shrink=1):
    """Rows of A (whole g groups) for a 10-30 s CPU sample; returns (text, A_sample, work fraction).
    shrink > 1 keeps 1/shrink of those groups (the 1-thread figure)."""
    import datagen
    if config in ("c1", "c5", "c5s") or (config == "c2" and shrink == 1):
        return f"full {config} workload", A, 1.0
    gs = np.unique(A["g"])
    keep_n = {"c3": max(1, len(gs) // 4), "c4": 64, "c4s": 64}.get(config, len(gs))
    keep_n = max(1, keep_n // shrink)
    keep = gs[:keep_n]
    sel = np.isin(A["g"], keep)
    As = datagen.Table(A["k"][sel], A["g"][sel], A["v"][sel] if A["v"] is not None else None)
    frac = sel.sum() / len(A["g"])  # join work is ~proportional to A rows for these configs
    return (f"{config}: {keep_n} of {len(gs)} A groups ({sel.sum()} A rows, {frac:.4f} of the join work), "
            f"time extrapolated linearly in J"), As, float(frac)


# ---------------------------------------------------------------------------- rooflines
_ELEM = {0: ("kind::i8 (u8/s8 -> s32)", 2.0, "TOP/s"), 1: ("kind::f16 (bf16 -> f32)", 1.0, "TFLOP/s"),
         2: ("kind::f16 (bf16 hi/lo split, fp64 sum)", 1.0, "TFLOP/s"),
         3: ("kind::mxf4 (e2m1 0/1 -> f32, unit scales)", 4.0, "TFLOP/s")}


def input_bytes(T):
    return sum(v.nbytes for v in T.values() if v is not None)


def query_roofline(st, in_bytes, peaks):
    """T_roof = max(T_tc, T_hbm) of the path the selector took.
    T_tc = the GEMM launches' ops (2·Gp·Hp·Kp summed) at the contraction dtype's measured
    peak; T_hbm = algorithmic bytes at the measured copy bandwidth: input columns read once
    + result tuples written once, + for the dense path operands written and read once and
    C written and read once (unfused)."""
    gb = 8 if st.get("_g64") else 4
    hb = 8 if st.get("_h64") else 4
    res_bytes = st["n_result"] * (gb + hb + 8)
    b = in_bytes + res_bytes
    t_tc = 0.0
    if st["path"] == 0:
        Gp, Hp = -(-st["G"] // 256) * 256, -(-st["H"] // 256) * 256
        Kp = -(-st["K"] // 128) * 128
        esz = {0: st["planes_a"] * 1.0, 1: 2.0, 2: 8.0, 3: 0.5}[st["elem"]]
        csz = {0: 8.0 if (st["kchunks"] > 1 or st["planes_a"] * st["planes_b"] > 1) else 4.0, 1: 4.0, 2: 8.0,
               3: 2.0 if st["K"] < 65536 else 4.0}[st["elem"]]
        ops_b = (Gp + Hp) * Kp * esz
        if st["existence"]:
            ops_b += (Gp + Hp) * Kp
        b += 2 * ops_b + 2 * Gp * Hp * csz + (2 * Gp * Hp * 4 if st["existence"] else 0)
        ratio = _ELEM[st["elem"]][1]
        t_tc = st["gemm_ops"] / (peaks["bf16_tflops"] * ratio * 1e12)
    t_hbm = b / (peaks["hbm_gbs"] * 1e9)
    return {"t_roof_ms": max(t_tc, t_hbm) * 1e3, "t_tc_ms": t_tc * 1e3, "t_hbm_ms": t_hbm * 1e3,
            "bytes": b, "bound": "tensor" if t_tc >= t_hbm else "hbm"}


def kernel_roofline(st, gemm_ms, kernel_ms, config, peaks):
    """Roofline of the dominant kernel (DESIGN.md §6 per-unit figures)."""
    if st["path"] == 0:
        ops = st["gemm_ops"]             # 2 * Gp * Hp * Kp per launch (SURVEY §8(d) per-unit figure)
        g_ms = statistics.mean(gemm_ms)
        achieved = ops / (g_ms * 1e-3) / 1e12
        # the contraction's own dtype peak: measured bf16 x the nominal ratio (int8 / fp8 2x, fp4 4x)
        kind, ratio, unit = _ELEM[st["elem"]]
        peak = peaks["bf16_tflops"] * ratio
        peak_sus = peaks["bf16_tflops_sustained"] * ratio
        int8_peak = peaks["bf16_tflops"] * 2.0
        # e2m1 products run on the CTA-pair kernel (cta_group::2, 256 x 240 pair tiles)
        # (the block-sparse and fused-compaction variants stay on the 1-CTA kernel)
        pair = st["elem"] == 3 and not st.get("fused_compact") and not (0 < st.get("block_active", 0) < 1)
        kname = f"k_gemm_tc2 (tcgen05 cta_group::2 {kind})" if pair else f"k_gemm_tc (tcgen05 {kind})"
        return {"bound": "tensor", "kernel": kname,
                "achieved": achieved, "peak": peak, "unit": unit,
                "frac": achieved / peak, "peak_sustained": peak_sus, "frac_of_sustained": achieved / peak_sus,
                "peak_source": f"{peaks['source']} bf16 x {ratio:g} (nominal {kind.split()[0]}/bf16 ratio)",
                "vs_int8_peak": achieved / int8_peak,
                # B200 dense nominal (bf16 2.25 PF, int8 4.5 POPS, fp4 9 PF): frac above 1 only
                # means the kernel reaches a larger share of ITS nominal than cuBLAS bf16 does
                "nominal_peak": 2250.0 * ratio, "frac_of_nominal": achieved / (2250.0 * ratio),
                "ops_per_launch": ops, "avg_launch_ms": g_ms,
                "traffic": gemm_traffic_from_profiles(config, st["elem"])}
    if st["ms_kernel"] > 0:
        # sparse path: the persistent band kernel k_spa_fused (expand into shared-memory rows +
        # ordered write) or the hash-partitioned expand; algorithmic bytes per launch
        k_ms = statistics.mean(kernel_ms)
        achieved = st["kernel_bytes"] / (k_ms * 1e-3) / 1e9
        kname = ("k_part_expand (hash-partitioned expand, one L2 reduction per joined pair)" if st["spa_mode"] == 4
                 else "k_spa_fused (band SPA: expand + ordered write)")
        return {"bound": "hbm", "kernel": kname, "achieved": achieved,
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                "peak_source": f"{peaks['source']} copy bandwidth", "bytes_per_launch": st["kernel_bytes"],
                "avg_launch_ms": k_ms, "spa_mode": {2: "count pass + band writer", 3: "one pass (look-back)",
                                                    4: "hash-partitioned",
                                                    5: "hub-band count pass + one pass (look-back)"}.get(
                    st["spa_mode"], st["spa_mode"]),
                "traffic": sparse_traffic_from_profiles(config, st["spa_mode"])}
    # sparse or reduction path without the band kernel: stage time, 16 B per joined pair
    b = st["join_pairs"] * 16.0
    g_ms = statistics.mean(gemm_ms)
    achieved = b / (max(g_ms, 1e-6) * 1e-3) / 1e9
    return {"bound": "hbm", "kernel": "sparse stage", "achieved": achieved, "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": None}


def cpu_baseline(config, A, B, agg):
    """The oracle as it stands on the host cores: median of up to 3 all-core runs of the
    bounded sample, plus a 1-thread figure on a smaller sample; both scaled to the full
    workload (linearly in the sampled A rows' share of the join work where sampled)."""
    import oracle
    cores = len(os.sched_getaffinity(0))
    n_tuples = len(A["k"]) + len(B["k"])
    sample, A_s, frac = bounded_sample(config, A)
    ts = []
    while len(ts) < 3 and sum(ts) < 20.0:
        t0 = time.perf_counter()
        oracle.join_agg(A_s, B, agg, threads=cores)
        ts.append(time.perf_counter() - t0)
    dt = statistics.median(ts) / frac
    # 1 thread: shrink the sample so the run stays ~10 s
    shrink = max(1, int(np.ceil(statistics.median(ts) * cores / 10.0)))
    s1, A_1, f1 = bounded_sample(config, A, shrink=shrink) if shrink > 1 else (sample, A_s, frac)
    t0 = time.perf_counter()
    oracle.join_agg(A_1, B, agg, threads=1)
    dt1 = (time.perf_counter() - t0) / f1
    return {"value": n_tuples / dt, "unit": "tuples/s", "cores": cores, "kind": "oracle", "sample": sample,
            "ms_per_query": dt * 1e3, "runs": len(ts), "stat": "median",
            "one_thread": {"value": n_tuples / dt1, "ms_per_query": dt1 * 1e3, "sample": s1}}


# ---------------------------------------------------------------------------- our arm
def measure(eng, torch, dev, config, steps, warmup, ws, rank, sharded, flush, stream, do_cpu, e2e_steps):
    """One config: W warm-up + K timed queries (CUDA events on the query stream, L2 flush
    between steps outside the events), dominant-kernel and query rooflines, e2e, oracle."""
    import datagen
    A, B, agg = datagen.make_config(config)
    n_tuples = len(A["k"]) + len(B["k"])
    sA, sB = (datagen.local_slice(A, ws, rank), datagen.local_slice(B, ws, rank)) if sharded else (A, B)
    to_dev = lambda T: {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in T.items() if v is not None}
    dA, dB = to_dev(sA), to_dev(sB)
    # the timed queries are the user's call (no stats: the call returns while its result write
    # runs, tcudb.h); the stage and kernel timings come from a second loop with stats
    step = lambda stats: eng.join_agg(dA, dB, agg, with_stats=stats)
    for _ in range(warmup):
        out, st = step(True)
        del out
    torch.cuda.synchronize()
    launches0 = eng.launch_count
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    gemm_ms, kernel_ms, st_last = [], [], None
    if sharded:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for i in range(steps):
        flush.fill_(i & 0xFF)                    # L2 flush between timed steps (outside the events)
        ev[i][0].record(stream)
        out = step(False)
        ev[i][1].record(stream)
        del out
    torch.cuda.synchronize()
    if sharded:
        torch.distributed.barrier()
    launches = eng.launch_count - launches0
    step_ms = [s.elapsed_time(e) for s, e in ev]
    for i in range(steps):                       # stage / kernel timings (same flush between queries)
        flush.fill_(i & 0xFF)
        out, st = step(True)
        gemm_ms.append(st["ms_gemm"] if st["path"] == 0 else st["ms_sparse"])
        kernel_ms.append(st["ms_kernel"])
        st_last = st
        del out
    torch.cuda.synchronize()
    total_ms = sum(step_ms)
    if sharded:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    # ---- e2e: host (pinned) columns -> query through the public API -> host result tuples
    e2e = None
    if e2e_steps > 0:
        pin = lambda T: {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory().numpy()
                         for k, v in T.items() if v is not None}
        hA, hB = pin(sA), pin(sB)
        h2d = sum(v.nbytes for v in hA.values()) + sum(v.nbytes for v in hB.values())
        r = eng.join_agg_host(hA, hB, agg)  # warm-up (sizes the pinned result cache)
        d2h = sum(v.nbytes for v in r.values())
        del r
        ts = []
        for _ in range(e2e_steps):
            if sharded:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = eng.join_agg_host(hA, hB, agg)
            ts.append(time.perf_counter() - t0)
            del r
        e_s = statistics.mean(ts)
        if sharded:
            tmax = torch.tensor([e_s], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
            e_s = float(tmax.item())
        e2e = {"value": n_tuples / e_s, "unit": "tuples/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_s * 1e3,
               "note": ("per rank: pinned host slices in, collective query (NCCL exchange), full result out; "
                        "max over ranks" if sharded else
                        "tcudb_join_agg_host: pinned host columns in, pinned host result tuples out")}
    if rank != 0:
        return None
    peaks = measured_peaks()
    st = dict(st_last)
    st["_g64"] = A["g"] is not None and A["g"].dtype == np.int64
    st["_h64"] = B["g"] is not None and B["g"].dtype == np.int64
    ms = total_ms / steps
    qroof = query_roofline(st, input_bytes(A) + input_bytes(B), peaks)
    qroof["frac"] = qroof["t_roof_ms"] / ms
    if config in ("c1", "c1s"):
        # latency-bound (T_roof < 1 us); a roofline fraction says nothing here
        qroof["frac"] = None
        qroof["note"] = "launch/latency-bound: T_roof < 1 us, fraction not meaningful (SURVEY 8(d) c1)"
    qroof["peak_source"] = f"{peaks['source']} (bf16 x dtype ratio, copy bandwidth)"
    if sharded:
        qroof["note"] = "single-GPU roofline of the whole query vs the N-GPU query time"
    tri = None
    if config == "c3" and not sharded:
        # c3 also names the triangle query (a9): device-timed on the symmetrised graph
        s_np, d_np = datagen.c3_graph_edges()
        S_, D_ = torch.from_numpy(s_np).to(dev), torch.from_numpy(d_np).to(dev)
        for _ in range(2):
            eng.triangle_count(S_, D_)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(5):
            t_count, t_st = eng.triangle_count(S_, D_, with_stats=True)
        e1.record(stream)
        torch.cuda.synchronize()
        tri = {"triangles": t_count, "ms": e0.elapsed_time(e1) / 5, "edges": int(len(s_np)),
               "path": "sparse wedge check" if t_st["path"] == 1 else "dense masked GEMM"}
    cpu = cpu_baseline(config, A, B, agg) if do_cpu else None
    rec = {
        "value": n_tuples * steps / (total_ms * 1e-3), "unit": "tuples/s", "ms_per_step": ms, "steps": steps,
        "dtype": ({0: "u8", 1: "bf16", 2: "bf16", 3: "e2m1"}[st["elem"]] if st["path"] == 0 else
                  ("f64" if agg == "sum" and A["v"] is not None and A["v"].dtype == np.float32 else "int64")),
        "config": {"workload": WORKLOADS[config], "n_A": len(A["k"]), "n_B": len(B["k"]),
                   "G": st["G"], "H": st["H"], "K": st["K"], "join_pairs": st["join_pairs"],
                   "result_groups": st["n_result"], "path": {0: "dense", 1: "sparse", 2: "segmented", 3: "key-partitioned"}[st["path"]],
                   "l2": "flushed (256 MiB write) between timed steps"},
        "stage_ms": {k: st[k] for k in ("ms_stats", "ms_encode", "ms_fill", "ms_gemm", "ms_sparse", "ms_compact")
                     + (("ms_comm",) if sharded else ())},
        "step_ms": [round(x, 4) for x in step_ms],
        "roofline": kernel_roofline(st, gemm_ms, kernel_ms, config, peaks),
        "query_roofline": qroof,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
    }
    if tri:
        rec["triangle_query"] = tri
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--also", default="c1,c3,c4,c5",
                    help="other configs measured in the same run (reported under 'configs'); '' for none")
    ap.add_argument("--also-steps", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--force-shard", action="store_true",
                    help="run the collective (row-sharded) path even on one rank (NCCL group of 1; test hook)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = ws > 1 or args.force_shard
    if sharded:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2112_07552_b200 import Engine

    # the collective tcudb_join_agg (NCCL inside libtcudb, collective.cu) under torchrun
    eng = Engine(local, group=torch.distributed.group.WORLD) if sharded else Engine(local)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    also = [c for c in args.also.split(",") if c and c != args.config]
    for c in also:
        if c not in WORKLOADS:
            raise SystemExit(f"unknown config {c}")
    do_cpu = not args.no_cpu_baseline and ws == 1  # the CPU baseline runs on rank 0 at N=1 only
    with ClockSampler(local) as clk:
        head = measure(eng, torch, dev, args.config, args.steps, args.warmup, ws, rank, sharded, flush, stream,
                       do_cpu, args.e2e_steps)
        others = {}
        for c in also:
            others[c] = measure(eng, torch, dev, c, min(args.steps, args.also_steps), args.warmup, ws, rank, sharded,
                                flush, stream, do_cpu, min(args.e2e_steps, 2))
    clocks = clk.summary()
    if rank != 0:
        if sharded:
            torch.distributed.destroy_process_group()
        return 0
    par = (f"row-shard x{ws} (grouped side routed by row-balanced group ranges, other side allgathered, "
           f"results allgathered; collective libtcudb call over NCCL; G/H/K/stage_ms are rank 0's local query)"
           if sharded else "single GPU")
    cfg = dict(head["config"], parallelism=par)
    line = {
        "metric": METRIC, "value": head["value"], "unit": "tuples/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": head["dtype"], "data": "synthetic",
        "config": cfg, "stage_ms": head["stage_ms"], "step_ms": head["step_ms"],
        "roofline": head["roofline"], "query_roofline": head["query_roofline"],
        "cpu_baseline": head["cpu_baseline"], "e2e": head["e2e"], "clocks": clocks,
        "gpu_launches": head["gpu_launches"],
        "selector_calibration": eng.calibration,
        "configs": {c: {k: v for k, v in r.items()} for c, r in others.items()},
        "context": PAPER_CONTEXT,
    }
    print(json.dumps(line))
    if sharded:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
