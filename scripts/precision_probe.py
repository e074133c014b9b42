"""Accumulation-precision probe of the tcgen05 GEMM kinds (the float-SUM guard, DESIGN R9).

Measures on the B200, against exact fp64 references:
  1. kind::f16 (bf16 in, fp32 TMEM accumulate): max |C - exact| / S_abs vs K on signed
     N(0,1) bf16-exact operands, next to two emulations of the accumulation order
     (per-MMA step of 16 products: exact step sum, then fp32 round-to-nearest [rn16] or
     round-toward-zero [rz16] into the accumulator);
  2. the hi/lo split of fp32 values (x = hi + lo, hi = bf16(x), lo = bf16(x - hi)) as ONE
     GEMM over [hi|hi|lo|lo]·[hi|lo|hi|lo] (round-1 layout) vs two GEMMs (hi·hi, and the
     three correction products) summed in fp64 (round-2 layout);
  3. kind::mxf4 (e2m1 0/1, fp32 accumulate): large odd integer sums (> 2^20), exact or not;
  4. groups of few products: the two-way split (residual 2^-16 |x|) vs the three-way split
     (hi, mid, lo; residual 2^-24 |x|) against the 1e-5 S_abs floor of R9.

usage: python scripts/precision_probe.py [out.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2112_07552_b200 import Engine  # noqa: E402


def exact(A, B, chunk=8192):
    """fp64 A·Bᵀ (bf16/fp32 products are exact in fp64; fp64 sums ~1e-16 relative)."""
    C = torch.zeros(A.shape[0], B.shape[0], dtype=torch.float64, device=A.device)
    for k0 in range(0, A.shape[1], chunk):
        C += A[:, k0:k0 + chunk].double() @ B[:, k0:k0 + chunk].double().T
    return C


def emulate(A, B, mode, step=16):
    """fp32 accumulator updated once per MMA step of `step` products (step sum exact)."""
    Ad, Bd = A.double(), B.double()
    acc = torch.zeros(A.shape[0], B.shape[0], dtype=torch.float32, device=A.device)
    for k0 in range(0, A.shape[1], step):
        s = acc.double() + Ad[:, k0:k0 + step] @ Bd[:, k0:k0 + step].T
        f = s.float()
        if mode == "rz16":
            over = f.double().abs() > s.abs()
            f = torch.where(over, torch.nextafter(f, torch.zeros_like(f)), f)
        acc = f
    return acc.double()


def split(x):
    hi = x.to(torch.bfloat16)
    lo = (x - hi.float()).to(torch.bfloat16)
    return hi, lo


def split3(x):
    hi = x.to(torch.bfloat16)
    mid = (x - hi.float()).to(torch.bfloat16)
    lo = (x - hi.float() - mid.float()).to(torch.bfloat16)
    return hi, mid, lo


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    eng = Engine(0)
    g = torch.Generator(device="cuda").manual_seed(2112)
    M, N = 128, 256
    rep = {"bf16_exact_inputs": [], "split": [], "split3_few_products": [], "e2m1": []}
    for K in (1024, 4096, 8192, 32768):
        A = torch.randn(M, K, generator=g, device="cuda").to(torch.bfloat16)
        B = torch.randn(N, K, generator=g, device="cuda").to(torch.bfloat16)
        ex = exact(A, B)
        sabs = exact(A.abs(), B.abs())
        C = eng.gemm(A, B).double()
        row = {"K": K, "measured": ((C - ex).abs() / sabs).max().item()}
        if K <= 8192:
            for mode in ("rn16", "rz16"):
                em = emulate(A, B, mode)
                row[mode] = ((em - ex).abs() / sabs).max().item()
                row[mode + "_bitwise_equal_frac"] = (em == C).double().mean().item()
        rep["bf16_exact_inputs"].append(row)
        print("bf16", row, flush=True)
    for K in (1024, 3000 // 64 * 64, 8192):
        a = torch.randn(M, K, generator=g, device="cuda")
        b = torch.randn(N, K, generator=g, device="cuda")
        ex = exact(a, b)
        sabs = exact(a.abs(), b.abs())
        ah, al = split(a)
        bh, bl = split(b)
        one = eng.gemm(torch.cat([ah, ah, al, al], 1).contiguous(), torch.cat([bh, bl, bh, bl], 1).contiguous())
        hh = eng.gemm(ah, bh).double()
        corr = eng.gemm(torch.cat([ah, al, al], 1).contiguous(), torch.cat([bl, bh, bl], 1).contiguous()).double()
        two = hh + corr
        resid = exact(torch.cat([ah, ah, al, al], 1), torch.cat([bh, bl, bh, bl], 1))  # exact split products
        row = {"K": K,
               "one_gemm": ((one.double() - ex).abs() / sabs).max().item(),
               "two_gemms_f64": ((two - ex).abs() / sabs).max().item(),
               "split_residual_only": ((resid - ex).abs() / sabs).max().item(),
               "hh_accumulation_only": ((hh - exact(ah, bh)).abs() / sabs).max().item()}
        rep["split"].append(row)
        print("split", row, flush=True)
    # groups of FEW products (the fuzz sweep's failing shape): U(-4, 4) values, ~2-3 nonzero
    # products per output; two-way (hi, lo: 4 products) vs three-way (hi, mid, lo: 6 products)
    # split, each as hi·hi + corrections summed in fp64 (the library's layout per round)
    for K, dens in ((64, 0.2), (64, 0.05), (1024, 0.003), (8192, 0.0004)):
        mask_a = torch.rand(M, K, generator=g, device="cuda") < dens ** 0.5
        mask_b = torch.rand(N, K, generator=g, device="cuda") < dens ** 0.5
        a = (torch.rand(M, K, generator=g, device="cuda") * 8 - 4) * mask_a
        b = (torch.rand(N, K, generator=g, device="cuda") * 8 - 4) * mask_b
        ex = exact(a, b)
        sabs = exact(a.abs(), b.abs())
        live = sabs > 0
        ah, al = split(a)
        bh, bl = split(b)
        two = eng.gemm(ah, bh).double() + eng.gemm(torch.cat([ah, al, al], 1).contiguous(),
                                                   torch.cat([bl, bh, bl], 1).contiguous()).double()
        a3, b3 = split3(a), split3(b)
        three = eng.gemm(a3[0], b3[0]).double() + eng.gemm(
            torch.cat([a3[0], a3[0], a3[1], a3[1], a3[2]], 1).contiguous(),
            torch.cat([b3[1], b3[2], b3[0], b3[1], b3[0]], 1).contiguous()).double()
        e2 = ((two - ex).abs() / sabs)[live]
        e3 = ((three - ex).abs() / sabs)[live]
        row = {"K": K, "density": dens, "groups": int(live.sum().item()),
               "two_way_max_err_over_sabs": e2.max().item(), "three_way_max_err_over_sabs": e3.max().item(),
               "two_way_over_1e-5": int((e2 > 1e-5).sum().item()), "three_way_over_1e-5": int((e3 > 1e-5).sum().item())}
        rep["split3_few_products"].append(row)
        print("split3", row, flush=True)
    # e2m1 0/1 operands, sums far above 2^20 with odd values: exact iff fp32 accumulation
    # keeps every integer < 2^24
    for K, dens in ((1 << 21, 0.5), ((1 << 22) - 256, 0.75), ((1 << 24) - 256, 0.9)):
        Mx, Nx = 128, 240
        A = (torch.rand(Mx, K, generator=g, device="cuda") < dens).to(torch.uint8)
        B = (torch.rand(Nx, K, generator=g, device="cuda") < dens).to(torch.uint8)
        pack = lambda X: ((X * 2)[:, 0::2] | ((X * 2)[:, 1::2] << 4)).contiguous()  # noqa: E731
        C = eng.gemm(pack(A), pack(B), fp4=True).long()
        ref = torch.zeros(Mx, Nx, dtype=torch.int64, device="cuda")
        for k0 in range(0, K, 1 << 16):
            ref += (A[:, k0:k0 + (1 << 16)].double() @ B[:, k0:k0 + (1 << 16)].double().T).long()
        row = {"K": K, "density": dens, "min_sum": ref.min().item(), "max_sum": ref.max().item(),
               "odd_frac": (ref % 2).double().mean().item(), "mismatches": int((C != ref).sum().item()),
               "max_abs_err": int((C - ref).abs().max().item())}
        rep["e2m1"].append(row)
        print("e2m1", row, flush=True)
        del A, B
        torch.cuda.empty_cache()
    if out:
        with open(out, "w") as f:
            json.dump(rep, f, indent=1)
    eng.close()


if __name__ == "__main__":
    main()
