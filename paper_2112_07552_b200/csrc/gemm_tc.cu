// gemm_tc.cu — step a6: the tensor-core GEMM C = A_op · B_opᵀ on sm_100a.
//
// PAPER.md §3.1 "C = mat(A) × mat(B)^T", §3.3 the
// group-by aggregate as a product, Eq. 3 CT = 2MNK / peak.
// The paper ran WMMA/cuBLAS fp16 on Turing/Ampere; here:
//   * tcgen05.mma kind::i8 (u8/s8 -> s32, exact) or kind::f16 (bf16 -> f32),
//     issued by one thread, accumulators in TMEM (2 x 256 columns: the epilogue
//     of tile t overlaps the main loop of tile t+1);
//   * TMA 2D tile loads with 128-byte swizzle into a 4-stage mbarrier ring;
//   * persistent CTAs (grid = #SMs) walking a grouped tile order;
//   * warp roles: w0 TMA producer, w1 MMA issuer (+TMEM owner), w2-5 epilogue.
// Tile 128 x 256 x (128 bytes of K) per stage (1-CTA kernel, kind::i8 / kind::f16); the e2m1
// product runs on the CTA-pair kernel k_gemm_tc2 (cta_group::2, 256 x 240 pair tiles, each CTA
// staging 128 A rows + 120 B rows per stage), which halves B's L2 -> SM bytes per MAC.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace tcudb {
namespace {

constexpr int BM = kGemmBM, BN = kGemmBN, BKB = kGemmBKBytes;
constexpr int A_STAGE_BYTES = BM * BKB;  // 16 KB
constexpr int NUM_THREADS = 192;         // 6 warps
constexpr int TMEM_COLS = 512;           // 2 accumulators x 256 fp32/s32 columns (fp4: 2 x 240 + scales)
constexpr int GROUP_M = 16;              // tile raster: 16 M-blocks per band
#ifndef TCUDB_CMP_WARPS
#define TCUDB_CMP_WARPS 8
#endif
#ifndef TCUDB_CMP_GROUP_M
#define TCUDB_CMP_GROUP_M 2
#endif
constexpr int kCmpWarps = TCUDB_CMP_WARPS;
constexpr int kCmpGroupM = TCUDB_CMP_GROUP_M;

// Per-BN kernel geometry (BN = 256 for kind::i8 / kind::f16, 240 for kind::mxf4 so
// that two accumulators plus the block-scale columns fit the 512 TMEM columns).
template <int BN_, int KB_ = 128>
struct Geo {
  static constexpr int A_BYTES = BM * KB_;
  static constexpr int B_STAGE_BYTES = BN_ * KB_;
  static constexpr int STAGE_BYTES = A_BYTES + B_STAGE_BYTES;
  static constexpr int STAGES = KB_ == 128 ? 4 : 8;  // same ~190 KB of smem in flight
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};
constexpr int SF_COL = 480;  // fp4: scale-factor columns [480, 512): SFA at 480, SFB at 496

// Shared-memory descriptor for a K-major tile with a KB-byte swizzle (128: SWIZZLE_128B,
// 8-row atoms of 1024 B; 64: SWIZZLE_64B, 8-row atoms of 512 B).
template <int KB_>
TCUDB_DEV uint64_t sw_desc(uint32_t smem_addr) {
  if (KB_ == 128) return sw128_desc(smem_addr);
  return (uint64_t)((smem_addr & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(512 >> 4) << 32) | (1ull << 46) |
         (4ull << 61);
}

struct KParams {
  int64_t M, N;
  int tiles_m, tiles_n;
  int num_kb;        // K blocks of 128 bytes
  int kb_begin;      // first K block (elements / elems_per_kb)
  int elems_per_kb;  // 128 (i8, fp4 bytes) or 64 (bf16)
  int is_bf16;
  uint32_t idesc;
  int epi;
  void* C; int64_t ldc; int shift;
  const uint8_t* mask; int64_t ldm, mask_rows, mask_cols;
  unsigned long long* tri_out;
  int32_t* cnt_out; int64_t ldcnt;
  int group_m;       // M-blocks per raster band
  FusedCompact fc;   // fused compaction (CMP kernels only)
  // block-sparse (§8(f) f4, TCU-SpMM's zero-tile skipping P:1241-1251): per M-tile / N-tile
  // bitmaps over the absolute K-blocks (bmw 64-bit words per tile); a K-block enters the
  // product of tile (mb, nb) only when both bits are set. NULL: dense.
  const unsigned long long* bmA;
  const unsigned long long* bmB;
  int bmw;
  const int* abort_a; const int* abort_b;  // GemmArgs::abort_a / abort_b
};

// the optimistic fill failed (GemmArgs::abort_a / abort_b): every thread of every CTA sees the
// same flags, so the whole grid leaves before any barrier, TMEM allocation or cluster sync
__device__ __forceinline__ bool gemm_aborted(const KParams& p) {
  return p.abort_a && (__ldcg(p.abort_a) | __ldcg(p.abort_b)) != 0;
}

// Calls f(kb, first) for the K-blocks of tile (mb, nb) in ascending order: all of them
// (dense), or those active in both operands' block bitmaps. Returns the count.
template <typename F>
__device__ __forceinline__ int for_active_kb(const KParams& p, int mb, int nb, F&& f) {
  if (!p.bmA) {
    for (int kb = 0; kb < p.num_kb; ++kb) f(kb, kb == 0);
    return p.num_kb;
  }
  const unsigned long long* a = p.bmA + (int64_t)mb * p.bmw;
  const unsigned long long* b = p.bmB + (int64_t)nb * p.bmw;
  const int k0 = p.kb_begin, k1 = p.kb_begin + p.num_kb;
  int n = 0;
  for (int w = k0 >> 6; w <= ((k1 - 1) >> 6); ++w) {
    unsigned long long m = __ldg(a + w) & __ldg(b + w);
    if (w == (k0 >> 6) && (k0 & 63)) m &= ~0ull << (k0 & 63);
    if (w == ((k1 - 1) >> 6) && (k1 & 63)) m &= ~0ull >> (64 - (k1 & 63));
    while (m) {
      const int bit = __ffsll((long long)m) - 1;
      m &= m - 1;
      f(w * 64 + bit - k0, n == 0);
      ++n;
    }
  }
  return n;
}
__device__ __forceinline__ bool tile_active(const KParams& p, int mb, int nb) {
  if (!p.bmA) return true;
  return for_active_kb(p, mb, nb, [](int, bool) {}) > 0;
}

// Grouped raster: bands of group_m M-blocks, N-blocks swept inside a band, so a band's
// A panel stays L2-resident while B streams through once per band.
__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int group_m, int& mb, int& nb) {
  const int band = t / (group_m * tiles_n);
  const int first_m = band * group_m;
  const int gsz = min(tiles_m - first_m, group_m);
  const int r = t - band * group_m * tiles_n;
  mb = first_m + r % gsz;
  nb = r / gsz;
}

TCUDB_DEV void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
TCUDB_DEV void tmem_st_32x32b_x16(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
      "r"(v)
      : "memory");
}
TCUDB_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A·Bᵀ with e2m1 operands and UE8M0 block scales (32-element blocks) read from TMEM.
TCUDB_DEV void mma_mxf4(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t sfa,
                        uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate)
      : "memory");
}

// One W-column chunk (W = 32 or 16) of the epilogue for the row this thread owns.
template <int W, bool FP4>
__device__ __forceinline__ void epilogue_chunk(const KParams& p, const uint32_t* rr, int64_t row, int64_t col,
                                               int& nzc, long long& tri) {
  uint32_t r[W];
#pragma unroll
  for (int i = 0; i < W; ++i) r[i] = FP4 ? (uint32_t)__float2int_rn(__uint_as_float(rr[i])) : rr[i];
  if (p.epi == EPI_STORE32) {
    int4* dst = reinterpret_cast<int4*>(reinterpret_cast<uint32_t*>(p.C) + row * p.ldc + col);
#pragma unroll
    for (int i = 0; i < W / 4; ++i) dst[i] = make_int4(r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
    if (p.cnt_out) {
      const uint32_t m = (p.is_bf16 && !FP4) ? 0x7fffffffu : 0xffffffffu;  // fp32: +-0 are both zero
#pragma unroll
      for (int i = 0; i < W; ++i) nzc += (r[i] & m) != 0u;
    }
  } else if (p.epi == EPI_STORE16) {
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.C) + row * p.ldc + col);
#pragma unroll
    for (int i = 0; i < W / 8; ++i)
      dst[i] = make_uint4(r[8 * i] | (r[8 * i + 1] << 16), r[8 * i + 2] | (r[8 * i + 3] << 16),
                          r[8 * i + 4] | (r[8 * i + 5] << 16), r[8 * i + 6] | (r[8 * i + 7] << 16));
    if (p.cnt_out) {
#pragma unroll
      for (int i = 0; i < W; ++i) nzc += r[i] != 0u;
    }
  } else if (p.epi == EPI_SET64 || p.epi == EPI_ACC64) {
    longlong2* d2 = reinterpret_cast<longlong2*>(reinterpret_cast<long long*>(p.C) + row * p.ldc + col);
#pragma unroll
    for (int i = 0; i < W / 2; ++i) {
      // wrapping (mod 2^64) arithmetic: exact whenever the true sum fits int64 (guard a3)
      unsigned long long x0 = (unsigned long long)(long long)(int)r[2 * i] << p.shift;
      unsigned long long x1 = (unsigned long long)(long long)(int)r[2 * i + 1] << p.shift;
      if (p.epi == EPI_ACC64) { const longlong2 o = d2[i]; x0 += (unsigned long long)o.x; x1 += (unsigned long long)o.y; }
      d2[i] = make_longlong2((long long)x0, (long long)x1);
      if (p.cnt_out) nzc += (x0 != 0ull) + (x1 != 0ull);
    }
  } else if (p.epi == EPI_SETF64 || p.epi == EPI_ACCF64) {
    // fp32 accumulator of one K range -> fp64 C (the bf16 split's partial products are
    // accumulated in separate launches and summed here in fp64, R9)
    double2* d2 = reinterpret_cast<double2*>(reinterpret_cast<double*>(p.C) + row * p.ldc + col);
#pragma unroll
    for (int i = 0; i < W / 2; ++i) {
      double x0 = (double)__uint_as_float(r[2 * i]), x1 = (double)__uint_as_float(r[2 * i + 1]);
      if (p.epi == EPI_ACCF64) { const double2 o = d2[i]; x0 += o.x; x1 += o.y; }
      d2[i] = make_double2(x0, x1);
      if (p.cnt_out) nzc += (x0 != 0.0) + (x1 != 0.0);
    }
  } else {  // EPI_TRI
    if (row < p.mask_rows && col < p.mask_cols) {
      const uint4* m4 = reinterpret_cast<const uint4*>(p.mask + row * p.ldm + col);
#pragma unroll
      for (int q = 0; q < W / 16; ++q) {
        const uint4 ma = m4[q];
        const uint32_t mw[4] = {ma.x, ma.y, ma.z, ma.w};
#pragma unroll
        for (int i = 0; i < 16; ++i)
          tri += (long long)(int)r[16 * q + i] * (long long)((mw[i >> 2] >> (8 * (i & 3))) & 0xFF);
      }
    }
  }
}

// Epilogue for one accumulator tile: this thread owns one row (its TMEM lane) and
// the BN_ accumulator columns at taddr. Returns the row's nonzero count.
template <int BN_, bool FP4>
__device__ __forceinline__ int epilogue_rows(const KParams& p, uint32_t taddr, int64_t row, int nb, long long& tri,
                                             bool zero = false) {
  int nzc = 0;  // nonzeros of this row inside the BN_-column tile (compaction count, a8)
  // zero: a block-sparse tile with no active K-block — its zeros are written without a
  // TMEM accumulator (accumulating epilogues add nothing, so they skip it)
  if (zero && (p.epi == EPI_ACC64 || p.epi == EPI_ACCF64 || p.epi == EPI_TRI)) {
    if (p.epi == EPI_ACC64 && p.cnt_out) {
      for (int c = 0; c < BN_; ++c) nzc += reinterpret_cast<const long long*>(p.C)[row * p.ldc + (int64_t)nb * BN_ + c] != 0;
    } else if (p.epi == EPI_ACCF64 && p.cnt_out) {
      for (int c = 0; c < BN_; ++c) nzc += reinterpret_cast<const double*>(p.C)[row * p.ldc + (int64_t)nb * BN_ + c] != 0.0;
    }
    return nzc;
  }
#pragma unroll 1
  for (int c = 0; c < BN_ / 32; ++c) {
    uint32_t r[32];
    if (zero) {
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = 0u;
    } else {
      tmem_ld_32x32b_x32(taddr + c * 32, r);
      tmem_ld_wait();
    }
    epilogue_chunk<32, FP4>(p, r, row, (int64_t)nb * BN_ + c * 32, nzc, tri);
  }
  if (BN_ % 32) {
    uint32_t r[16];
    if (zero) {
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = 0u;
    } else {
      tmem_ld_32x32b_x16(taddr + (BN_ / 32) * 32, r);
      tmem_ld_wait();
    }
    epilogue_chunk<16, FP4>(p, r, row, (int64_t)nb * BN_ + (BN_ / 32) * 32, nzc, tri);
  }
  return nzc;
}

// ------------------------------------------------------------------ fused compaction (f1)
// The ordered compaction (a8) runs inside the GEMM kernel: four extra warps per CTA
// turn finished C tiles (u16, still L2-resident) into (g, h, COUNT) tuples while the
// tensor cores work on later tiles, so the result write overlaps the MMA main loop.
//   * Each epilogue warp stores its 32 rows of a tile plus their nonzero counts
//     (tcnt[nb][row]) and arrives on the tile's M-block counter; the warp completing
//     the M-block (4 x tiles_n arrivals) turns the counts into per-row offsets
//     (exclusive along N tiles, rowbase = exclusive over the 128 rows) and publishes
//     the M-block's tuple count (look-back state AGG). It never waits.
//   * Compaction warps walk the CTA's own tiles in order; for a tile of M-block mb they
//     need P(mb) = sum of the counts of M-blocks < mb, found by a decoupled look-back
//     over the AGG / INC states (every AGG comes from an epilogue warp, so the wait ends).
//     A row's tuples in the tile go to P(mb) + rowbase[row] + tcnt[nb][row], in column
//     order: the output is (g, h)-sorted exactly as the separate compaction kernel's.
constexpr int CMP_WARPS = kCmpWarps;  // groups of 4 (TCUDB build-time knob)
constexpr unsigned long long kMbAgg = 1ull << 62, kMbInc = 2ull << 62, kMbVal = (1ull << 62) - 1;

__device__ __noinline__ void mblock_finish(const KParams& p, int mb) {
  const FusedCompact& f = p.fc;
  const int lane = lane_id();
  const int64_t Mp = (int64_t)p.tiles_m * BM;
  const int64_t r0 = (int64_t)mb * BM + lane * 4;  // this lane's 4 consecutive rows
  int4 run = make_int4(0, 0, 0, 0);
  for (int nb = 0; nb < p.tiles_n; nb += 4) {
    int4 c[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      c[q] = nb + q < p.tiles_n ? __ldcg(reinterpret_cast<const int4*>(f.tcnt + (int64_t)(nb + q) * Mp + r0))
                                : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (nb + q >= p.tiles_n) break;
      __stcg(reinterpret_cast<int4*>(f.tcnt + (int64_t)(nb + q) * Mp + r0), run);
      run.x += c[q].x; run.y += c[q].y; run.z += c[q].z; run.w += c[q].w;
    }
  }
  const int tot = run.x + run.y + run.z + run.w;
  int incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int ex = incl - tot;
  __stcg(reinterpret_cast<int4*>(f.rowbase + r0),
         make_int4(ex, ex + run.x, ex + run.x + run.y, ex + run.x + run.y + run.z));
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  __threadfence();
  __syncwarp();
  if (lane == 0) atomicExch(f.mstate + mb, kMbAgg | (unsigned long long)total);
}

// P(mb) (lane 0 of a compaction warp): waits for mb's own offsets, looks back over the
// M-blocks before it, publishes INC(mb) and, for the last M-block, the result size.
__device__ __noinline__ int64_t mblock_prefix(const KParams& p, int mb) {
  volatile unsigned long long* st = p.fc.mstate;
  unsigned long long v;
  while (((v = st[mb]) >> 62) == 0) __nanosleep(200);
  int64_t acc = 0;
  for (int j = mb - 1; j >= 0;) {
    const unsigned long long w = st[j];
    const unsigned fl = (unsigned)(w >> 62);
    if (fl == 0) { __nanosleep(100); continue; }
    acc += (int64_t)(w & kMbVal);
    if (fl == 2) break;
    --j;
  }
  int64_t incl = (int64_t)(v & kMbVal);
  if ((v >> 62) == 1) {
    incl += acc;
    atomicCAS(p.fc.mstate + mb, v, kMbInc | (unsigned long long)incl);
  }
  if (mb == p.tiles_m - 1) *p.fc.total = incl;
  __threadfence();
  return acc;
}

// Compacts this warp's 32 rows of tile (mb, nb): one row at a time, 8 chunks of 32
// columns loaded before the ballots; stores are 32-wide contiguous.
template <int BN_>
__device__ __forceinline__ void compact_tile_rows(const KParams& p, int mb, int nb, int cw, int64_t P) {
  const FusedCompact& f = p.fc;
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt();
  const int64_t Mp = (int64_t)p.tiles_m * BM;
  const int64_t rw0 = (int64_t)mb * BM + cw * 32;
  if (rw0 >= f.G) return;
  const int64_t my_row = rw0 + lane;
  const int64_t my_off = P + __ldcg(f.rowbase + my_row) + __ldcg(f.tcnt + (int64_t)nb * Mp + my_row);
  const long long my_g = my_row < f.G ? __ldg(f.dict_g + my_row) : 0;
  const int64_t c0 = (int64_t)nb * BN_;
  const int64_t lim = min(f.H, c0 + (int64_t)BN_);
  const uint16_t* C = static_cast<const uint16_t*>(p.C);
  long long hv[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t col = c0 + j * 32 + lane;
    hv[j] = col < lim ? __ldg(f.dict_h + col) : 0;
  }
  const int nrows = (int)min((int64_t)32, f.G - rw0);
  constexpr int RB = 4;  // rows per batch: 32 cell loads in flight per lane before the ballots
  for (int i0 = 0; i0 < nrows; i0 += RB) {
    uint32_t e[RB][8];
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const int64_t row = rw0 + i0 + q;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t col = c0 + j * 32 + lane;
        e[q][j] = (i0 + q < nrows && col < lim) ? (uint32_t)__ldcg(C + row * p.ldc + col) : 0u;
      }
    }
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      if (i0 + q >= nrows) break;
      int64_t base = __shfl_sync(0xffffffffu, my_off, i0 + q);
      const long long gv = __shfl_sync(0xffffffffu, my_g, i0 + q);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool nz = e[q][j] != 0u;
        const uint32_t m = __ballot_sync(0xffffffffu, nz);
        if (nz) {
          const int64_t pos = base + __popc(m & lt);
          if (f.g_out_type) __stcs(static_cast<long long*>(f.out_g) + pos, gv);
          else __stcs(static_cast<int*>(f.out_g) + pos, (int)gv);
          if (f.h_out_type) __stcs(static_cast<long long*>(f.out_h) + pos, hv[j]);
          else __stcs(static_cast<int*>(f.out_h) + pos, (int)hv[j]);
          __stcs(static_cast<long long*>(f.out_agg) + pos, (long long)e[q][j]);
        }
        base += __popc(m);
      }
    }
  }
}

template <int BN_, bool FP4, int KB_, bool CMP = false>
__global__ void __launch_bounds__(CMP ? NUM_THREADS + 32 * CMP_WARPS : NUM_THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const KParams p) {
  using G = Geo<BN_, KB_>;
  constexpr int A_STAGE_BYTES = G::A_BYTES;
  constexpr int STAGES = G::STAGES;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment required by the 128B swizzle atoms.
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * G::STAGE_BYTES);
  uint64_t* full = bars;                 // [STAGES]
  uint64_t* empty = bars + STAGES;       // [STAGES]
  uint64_t* tfull = bars + 2 * STAGES;   // [2]
  uint64_t* tempty = bars + 2 * STAGES + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = warp_id(), lane = lane_id();
  const int num_tiles = p.tiles_m * p.tiles_n;
  if (gemm_aborted(p)) return;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (FP4) {
    // all block scales = 2^0 (UE8M0 0x7F): the e2m1 operands carry the exact small
    // integers themselves; written once into TMEM columns [480, 512) by the epilogue warps
    if (warp >= 2 && warp < 6) {
      const uint32_t q = (uint32_t)((warp & 3) * 32) << 16;
      tmem_st_32x32b_x16(tmem_base + q + SF_COL, 0x7F7F7F7Fu);
      tmem_st_32x32b_x16(tmem_base + q + SF_COL + 16, 0x7F7F7F7Fu);
      tmem_st_wait();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      int stage = 0; uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb; tile_coords(t, p.tiles_m, p.tiles_n, p.group_m, mb, nb);
        for_active_kb(p, mb, nb, [&](int kb, bool) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], G::STAGE_BYTES);
          const int kc = (p.kb_begin + kb) * p.elems_per_kb;
          tma_load_2d(&tmA, sA + stage * A_STAGE_BYTES, &full[stage], kc, mb * BM, pol);
          tma_load_2d(&tmB, sB + stage * G::B_STAGE_BYTES, &full[stage], kc, nb * BN_, pol);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        });
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb = 0, nb = 0;
        if (p.bmA) {
          tile_coords(t, p.tiles_m, p.tiles_n, p.group_m, mb, nb);
          if (!tile_active(p, mb, nb)) continue;  // an all-zero tile: no accumulator (epilogue writes zeros)
        }
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN_;
        for_active_kb(p, mb, nb, [&](int, bool first) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = sw_desc<KB_>(smem_u32(sA + stage * A_STAGE_BYTES));
          const uint64_t bdesc = sw_desc<KB_>(smem_u32(sB + stage * G::B_STAGE_BYTES));
#pragma unroll
          for (int kk = 0; kk < KB_ / 32; ++kk) {  // 32 bytes of K per MMA
            const uint32_t accum = (!first || kk != 0) ? 1u : 0u;
            if (FP4) mma_mxf4(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, p.idesc, tmem_base + SF_COL,
                              tmem_base + SF_COL + 16, accum);
            else if (p.is_bf16) mma_f16(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, p.idesc, accum);
            else mma_i8(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, p.idesc, accum);
          }
          mma_commit(&empty[stage]);  // frees the smem slot once these MMAs retire
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        });
        mma_commit(&tfull[acc]);      // accumulator ready for the epilogue
        acc ^= 1; if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp < 6) {
    // ===================== epilogue warps 2..5 =====================
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0; uint32_t acc_phase = 0;
    long long tri = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mb, nb; tile_coords(t, p.tiles_m, p.tiles_n, p.group_m, mb, nb);
      const int64_t row = (int64_t)mb * BM + quarter * 32 + lane;
      if (!tile_active(p, mb, nb)) {  // block-sparse: no accumulator for this tile
        const int nzc = epilogue_rows<BN_, FP4>(p, 0, row, nb, tri, true);
        if (!CMP && p.cnt_out) p.cnt_out[row * p.ldcnt + nb] = nzc;
        continue;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN_;
      const int nzc = epilogue_rows<BN_, FP4>(p, taddr, row, nb, tri);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (CMP) {
        p.fc.tcnt[(int64_t)nb * p.tiles_m * BM + row] = nzc;
        __threadfence();  // this warp's C rows and counts before its arrival
        __syncwarp();
        unsigned old = 0;
        if (lane == 0) old = atomicAdd(p.fc.mdone + mb, 1u);
        old = __shfl_sync(0xffffffffu, old, 0);
        if (old == 4u * (unsigned)p.tiles_n - 1u) {
          __threadfence();
          mblock_finish(p, mb);
        }
      } else if (p.cnt_out) {
        p.cnt_out[row * p.ldcnt + nb] = nzc;
      }
      acc ^= 1; if (acc == 0) acc_phase ^= 1;
    }
    if (p.epi == EPI_TRI) {
      tri = warp_sum(tri);
      if (lane == 0 && tri != 0) atomicAdd(p.tri_out, (unsigned long long)tri);
    }
  } else if (CMP) {
    // ===================== compaction warps 6.. (groups of 4, one tile each in turn) =====
    const int cw = (warp - 6) & 3, grp = (warp - 6) >> 2;
    constexpr int NG = CMP_WARPS / 4;
    int cached_mb = -1;
    int64_t P = 0;
    for (int t = blockIdx.x + grp * gridDim.x; t < num_tiles; t += NG * gridDim.x) {
      int mb, nb; tile_coords(t, p.tiles_m, p.tiles_n, p.group_m, mb, nb);
      if (mb != cached_mb) {
        int64_t v = 0;
        if (lane == 0) v = mblock_prefix(p, mb);
        P = __shfl_sync(0xffffffffu, v, 0);
        cached_mb = mb;
        __threadfence();
      }
      compact_tile_rows<BN_>(p, mb, nb, cw, P);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ CTA-pair kernel (cta_group::2)
// Two CTAs of a cluster share one 256 x 256 accumulator tile: each holds 128 rows
// of A and 128 rows (half of N) of B per stage; the leader's single thread issues
// tcgen05.mma.cta_group::2 (M = 256) and its commits multicast to both CTAs'
// barriers. Per SM this halves the B bytes staged per MMA compared with the
// 1-CTA 128 x 256 tile (L2 -> SM traffic per MAC drops by 1/3).
// kind::mxf4 (c2's e2m1 COUNT product): a 256 x 240 pair tile, 120 B rows per CTA (two 240-column
// accumulators + the block-scale columns fill the 512 TMEM columns, as in the 1-CTA kernel).
template <int BN_, bool FP4>
struct Geo2 {
  static constexpr int STAGES = FP4 ? 7 : 6;
  static constexpr int A_BYTES = 128 * BKB;             // 16 KB (this CTA's 128 rows of A)
  static constexpr int B_BYTES = (BN_ / 2) * BKB;       // this CTA's half of the BN_ rows of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
};

TCUDB_DEV void mma_mxf4_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t sfa,
                             uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n\t}" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate)
      : "memory");
}

template <int BN_, bool FP4>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    k_gemm_tc2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const KParams p) {
  using G2 = Geo2<BN_, FP4>;
  constexpr int STAGES2 = G2::STAGES, A2_BYTES = G2::A_BYTES, B2_BYTES = G2::B_BYTES;
  constexpr int STAGE2_BYTES = G2::STAGE_BYTES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES2 * A2_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES2 * STAGE2_BYTES);
  uint64_t* full = bars;                          // [STAGES2] (used in the leader)
  uint64_t* empty = bars + STAGES2;               // [STAGES2] (each CTA)
  uint64_t* tfull = bars + 2 * STAGES2;           // [2]       (each CTA)
  uint64_t* tempty = bars + 2 * STAGES2 + 2;      // [2]       (used in the leader: 8 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES2 + 4);

  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
  const int num_tiles = p.tiles_m * p.tiles_n;  // pair tiles (256 x BN_)
  if (gemm_aborted(p)) return;  // both CTAs of the pair read the same flags

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES2; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 8); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (FP4) {
    // unit block scales (UE8M0 0x7F) in both CTAs' scale columns [480, 512), all 128 lanes:
    // whichever lanes / columns the pair MMA reads for SFA and SFB hold 2^0
    if (warp >= 2 && warp < 6) {
      const uint32_t q = (uint32_t)((warp & 3) * 32) << 16;
      tmem_st_32x32b_x16(tmem_base + q + SF_COL, 0x7F7F7F7Fu);
      tmem_st_32x32b_x16(tmem_base + q + SF_COL + 16, 0x7F7F7F7Fu);
      tmem_st_wait();
    }
    tc_fence_before();
  }
  __syncwarp();
  cluster_sync();  // barriers (and the scale columns) of both CTAs initialised before any remote arrive / MMA
  tc_fence_after();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();
      const uint32_t leader_full = mapa_shared(smem_u32(full), 0);
      int stage = 0; uint32_t phase = 0;
      for (int t = cid; t < num_tiles; t += ncl) {
        int mb, nb; tile_coords(t, p.tiles_m, p.tiles_n, p.group_m, mb, nb);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          // Only the leader arrives (expecting both CTAs' bytes); the peer's TMA bytes
          // complete_tx on the leader's barrier. The peer cannot reach the next phase of
          // this stage before the MMA consumed it (it waits on its own empty[stage]).
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * STAGE2_BYTES);
          const int kc = (p.kb_begin + kb) * p.elems_per_kb;
          tma_load_2d_pair(&tmA, sA + stage * A2_BYTES, leader_full + 8 * stage, kc, mb * 256 + rank * 128, pol);
          tma_load_2d_pair(&tmB, sB + stage * B2_BYTES, leader_full + 8 * stage, kc, nb * BN_ + rank * (BN_ / 2), pol);
          if (++stage == STAGES2) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int t = cid; t < num_tiles; t += ncl) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN_;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = sw128_desc(smem_u32(sA + stage * A2_BYTES));
          const uint64_t bdesc = sw128_desc(smem_u32(sB + stage * B2_BYTES));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t accum = (kb | kk) != 0;
            if (FP4) mma_mxf4_pair(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, p.idesc, tmem_base + SF_COL,
                                   tmem_base + SF_COL + 16, accum);
            else if (p.is_bf16) mma_f16_pair(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, p.idesc, accum);
            else mma_i8_pair(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, p.idesc, accum);
          }
          mma_commit_pair(&empty[stage], 0x3);  // frees this stage in both CTAs
          if (++stage == STAGES2) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair(&tfull[acc], 0x3);      // both CTAs' accumulator halves ready
        acc ^= 1; if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    const int quarter = warp & 3;
    const uint32_t leader_tempty = mapa_shared(smem_u32(tempty), 0);
    int acc = 0; uint32_t acc_phase = 0;
    long long tri = 0;
    for (int t = cid; t < num_tiles; t += ncl) {
      int mb, nb; tile_coords(t, p.tiles_m, p.tiles_n, p.group_m, mb, nb);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t row = (int64_t)mb * 256 + rank * 128 + quarter * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN_;
      const int nzc = epilogue_rows<BN_, FP4>(p, taddr, row, nb, tri);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&tempty[acc]);
        else mbar_arrive_cluster(leader_tempty + 8 * acc);
      }
      if (p.cnt_out) p.cnt_out[row * p.ldcnt + nb] = nzc;
      acc ^= 1; if (acc == 0) acc_phase ^= 1;
    }
    if (p.epi == EPI_TRI) {
      tri = warp_sum(tri);
      if (lane == 0 && tri != 0) atomicAdd(p.tri_out, (unsigned long long)tri);
    }
  }

  tc_fence_before();
  __syncwarp();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    tmem_dealloc_pair(tmem_base, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2D tensor map: box = kb_bytes of K x box_rows rows, swizzle matching kb_bytes (128 or 64).
bool make_map(CUtensorMap* m, const void* base, int elem, int64_t rows, int64_t cols_elems, int64_t ld_elems,
              int box_rows, int kb_bytes = BKB) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  const int esz = elem == ELEM_BF16 ? 2 : 1;
  cuuint64_t dims[2] = {(cuuint64_t)cols_elems, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * esz)};
  cuuint32_t box[2] = {(cuuint32_t)(kb_bytes / esz), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, elem == ELEM_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   kb_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// K bytes per pipeline stage: 128 (4 stages) or 64 (8 stages; TCUDB_GEMM_KB=64).
int pick_kb() {
  static const int kb = (getenv("TCUDB_GEMM_KB") && atoi(getenv("TCUDB_GEMM_KB")) == 64) ? 64 : 128;
  return kb;
}

}  // namespace

// Raster band height: the band's A panel (rows x K bytes) should stay L2-resident while
// B streams (126 MB L2; budget 48 MB). TCUDB_GEMM_GROUP_M overrides (experiments).
int pick_group_m(int tiles_m, int64_t rows_per_mblock, int64_t k_bytes) {
  static const int env = getenv("TCUDB_GEMM_GROUP_M") ? atoi(getenv("TCUDB_GEMM_GROUP_M")) : 0;
  int64_t g = env > 0 ? env : (int64_t)(48e6 / (double)(rows_per_mblock * (k_bytes > 0 ? k_bytes : 1)));
  if (g < 1) g = 1;
  if (g > tiles_m) g = tiles_m;
  return (int)g;
}

// Builds the tensor maps and launches the 1-CTA kernel for the chosen stage width.
template <int BN_, bool FP4, bool CMP = false>
cudaError_t run_1cta(const GemmArgs& a, const KParams& p, int map_elem, int kb, cudaStream_t s, int64_t* launches) {
  cudaError_t e = set_func_attr(k_gemm_tc<BN_, FP4, 128, CMP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)Geo<BN_, 128>::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  e = set_func_attr(k_gemm_tc<BN_, FP4, 64, CMP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)Geo<BN_, 64>::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  constexpr int NT_ = CMP ? NUM_THREADS + 32 * CMP_WARPS : NUM_THREADS;
  const int64_t kcols = a.k_begin + a.k_len;
  CUtensorMap mA, mB;
  if (!make_map(&mA, a.A, map_elem, a.M, kcols, a.lda, BM, kb) ||
      !make_map(&mB, a.B, map_elem, a.N, kcols, a.ldb, BN_, kb))
    return cudaErrorInvalidValue;
  const int tiles = p.tiles_m * p.tiles_n;
  const int grid = tiles < kNumSMs ? tiles : kNumSMs;
  if (kb == 64) k_gemm_tc<BN_, FP4, 64, CMP><<<grid, NT_, Geo<BN_, 64>::SMEM_BYTES, s>>>(mA, mB, p);
  else k_gemm_tc<BN_, FP4, 128, CMP><<<grid, NT_, Geo<BN_, 128>::SMEM_BYTES, s>>>(mA, mB, p);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// kind::mxf4 path: e2m1 operands, two elements per byte. k_begin / k_len / lda / ldb
// are in BYTES; the N tile is 240 (two 240-column accumulators + block scales in TMEM),
// tiles_n = ceil(N / 240) with TMA zero-filling the rows past N; C must hold
// ceil(N/240)*240 columns (ldc).
cudaError_t launch_gemm_fp4(const GemmArgs& a, cudaStream_t s, int64_t* launches) {
  constexpr int BNF = kGemmBNFp4;
  if (a.M <= 0 || a.N <= 0 || a.k_len <= 0) return cudaSuccess;
  if (a.M % BM || a.k_len % BKB || a.k_begin % BKB || a.lda % 16 || a.ldb % 16 ||
      (a.epi != EPI_STORE32 && a.epi != EPI_STORE16) || (a.cmp && a.epi != EPI_STORE16))
    return cudaErrorInvalidValue;
  const int64_t tiles_n = (a.N + BNF - 1) / BNF;
  if (a.ldc < tiles_n * BNF) return cudaErrorInvalidValue;
  const int kb = a.bmA ? BKB : pick_kb();  // bitmaps are over 128-byte K-blocks
  KParams p{};
  p.M = a.M; p.N = a.N;
  p.tiles_m = (int)(a.M / BM); p.tiles_n = (int)tiles_n;
  p.elems_per_kb = kb;  // bytes
  p.num_kb = (int)(a.k_len / kb);
  p.kb_begin = (int)(a.k_begin / kb);
  p.is_bf16 = 0;
  // Block-scaled instruction descriptor (kind::mxf4): A/B format E2M1 = 1 (bits 7-9, 10-12),
  // K-major, N >> 3 (bits 17-22), scale format UE8M0 (bit 23), M >> 4 (bits 24-28),
  // scale-factor ids 0, K = 64 per MMA (bit 31 = 0).
  uint32_t idesc = (1u << 7) | (1u << 10) | ((uint32_t)(BNF >> 3) << 17) | (1u << 23) | ((uint32_t)(BM >> 4) << 24);
  p.idesc = idesc;
  p.epi = a.epi; p.C = a.C; p.ldc = a.ldc; p.shift = 0;
  p.cnt_out = a.cnt_out; p.ldcnt = a.ldcnt;
  p.group_m = pick_group_m(p.tiles_m, BM, a.k_len);
  p.bmA = a.bmA; p.bmB = a.bmB; p.bmw = a.bmw;
  p.abort_a = a.abort_a; p.abort_b = a.abort_b ? a.abort_b : a.abort_a;
  if (a.cmp && a.bmA) return cudaErrorInvalidValue;  // fused compaction needs every tile's epilogue
  // CTA-pair kernel (cta_group::2, 256 x 240 pair tiles): each SM stages 128 A rows + 120 B rows
  // per K-block instead of 128 + 240 (a third less L2 -> SM traffic per MAC). Default when M
  // splits into 256-row pair tiles; TCUDB_GEMM_PAIR4=0 keeps the 1-CTA kernel.
  static const bool no_pair4 = getenv("TCUDB_GEMM_PAIR4") && getenv("TCUDB_GEMM_PAIR4")[0] == '0';
  if (!no_pair4 && !a.cmp && !a.bmA && a.M % 256 == 0 && kb == BKB) {
    using G2 = Geo2<BNF, true>;
    cudaError_t e = set_func_attr(k_gemm_tc2<BNF, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)G2::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    p.tiles_m = (int)(a.M / 256);
    p.idesc = (idesc & ~(0x1Fu << 24)) | ((uint32_t)(256 >> 4) << 24);
    p.group_m = pick_group_m(p.tiles_m, 256, a.k_len);
    const int64_t kcols = a.k_begin + a.k_len;
    CUtensorMap mA, mB;
    if (!make_map(&mA, a.A, ELEM_I8, a.M, kcols, a.lda, 128) ||
        !make_map(&mB, a.B, ELEM_I8, a.N, kcols, a.ldb, BNF / 2))
      return cudaErrorInvalidValue;
    const int tiles = p.tiles_m * p.tiles_n;
    const int grid = 2 * (tiles < kNumSMs / 2 ? tiles : kNumSMs / 2);
    k_gemm_tc2<BNF, true><<<grid, NUM_THREADS, G2::SMEM_BYTES, s>>>(mA, mB, p);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  if (a.cmp) {
    // M-blocks must complete early for their compaction to overlap later tiles: bands of
    // 2 M-blocks (measured best of 1..40 on c2)
    if (!getenv("TCUDB_GEMM_GROUP_M")) p.group_m = p.tiles_m < kCmpGroupM ? p.tiles_m : kCmpGroupM;
    p.fc = *static_cast<const FusedCompact*>(a.cmp);
    p.cnt_out = p.fc.tcnt;  // non-null: the epilogue counts nonzeros (stored as tcnt[nb][row])
    return run_1cta<BNF, true, true>(a, p, ELEM_I8, kb, s, launches);
  }
  return run_1cta<BNF, true>(a, p, ELEM_I8, kb, s, launches);
}

cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.elem == ELEM_FP4) return launch_gemm_fp4(a, s, launches);
  const int esz = a.elem == ELEM_BF16 ? 2 : 1;
  if (a.M <= 0 || a.N <= 0 || a.k_len <= 0) return cudaSuccess;
  if (a.M % BM || a.N % BN || (a.k_len * esz) % BKB || (a.k_begin * esz) % BKB) return cudaErrorInvalidValue;
  if ((a.lda * esz) % 16 || (a.ldb * esz) % 16) return cudaErrorInvalidValue;
  cudaError_t e = set_func_attr(k_gemm_tc2<BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)Geo2<BN, false>::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  // Kernel choice: the 1-CTA 128x256 kernel is the default (measured faster on c2: 1.31 vs
  // 1.40 ms; both MMA-bound at ~65-70 % tensor-pipe activity). TCUDB_GEMM_PAIR=1 selects the
  // CTA-pair (cta_group::2) kernel when M splits into 256-row pair tiles.
  static const bool want_pair = getenv("TCUDB_GEMM_PAIR") && getenv("TCUDB_GEMM_PAIR")[0] == '1';
  const bool pair = want_pair && a.M % 256 == 0 && !a.bmA;
  const int kb = (pair || a.bmA) ? BKB : pick_kb();  // bitmaps are over 128-byte K-blocks
  KParams p{};
  p.M = a.M; p.N = a.N;
  p.tiles_m = (int)(a.M / (pair ? 256 : BM)); p.tiles_n = (int)(a.N / BN);
  p.elems_per_kb = kb / esz;
  p.num_kb = (int)(a.k_len / p.elems_per_kb);
  p.kb_begin = (int)(a.k_begin / p.elems_per_kb);
  p.is_bf16 = a.elem == ELEM_BF16;
  // Instruction descriptor: D format (bits 4-5: 1 F32, 2 S32), A/B format (bits 7-9, 10-12:
  // kind::i8 0 U8 / 1 S8; kind::f16 1 BF16), K-major A and B (bits 15, 16 = 0),
  // N >> 3 (bits 17-22), M >> 4 (bits 24-28).
  uint32_t idesc = 0;
  if (p.is_bf16) idesc |= (1u << 4) | (1u << 7) | (1u << 10);
  else idesc |= (2u << 4) | ((uint32_t)(a.a_signed != 0) << 7) | ((uint32_t)(a.b_signed != 0) << 10);
  idesc |= (uint32_t)(BN >> 3) << 17;
  idesc |= (uint32_t)((pair ? 256 : BM) >> 4) << 24;
  p.idesc = idesc;
  p.epi = a.epi; p.C = a.C; p.ldc = a.ldc; p.shift = a.shift;
  p.mask = a.mask; p.ldm = a.ldm; p.mask_rows = a.mask_rows; p.mask_cols = a.mask_cols; p.tri_out = a.tri_out;
  p.cnt_out = a.cnt_out; p.ldcnt = a.ldcnt;
  p.group_m = pick_group_m(p.tiles_m, pair ? 256 : BM, a.k_len * esz);
  p.bmA = a.bmA; p.bmB = a.bmB; p.bmw = a.bmw;
  p.abort_a = a.abort_a; p.abort_b = a.abort_b ? a.abort_b : a.abort_a;
  if (!pair) return run_1cta<BN, false>(a, p, a.elem, kb, s, launches);
  const int64_t kcols = a.k_begin + a.k_len;
  CUtensorMap mA, mB;
  if (!make_map(&mA, a.A, a.elem, a.M, kcols, a.lda, 128) || !make_map(&mB, a.B, a.elem, a.N, kcols, a.ldb, 128))
    return cudaErrorInvalidValue;
  const int tiles = p.tiles_m * p.tiles_n;
  const int grid = 2 * (tiles < kNumSMs / 2 ? tiles : kNumSMs / 2);
  k_gemm_tc2<BN, false><<<grid, NUM_THREADS, Geo2<BN, false>::SMEM_BYTES, s>>>(mA, mB, p);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
