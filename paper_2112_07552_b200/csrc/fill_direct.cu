// fill_direct.cu — steps a2 + a5 fused for direct-offset dictionaries (the c4 class:
// dense float SUM over int32 key / group columns whose value spans fit shared memory).
//
// PAPER.md §4.2.2: the data transformation is "linear in records"; the
// fill writes mat(A)[g][k] = v (§3.3) pre-aggregated per cell (reading R5).
// The general path writes an int32 code per tuple and column (8 B per tuple) and the
// fill reads them back; here the per-tuple codes are never materialized:
//   k_direct_count  one pass over (k, g) of one side: per-key counts over the key span and
//                   group presence flags (shared-memory privatized), i.e. the direct
//                   dictionaries' marks (a2) and cntA / cntB for J (a4) at once;
//   k_dt_bin        one pass over (k, g, v): codes looked up from the dictionaries' code
//                   tables (u16 copies in shared memory), every tuple becomes an entry
//                   (cell-in-tile | value) binned by operand tile — batches are counting-
//                   sorted in shared memory and each tile's run is reserved with one atomic,
//                   so the entries leave as coalesced runs; no histogram pre-pass: each tile
//                   owns a region of `cells` entries (more would be a duplicate cell);
//   k_dt_tile       one CTA per tile builds the tile in shared memory (occupancy bits
//                   detect a duplicate cell -> fs->overflow; the caller then takes the
//                   scratch path) and writes it coalesced, zeros included — bf16 cells, or
//                   fp32 cells written as the three-way split (R8/R9: hi = bf16(x),
//                   mid = bf16(x - hi), lo = bf16(x - hi - mid)) — plus, optionally, the e2m1 existence pattern (R3).
// Bytes per tuple: 8 (count) + 12 read + 4|8 written (bin) + 4|8 read + cells written (tile).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <type_traits>
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

// ------------------------------------------------------------------ a2: counts + marks
constexpr int kCntThreads = 1024;

__global__ void __launch_bounds__(kCntThreads) k_direct_count(const int32_t* __restrict__ key,
                                                               const int32_t* __restrict__ grp, int64_t n, int kmin,
                                                               int kspan, int gmin, int gspan,
                                                               int32_t* __restrict__ cnt_span,
                                                               uint8_t* __restrict__ kflag,
                                                               uint8_t* __restrict__ gflag) {
  extern __shared__ __align__(16) int32_t s_cnt[];
  uint8_t* s_gf = reinterpret_cast<uint8_t*>(s_cnt + kspan);
  for (int i = threadIdx.x; i < kspan; i += blockDim.x) s_cnt[i] = 0;
  for (int i = threadIdx.x; i < gspan; i += blockDim.x) s_gf[i] = 0;
  __syncthreads();
  const int64_t n4 = n / 4;
  const int4* k4 = reinterpret_cast<const int4*>(key);
  const int4* g4 = reinterpret_cast<const int4*>(grp);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto one = [&](int k, int g) {
    atomicAdd(s_cnt + (k - kmin), 1);
    s_gf[g - gmin] = 1;
  };
  constexpr int U = 4;  // 16-byte vectors in flight per column and thread
  for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v0 < n4; v0 += U * stride) {
    int4 ka[U], ga[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = v0 + u * stride;
      if (v < n4) { ka[u] = __ldcs(k4 + v); ga[u] = __ldcs(g4 + v); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (v0 + u * stride >= n4) break;
      one(ka[u].x, ga[u].x); one(ka[u].y, ga[u].y); one(ka[u].z, ga[u].z); one(ka[u].w, ga[u].w);
    }
  }
  for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) one(key[i], grp[i]);
  __syncthreads();
  for (int i = threadIdx.x; i < kspan; i += blockDim.x) {
    const int c = s_cnt[i];
    if (c) {
      atomicAdd(cnt_span + i, c);
      if (!kflag[i]) kflag[i] = 1;
    }
  }
  for (int i = threadIdx.x; i < gspan; i += blockDim.x)
    if (s_gf[i] && !gflag[i]) gflag[i] = 1;
}

// ------------------------------------------------------------------ a5: bin + tile
constexpr int kDtThreads = 512;
constexpr int kDtTileThreads = 1024;
constexpr int kDtMaxTiles = 4096;
template <bool SPLIT> struct Dt {
  using Ent = typename std::conditional<SPLIT, unsigned long long, uint32_t>::type;
  static constexpr int kCells = SPLIT ? 32768 : 65536;  // tile cells (fp32 / bf16 in shared memory)
  static constexpr int kPer = SPLIT ? 8 : 16;           // tuples per thread and batch
  static constexpr int kBatch = kPer * kDtThreads;
};
struct DtPlan {
  int KW = 0, kw_bits = 0, R = 0, r_bits = 0, nkt = 0, ntiles = 0;
  int64_t cap = 0;  // entries per tile region
  size_t off_ent = 0, bytes = 0;
};
inline size_t al256(size_t x) { return (x + 255) / 256 * 256; }
DtPlan dt_plan(int64_t rows, int64_t Kp, bool split) {
  DtPlan p;
  if (Kp <= 0 || Kp % 128 || rows <= 0 || rows % 8) return p;
  const int cells = split ? Dt<true>::kCells : Dt<false>::kCells;
  int KW = 128, kb = 7;
  while (KW < Kp && KW < 8192) { KW *= 2; ++kb; }
  const int R = cells / KW;
  const int64_t nkt = (Kp + KW - 1) / KW, nrt = (rows + R - 1) / R;
  if (nkt * nrt > kDtMaxTiles) return p;
  p.KW = KW; p.kw_bits = kb; p.R = R; p.nkt = (int)nkt; p.ntiles = (int)(nkt * nrt);
  while ((1 << p.r_bits) < R) ++p.r_bits;  // R = cells / KW: a power of two
  p.cap = cells;
  p.off_ent = al256((size_t)p.ntiles * 4);
  p.bytes = p.off_ent + (size_t)p.ntiles * cells * (split ? 8 : 4);
  return p;
}

template <bool SPLIT>
__global__ void __launch_bounds__(kDtThreads, 2) k_dt_bin(const DtFill f, const DtPlan p,
                                                                       int32_t* __restrict__ cursor,
                                                                       typename Dt<SPLIT>::Ent* __restrict__ ent,
                                                                       int64_t chunk) {
  using Ent = typename Dt<SPLIT>::Ent;
  constexpr int kBatch = Dt<SPLIT>::kBatch, kPer = Dt<SPLIT>::kPer;
  extern __shared__ __align__(16) uint8_t smem[];
  Ent* stage = reinterpret_cast<Ent*>(smem);                                       // [kBatch]
  uint32_t* sdst = reinterpret_cast<uint32_t*>(stage + kBatch);                  // [kBatch] entry index
  int* cnt = reinterpret_cast<int*>(sdst + kBatch);                               // [ntiles]
  int* start = cnt + p.ntiles;                                                     // [ntiles]
  int* gpos = start + p.ntiles;                                                    // [ntiles]
  uint16_t* tk = reinterpret_cast<uint16_t*>(gpos + p.ntiles);                    // [kspan] key codes
  uint16_t* tg = tk + f.kspan;                                                     // [gspan] row codes
  __shared__ int wsum[kDtThreads / 32];
  __shared__ int s_total;
  for (int i = threadIdx.x; i < f.kspan; i += blockDim.x) tk[i] = (uint16_t)__ldg(f.kcode + i);  // -1 -> 0xFFFF
  for (int i = threadIdx.x; i < f.gspan; i += blockDim.x) tg[i] = (uint16_t)__ldg(f.gcode + i);
  for (int t = threadIdx.x; t < p.ntiles; t += blockDim.x) cnt[t] = 0;
  __syncthreads();
  const int kmin = (int)f.kmin, gmin = (int)f.gmin;
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(f.n, lo + chunk);
  const int per = (p.ntiles + kDtThreads - 1) / kDtThreads;  // tile counters per thread in the scan
  int ovf = 0;
  for (int64_t b0 = lo; b0 < hi; b0 += kBatch) {
    // ---- 1: load, look the codes up, rank inside the tile
    constexpr int U = kPer / 4;
    Ent e[kPer];
    uint32_t tr[kPer];  // tile << 16 | rank inside the tile's batch run (~0u: no entry)
    // loads in two halves of U/2 vectors per column (volatile 16-byte loads stay batched: one
    // latency per half; all of them at once would exceed the 64 registers of 2 CTAs x 512)
    const bool full = b0 + kBatch <= hi;
    constexpr int UH = U / 2;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      int4 k4[UH], g4[UH];
      uint4 v4[UH];
      if (full) {
#pragma unroll
        for (int uu = 0; uu < UH; ++uu) {
          const int64_t i = b0 + ((int64_t)(h * UH + uu) * kDtThreads + threadIdx.x) * 4;
          k4[uu] = ld_stream_v4(f.key + i);
          g4[uu] = ld_stream_v4(f.grp + i);
          if (f.val) { const int4 t4 = ld_stream_v4(f.val + i); v4[uu] = make_uint4(t4.x, t4.y, t4.z, t4.w); }
          else v4[uu] = make_uint4(0x3F800000u, 0x3F800000u, 0x3F800000u, 0x3F800000u);  // absent value = 1.0
        }
      } else {
#pragma unroll
        for (int uu = 0; uu < UH; ++uu) {
          const int64_t i = b0 + ((int64_t)(h * UH + uu) * kDtThreads + threadIdx.x) * 4;
          int kx[4], gx[4];
          uint32_t vb[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool ok = i + q < hi;
            kx[q] = ok ? f.key[i + q] : (int)((unsigned)kmin + (unsigned)f.kspan);  // past the span: no entry
            gx[q] = ok ? f.grp[i + q] : gmin;
            vb[q] = ok && f.val ? __float_as_uint(f.val[i + q]) : 0x3F800000u;
          }
          k4[uu] = make_int4(kx[0], kx[1], kx[2], kx[3]);
          g4[uu] = make_int4(gx[0], gx[1], gx[2], gx[3]);
          v4[uu] = make_uint4(vb[0], vb[1], vb[2], vb[3]);
        }
      }
#pragma unroll
      for (int uu = 0; uu < UH; ++uu) {
        const int kx[4] = {k4[uu].x, k4[uu].y, k4[uu].z, k4[uu].w};
        const int gx[4] = {g4[uu].x, g4[uu].y, g4[uu].z, g4[uu].w};
        const uint32_t vb[4] = {v4[uu].x, v4[uu].y, v4[uu].z, v4[uu].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int x = 4 * (h * UH + uu) + q;
          const unsigned ko = (unsigned)kx[q] - (unsigned)kmin;
          const int kc = ko < (unsigned)f.kspan ? tk[ko] : 0xFFFF;
          const int rc = tg[gx[q] - gmin];
          tr[x] = ~0u;
          if (kc == 0xFFFF) continue;
          const int t = (rc >> p.r_bits) * p.nkt + (kc >> p.kw_bits);
          const uint32_t cell = (uint32_t)(((rc & (p.R - 1)) << p.kw_bits) | (kc & (p.KW - 1)));
          if constexpr (SPLIT) e[x] = ((unsigned long long)cell << 32) | vb[q];
          else e[x] = (cell << 16) | (vb[q] >> 16);
          tr[x] = ((uint32_t)t << 16) | (uint32_t)atomicAdd(&cnt[t], 1);
        }
      }
    }
    __syncthreads();
    // ---- 2: exclusive scan of the tile counts, one reservation per non-empty tile
    {
      const int t0 = threadIdx.x * per;
      int run = 0;
      for (int q = 0; q < per; ++q) run += t0 + q < p.ntiles ? cnt[t0 + q] : 0;
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane_id() >= o) incl += y;
      }
      if (lane_id() == 31) wsum[warp_id()] = incl;
      __syncthreads();
      if (warp_id() == 0) {
        const int w = lane_id() < kDtThreads / 32 ? wsum[lane_id()] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, wi, o);
          if (lane_id() >= o) wi += y;
        }
        if (lane_id() < kDtThreads / 32) wsum[lane_id()] = wi - w;
      }
      __syncthreads();
      int x = wsum[warp_id()] + incl - run;
      for (int q = 0; q < per; ++q) {
        const int t = t0 + q;
        if (t >= p.ntiles) break;
        const int c = cnt[t];
        start[t] = x;
        x += c;
        if (c) {
          const int g = atomicAdd(cursor + t, c);
          gpos[t] = g;
          ovf |= g + c > p.cap;  // more tuples than cells: a duplicate cell
        }
        cnt[t] = 0;
      }
      if (threadIdx.x == kDtThreads - 1) s_total = x;  // the batch's entries (tuples with a ∩ key)
    }
    __syncthreads();
    // ---- 3: counting-sorted into the stage
#pragma unroll
    for (int x = 0; x < kPer; ++x)
      if (tr[x] != ~0u) {
        const int t = (int)(tr[x] >> 16), r = (int)(tr[x] & 0xFFFFu);
        const int j = start[t] + r;
        const uint32_t pos = (uint32_t)(gpos[t] + r);  // < 2^28: ntiles <= 4096, cap <= 65536
        stage[j] = e[x];
        sdst[j] = pos < (uint32_t)p.cap ? (uint32_t)t * (uint32_t)p.cap + pos : ~0u;
      }
    __syncthreads();
    // ---- 4: runs out (consecutive threads, consecutive addresses inside a run)
    const int total = s_total;
    for (int j = threadIdx.x; j < total; j += kDtThreads) {
      const uint32_t d = sdst[j];
      if (d != ~0u) __stcg(ent + d, stage[j]);
    }
    __syncthreads();
  }
  ovf = __syncthreads_or(ovf);
  if (threadIdx.x == 0 && ovf) atomicOr(&f.fs->overflow, 1);
}


template <bool SPLIT>
__global__ void __launch_bounds__(kDtTileThreads, 1) k_dt_tile(const DtFill f, const DtPlan p,
                                                              const int32_t* __restrict__ cursor,
                                                              const typename Dt<SPLIT>::Ent* __restrict__ ent) {
  using Ent = typename Dt<SPLIT>::Ent;
  using Cell = typename std::conditional<SPLIT, uint32_t, uint16_t>::type;
  constexpr int kCells = Dt<SPLIT>::kCells;
  extern __shared__ __align__(16) uint8_t smem[];
  Cell* tile = reinterpret_cast<Cell*>(smem);
  unsigned* occ = reinterpret_cast<unsigned*>(smem + (size_t)kCells * sizeof(Cell));
  for (int i = threadIdx.x; i < kCells * (int)sizeof(Cell) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(tile)[i] = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < kCells / 32; i += blockDim.x) occ[i] = 0;
  __syncthreads();
  const int t = blockIdx.x;
  const int raw = cursor[t];
  const int cnt = raw < (int)p.cap ? raw : (int)p.cap;
  const Ent* src = ent + (int64_t)t * p.cap;
  int dup = raw > (int)p.cap;
  // 16-byte vectors (4 or 2 entries), 4 in flight per thread
  constexpr int EV = 16 / sizeof(Ent), U = 4;
  auto put = [&](Ent x) {
    const uint32_t c = SPLIT ? (uint32_t)((unsigned long long)x >> 32) : (uint32_t)x >> 16;
    tile[c] = SPLIT ? (Cell)((unsigned long long)x & 0xFFFFFFFFull) : (Cell)((uint32_t)x & 0xFFFFu);
    dup |= (int)((atomicOr(&occ[c >> 5], 1u << (c & 31)) >> (c & 31)) & 1u);
  };
  const int nv = cnt / EV;
  const uint4* src4 = reinterpret_cast<const uint4*>(src);
  for (int v0 = threadIdx.x; v0 < nv; v0 += U * kDtTileThreads) {
    uint4 w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * kDtTileThreads;
      w[u] = v < nv ? __ldcs(src4 + v) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (v0 + u * kDtTileThreads >= nv) break;
      Ent x[EV];
      memcpy(x, &w[u], 16);
#pragma unroll
      for (int q = 0; q < EV; ++q) put(x[q]);
    }
  }
  for (int i = nv * EV + threadIdx.x; i < cnt; i += kDtTileThreads) put(__ldcs(src + i));
  __syncthreads();
  const int64_t r0 = (int64_t)(t / p.nkt) * p.R, c0 = (int64_t)(t % p.nkt) * p.KW;
  const int nrow = (int)min((int64_t)p.R, f.rows - r0);
  const int ncol = (int)min((int64_t)p.KW, f.Kp - c0);  // multiple of 128
  const int v8 = ncol / 8;
  for (int i = threadIdx.x; i < nrow * v8; i += blockDim.x) {
    const int r = i / v8, c = i - r * v8;
    if constexpr (!SPLIT) {
      __stcs(reinterpret_cast<uint4*>(f.op + (r0 + r) * f.ld_op + c0) + c,
             reinterpret_cast<const uint4*>(tile + (int64_t)r * p.KW)[c]);
    } else {
      const float4 a = reinterpret_cast<const float4*>(tile + (int64_t)r * p.KW)[2 * c];
      const float4 b = reinterpret_cast<const float4*>(tile + (int64_t)r * p.KW)[2 * c + 1];
      const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      store_split8<true>(f.op + (r0 + r) * f.ld_op + c0 + (int64_t)c * 8, f.Kp, x, f.roles, kSplitSegs);
    }
  }
  if (f.pat) {
    // e2m1 existence pattern: nibble 0b0010 (1.0) for every occupied cell, element e in
    // nibble (e & 7) of the little-endian word at byte (e >> 1) & ~3
    const int w32 = ncol / 32;  // occupancy words per row
    for (int i = threadIdx.x; i < nrow * w32; i += blockDim.x) {
      const int r = i / w32, w = i - r * w32;
      const unsigned m = occ[(r * p.KW >> 5) + w];
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const unsigned b = (m >> (8 * q)) & 0xFFu;
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) v |= ((b >> j) & 1u) << (4 * j + 1);
        o[q] = v;
      }
      *reinterpret_cast<uint4*>(f.pat + (r0 + r) * f.ld_pat + (c0 + 32 * (int64_t)w) / 2) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
  dup = __syncthreads_or(dup);
  if (threadIdx.x == 0 && dup) atomicOr(&f.fs->overflow, 1);
}

}  // namespace

bool direct_count_ok(int64_t kspan, int64_t gspan) {
  return kspan > 0 && gspan > 0 && kspan * 4 + gspan <= 160 * 1024;
}

cudaError_t launch_direct_count(const int32_t* key, const int32_t* grp, int64_t n, long long kmin, int64_t kspan,
                                long long gmin, int64_t gspan, int32_t* cnt_span, uint8_t* kflag, uint8_t* gflag,
                                cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  if (!direct_count_ok(kspan, gspan) || (reinterpret_cast<uintptr_t>(key) & 15) ||
      (reinterpret_cast<uintptr_t>(grp) & 15))
    return cudaErrorInvalidValue;
  const int smem = (int)(kspan * 4 + ((gspan + 15) & ~int64_t(15)));
  cudaError_t e = set_func_attr(k_direct_count, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int per_sm = smem <= 100 * 1024 ? 2 : 1;
  int64_t blocks = std::min<int64_t>((int64_t)per_sm * kNumSMs, (n + 16383) / 16384);
  if (blocks < 1) blocks = 1;
  k_direct_count<<<(int)blocks, kCntThreads, smem, s>>>(key, grp, n, (int)kmin, (int)kspan, (int)gmin, (int)gspan,
                                                        cnt_span, kflag, gflag);
  if (launches) ++*launches;
  return cudaGetLastError();
}

bool fill_direct_ok(const DtFill& f, bool split) {
  const DtPlan p = dt_plan(f.rows, f.Kp, split);
  if (!p.bytes || f.kspan <= 0 || f.gspan <= 0 || f.kspan > kDirectSpanMax || f.gspan > kDirectSpanMax) return false;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  return al16(f.key) && al16(f.grp) && (!f.val || al16(f.val)) && f.ld_op % 8 == 0 && (!f.pat || f.ld_pat % 16 == 0);
}

size_t fill_direct_ws(int64_t rows, int64_t Kp, bool split) { return dt_plan(rows, Kp, split).bytes; }

template <bool SPLIT>
static cudaError_t run_dt(const DtFill& f, void* ws, cudaStream_t s, int64_t* launches) {
  using Ent = typename Dt<SPLIT>::Ent;
  const DtPlan p = dt_plan(f.rows, f.Kp, SPLIT);
  if (!p.bytes || !fill_direct_ok(f, SPLIT)) return cudaErrorInvalidValue;
  uint8_t* w = static_cast<uint8_t*>(ws);
  int32_t* cursor = reinterpret_cast<int32_t*>(w);
  Ent* ent = reinterpret_cast<Ent*>(w + p.off_ent);
  cudaError_t e = cudaMemsetAsync(cursor, 0, (size_t)p.ntiles * 4, s);
  if (e != cudaSuccess) return e;
  if (f.n > 0) {
    const int bin_smem = Dt<SPLIT>::kBatch * (int)(sizeof(Ent) + 4) + p.ntiles * 12 + (f.kspan + f.gspan) * 2 + 16;
    if ((e = set_func_attr(k_dt_bin<SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bin_smem)) != cudaSuccess)
      return e;
    const int per_sm = bin_smem <= 110 * 1024 ? 2 : 1;
    const int64_t batches = (f.n + Dt<SPLIT>::kBatch - 1) / Dt<SPLIT>::kBatch;
    const int64_t nblk = std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * kNumSMs, batches));
    // chunks of whole batches, 16-byte aligned
    const int64_t chunk = (batches + nblk - 1) / nblk * Dt<SPLIT>::kBatch;
    k_dt_bin<SPLIT><<<(int)nblk, kDtThreads, bin_smem, s>>>(f, p, cursor, ent, chunk);
    if (launches) ++*launches;
  }
  const int tile_smem = Dt<SPLIT>::kCells * (SPLIT ? 4 : 2) + Dt<SPLIT>::kCells / 8;
  if ((e = set_func_attr(k_dt_tile<SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem)) != cudaSuccess)
    return e;
  k_dt_tile<SPLIT><<<p.ntiles, kDtTileThreads, tile_smem, s>>>(f, p, cursor, ent);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fill_direct(const DtFill& f, bool split, void* ws, cudaStream_t s, int64_t* launches) {
  return split ? run_dt<true>(f, ws, s, launches) : run_dt<false>(f, ws, s, launches);
}

}  // namespace tcudb
