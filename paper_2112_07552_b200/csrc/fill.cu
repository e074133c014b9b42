// fill.cu — step a5: operand fill (the paper's "Fill Matrices" stage,
// GPU-assisted data transformation, §4.2.2).
//
// A_op[g][k] = sum over A tuples with (A.g, A.k) = (g, k) of A.v (or 1 for
// COUNT) — the valued/indicator matrices of §3.3
// pre-aggregated per (g, k) cell so that the 1^{1×n} reduction of P:808-810 is
// folded into the fill (reading R5). Layout: row-major, K-major rows padded to
// 128 bytes (TMA / UMMA ready), zero padding.
//
// Paths chosen by the precision guard (a3):
//   COUNT        packed-u8 atomics straight into the operand; a carry out of a
//                byte is detected from the atomic's return value (the guard then
//                re-fills through the wide path);
//   int SUM      int64 scratch (wrapping adds, exact mod 2^64) -> stats -> D
//                base-256 digit planes (u8 low digits, s8 top digit);
//   float SUM    fp32 scratch -> bf16 hi (RNE); if any cell is not bf16-exact,
//                a second pass writes lo = bf16(x - hi) for the 3-product split.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <type_traits>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

constexpr int T = 256;

inline int grid_for(int64_t n, int per_block = T * 4) {
  int64_t g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > kNumSMs * 16) g = kNumSMs * 16;
  return (int)g;
}

__global__ void k_fill_count_u8(const int32_t* __restrict__ kcode, const int32_t* __restrict__ rcode, int64_t n,
                                uint8_t* __restrict__ op, int64_t ld, FillStats* __restrict__ fs) {
  const int64_t stride = (int64_t)gridDim.x * T;
  unsigned mx = 0;
  int ovf = 0;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t kc = kcode[i];
    if (kc < 0) continue;
    const int64_t idx = (int64_t)rcode[i] * ld + kc;
    const int sh = 8 * (int)(idx & 3);
    const unsigned old = atomicAdd(reinterpret_cast<unsigned*>(op + (idx & ~int64_t(3))), 1u << sh);
    const unsigned ob = (old >> sh) & 0xFFu;
    if (ob == 0xFFu) ovf = 1;
    mx = max(mx, ob + 1);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  ovf = __any_sync(0xffffffffu, ovf);
  if (lane_id() == 0) {
    if (mx) atomicMax(&fs->max_abs, (unsigned long long)mx);
    if (ovf) atomicOr(&fs->overflow, 1);
  }
}

// COUNT with 0/1 cells as e2m1 (fp4) nibbles, two per byte: 1.0 = 0b0010. The
// atomicOr's return value tells whether the nibble was already set (a second
// tuple in the same (row, k) cell) -> fs->overflow, and the guard falls back to
// the exact u8 path. Only the set/unset pattern is written, so no carries exist.
__global__ void k_fill_count_fp4(const int32_t* __restrict__ kcode, const int32_t* __restrict__ rcode, int64_t n,
                                 uint8_t* __restrict__ op, int64_t ld_elems, FillStats* __restrict__ fs) {
  const int64_t stride = (int64_t)gridDim.x * T;
  int dup = 0;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t kc = kcode[i];
    if (kc < 0) continue;
    const int64_t e = (int64_t)rcode[i] * ld_elems + kc;  // element index (nibble)
    const int sh = 4 * (int)(e & 7);
    // the OR's return value tells whether the nibble was already set: a duplicate cell
    const unsigned old = atomicOr(reinterpret_cast<unsigned*>(op + ((e >> 1) & ~int64_t(3))), 0x2u << sh);
    dup |= (old >> sh) & 0xFu;
  }
  dup = __any_sync(0xffffffffu, dup);
  if (lane_id() == 0 && dup) atomicOr(&fs->overflow, 1);
}

// Float SUM, optimistic direct fill: when every (row, k) cell holds at most one
// tuple and every value is bf16-exact, the cell IS the bf16 of the value — no fp32
// scratch, no atomics on values, no pack pass (c4: one tuple per cell). A 1-bit
// occupancy map (atomicOr) detects a second tuple in a cell (fs->overflow) and a
// value with nonzero low 16 bits is reported inexact (fs->inexact); either sends the
// guard to the fp32-scratch path.
__global__ void k_fill_bf16_direct(const int32_t* __restrict__ kcode, const int32_t* __restrict__ rcode,
                                   const float* __restrict__ val, int64_t n, uint16_t* __restrict__ op,
                                   int64_t ld_op, unsigned* __restrict__ occ, int64_t ld_occ,
                                   FillStats* __restrict__ fs) {
  const int64_t stride = (int64_t)gridDim.x * T;
  int inexact = 0;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t kc = kcode[i];
    if (kc < 0) continue;
    const int64_t r = rcode[i];
    const uint32_t b = val ? __float_as_uint(__ldg(val + i)) : 0x3F800000u;  // absent value = 1.0
    inexact |= (b & 0xFFFFu) != 0u;
    const int64_t bit = r * ld_occ + kc;
    atomicOr(occ + (bit >> 5), 1u << (bit & 31));  // fire-and-forget; popcount checked afterwards
    op[r * ld_op + kc] = (uint16_t)(b >> 16);
  }
  inexact = __any_sync(0xffffffffu, inexact);
  if (lane_id() == 0 && inexact) atomicOr(&fs->inexact, 1);
}

// Row-range pass of the direct fill (c4-sized operands exceed L2: scattered 2-byte stores
// into HBM-resident lines cost a read-modify-write each). The caller zeroes rows [r0, r1)
// (full lines, allocated in L2) and runs one pass per range sized to fit L2: the tuple
// columns stream through with evict_first loads, the 2-byte stores carry an evict_last
// policy, so each line is merged in L2 and written back once. A duplicate (row, k) cell
// is detected afterwards: #nonzero cells == #tuples with nonzero bits (a zero-valued
// duplicate cannot change a cell's correct value, any other duplicate loses a nonzero).
__global__ void k_fill_bf16_rows(const int32_t* __restrict__ kcode, const int32_t* __restrict__ rcode,
                                 const float* __restrict__ val, int64_t n, uint16_t* __restrict__ op, int64_t ld_op,
                                 int32_t r0, int32_t r1, FillStats* __restrict__ fs) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * T;
  int inexact = 0;
  unsigned long long nz = 0;
  for (int64_t i0 = (int64_t)blockIdx.x * T + threadIdx.x; i0 < n; i0 += U * stride) {
    // all loads of the U tuples are issued before any store (three phases)
    int32_t r[U], kc[U];
    uint32_t b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = i0 + u * stride < n ? __ldcs(rcode + i0 + u * stride) : -1;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool in = r[u] >= r0 && r[u] < r1;
      kc[u] = in ? __ldcs(kcode + i0 + u * stride) : -1;
      b[u] = in && val ? __float_as_uint(__ldcs(val + i0 + u * stride)) : 0x3F800000u;  // absent value = 1.0
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kc[u] < 0) continue;
      inexact |= (b[u] & 0xFFFFu) != 0u;
      const unsigned short h = (unsigned short)(b[u] >> 16);
      nz += h != 0;
      asm volatile("st.global.L2::cache_hint.b16 [%0], %1, %2;" ::"l"(op + (int64_t)r[u] * ld_op + kc[u]), "h"(h),
                   "l"(pol));
    }
  }
  inexact = __any_sync(0xffffffffu, inexact);
  nz = warp_sum(nz);
  if (lane_id() == 0) {
    if (inexact) atomicOr(&fs->inexact, 1);
    if (nz) atomicAdd(&fs->nzt, nz);
  }
}

__global__ void k_count_nonzero_u16(const uint16_t* __restrict__ op, int64_t ld_op, int64_t rows, int64_t cols,
                                    unsigned long long* __restrict__ out) {
  // cols % 8 == 0: 16-byte vectors, 8 cells each
  const int64_t vpr = cols / 8, nv = rows * vpr;
  unsigned long long c = 0;
  for (int64_t v = (int64_t)blockIdx.x * T + threadIdx.x; v < nv; v += (int64_t)gridDim.x * T) {
    const int64_t r = v / vpr, j = v - r * vpr;
    const uint4 x = __ldcs(reinterpret_cast<const uint4*>(op + r * ld_op) + j);
    const unsigned w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) c += ((w[q] & 0xFFFFu) != 0) + ((w[q] >> 16) != 0);
  }
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(out, c);
}

// ---- binned bf16 direct fill: the same result as k_fill_bf16_direct without the
// scattered 2-byte stores into HBM. Rows are grouped into bands of R rows (a band is one
// shared-memory tile of R x Kp bf16) and bands into coarse bins of P bands:
//   hist    per-(coarse bin, block) counts + global per-band totals
//   scatter tuples -> 8-byte entries grouped by coarse bin, staged in shared memory per
//           4096-tuple batch so the stores go out as runs (<= 256 coarse bins)
//   split   one CTA per coarse bin -> 4-byte entries grouped by band (<= 64 write fronts)
//   tile    one CTA per band builds its tile in shared memory and writes it out
//           coalesced (zeros included, so no memset)
// Coarse entry: band-in-bin << 32 | cell-in-band << 16 | bf16; band entry: the low 32 bits.
constexpr int kBinThreads = 1024;
constexpr int kBinBatch = 4 * kBinThreads;
constexpr int kBinMaxCoarse = 256;

__global__ void __launch_bounds__(kBinThreads) k_bin_hist(const int32_t* __restrict__ kcode,
                                                          const int32_t* __restrict__ rcode, int64_t n,
                                                          int64_t chunk, int R, int P, int nband, int ncoarse,
                                                          int32_t* __restrict__ counts,
                                                          int32_t* __restrict__ band_total) {
  extern __shared__ int32_t hist[];  // per band
  for (int b = threadIdx.x; b < nband; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = max(lo, min(n, lo + chunk));  // chunk % 4 == 0
  auto one = [&](int kc, int r) { if (kc >= 0) atomicAdd(&hist[r / R], 1); };
  const int64_t v1 = hi / 4;
  for (int64_t v = lo / 4 + threadIdx.x; v < v1; v += blockDim.x) {
    const int4 k = __ldg(reinterpret_cast<const int4*>(kcode) + v);
    const int4 r = __ldg(reinterpret_cast<const int4*>(rcode) + v);
    one(k.x, r.x); one(k.y, r.y); one(k.z, r.z); one(k.w, r.w);
  }
  for (int64_t i = v1 * 4 + threadIdx.x; i < hi; i += blockDim.x) one(kcode[i], rcode[i]);
  __syncthreads();
  for (int b = threadIdx.x; b < nband; b += blockDim.x)
    if (hist[b]) atomicAdd(band_total + b, hist[b]);
  for (int c = threadIdx.x; c < ncoarse; c += blockDim.x) {
    int sum = 0;
    for (int b = c * P; b < min(nband, (c + 1) * P); ++b) sum += hist[b];
    counts[(int64_t)c * gridDim.x + blockIdx.x] = sum;
  }
}

__global__ void __launch_bounds__(kBinThreads, 2) k_bin_scatter(const int32_t* __restrict__ kcode,
                                                             const int32_t* __restrict__ rcode,
                                                             const float* __restrict__ val, int64_t n, int64_t chunk,
                                                             int R, int P, int ncoarse, int64_t Kp,
                                                             const int64_t* __restrict__ coffs,
                                                             unsigned long long* __restrict__ ent,
                                                             FillStats* __restrict__ fs) {
  __shared__ unsigned long long stage[kBinBatch];
  __shared__ uint8_t sbin[kBinBatch];
  __shared__ int64_t gcur[kBinMaxCoarse];
  __shared__ int cnt[kBinMaxCoarse], bstart[kBinMaxCoarse];
  for (int c = threadIdx.x; c < ncoarse; c += blockDim.x) {
    gcur[c] = coffs[(int64_t)c * gridDim.x + blockIdx.x];
    cnt[c] = 0;
  }
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = max(lo, min(n, lo + chunk));
  const int RP = R * P;
  const bool vec_val = val && (reinterpret_cast<uintptr_t>(val) & 15) == 0;
  int inexact = 0;
  for (int64_t i0 = lo; i0 < hi; i0 += kBinBatch) {
    const int64_t i = i0 + 4 * threadIdx.x;
    int kc[4] = {-1, -1, -1, -1}, r[4] = {0, 0, 0, 0};
    uint32_t b[4] = {0x3F800000u, 0x3F800000u, 0x3F800000u, 0x3F800000u};  // absent value = 1.0
    if (i + 3 < hi) {
      const int4 k4 = __ldg(reinterpret_cast<const int4*>(kcode + i));
      const int4 r4 = __ldg(reinterpret_cast<const int4*>(rcode + i));
      kc[0] = k4.x; kc[1] = k4.y; kc[2] = k4.z; kc[3] = k4.w;
      r[0] = r4.x; r[1] = r4.y; r[2] = r4.z; r[3] = r4.w;
      if (vec_val) {
        const uint4 b4 = __ldcs(reinterpret_cast<const uint4*>(val + i));
        b[0] = b4.x; b[1] = b4.y; b[2] = b4.z; b[3] = b4.w;
      } else if (val) {
#pragma unroll
        for (int u = 0; u < 4; ++u) b[u] = __float_as_uint(val[i + u]);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i + u < hi) {
          kc[u] = kcode[i + u];
          r[u] = rcode[i + u];
          if (val) b[u] = __float_as_uint(val[i + u]);
        }
    }
    int cb[4], rank[4];
    unsigned long long e[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      cb[u] = -1;
      if (kc[u] < 0) continue;
      inexact |= (b[u] & 0xFFFFu) != 0u;
      cb[u] = r[u] / RP;
      const int band = r[u] / R;
      const uint32_t cell = (uint32_t)((r[u] - band * R) * Kp + kc[u]);  // < R * Kp <= 65536
      e[u] = ((unsigned long long)(band - cb[u] * P) << 32) | (cell << 16) | (b[u] >> 16);
      rank[u] = atomicAdd(&cnt[cb[u]], 1);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of <= 256 counts by one warp, 8 per lane
      int v[8], s = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = threadIdx.x * 8 + j;
        v[j] = c < ncoarse ? cnt[c] : 0;
        s += v[j];
      }
      int incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((int)threadIdx.x >= o) incl += t;
      }
      int run = incl - s;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = threadIdx.x * 8 + j;
        if (c < ncoarse) bstart[c] = run;
        run += v[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (cb[u] >= 0) {
        const int j = bstart[cb[u]] + rank[u];
        stage[j] = e[u];
        sbin[j] = (uint8_t)cb[u];
      }
    __syncthreads();
    const int total = bstart[ncoarse - 1] + cnt[ncoarse - 1];
    for (int j = threadIdx.x; j < total; j += blockDim.x) {
      const int c = sbin[j];
      ent[gcur[c] + (j - bstart[c])] = stage[j];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < ncoarse; c += blockDim.x) {
      gcur[c] += cnt[c];
      cnt[c] = 0;
    }
    __syncthreads();
  }
  inexact = __syncthreads_or(inexact);
  if (threadIdx.x == 0 && inexact) atomicOr(&fs->inexact, 1);
}

// One CTA per coarse bin: its 8-byte entries -> 4-byte entries at their band's position.
__global__ void __launch_bounds__(kBinThreads) k_bin_split(const unsigned long long* __restrict__ ent,
                                                           const int64_t* __restrict__ coffs, int nblk, int P,
                                                           int nband, const int64_t* __restrict__ boffs,
                                                           uint32_t* __restrict__ out) {
  __shared__ int64_t base[64];
  __shared__ int cur[64];
  const int c = blockIdx.x;
  for (int f = threadIdx.x; f < P; f += blockDim.x) {
    base[f] = c * P + f < nband ? boffs[c * P + f] : 0;
    cur[f] = 0;
  }
  __syncthreads();
  const int64_t lo = coffs[(int64_t)c * nblk], hi = coffs[(int64_t)(c + 1) * nblk];
  // few write fronts (P bands) shared by the whole CTA: warp-aggregated cursor updates
  for (int64_t i0 = lo + (threadIdx.x & ~31); i0 < hi; i0 += blockDim.x) {
    const int64_t i = i0 + lane_id();
    const unsigned long long e = i < hi ? __ldcs(ent + i) : 0ull;
    const int f = i < hi ? (int)(e >> 32) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, f);
    const int leader = __ffs(peers) - 1;
    int rel = 0;
    if (f >= 0 && lane_id() == leader) rel = atomicAdd(&cur[f], __popc(peers));
    rel = __shfl_sync(0xffffffffu, rel, leader);
    if (f >= 0) out[base[f] + rel + __popc(peers & lanemask_lt())] = (uint32_t)e;
  }
}

// One CTA per band: tile in shared memory, occupancy bits detect a second tuple in a cell.
__global__ void k_bin_tile(const uint32_t* __restrict__ ent, const int64_t* __restrict__ boffs, int R, int64_t Kp,
                           int64_t rows, uint16_t* __restrict__ op, int64_t ld_op, FillStats* __restrict__ fs) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int cells = R * (int)Kp;
  uint16_t* tile = reinterpret_cast<uint16_t*>(smem);
  unsigned* occ = reinterpret_cast<unsigned*>(smem + (size_t)cells * 2);
  const int words = cells / 32;
  for (int i = threadIdx.x; i < cells / 8; i += blockDim.x) reinterpret_cast<uint4*>(tile)[i] = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < words; i += blockDim.x) occ[i] = 0;
  __syncthreads();
  const int band = blockIdx.x;
  const int64_t lo = boffs[band], hi = boffs[band + 1];
  int dup = 0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const uint32_t e = __ldcs(ent + i);
    const uint32_t c = e >> 16;
    tile[c] = (uint16_t)(e & 0xFFFFu);
    dup |= (int)((atomicOr(&occ[c >> 5], 1u << (c & 31)) >> (c & 31)) & 1u);
  }
  __syncthreads();
  const int64_t r0 = (int64_t)band * R;
  const int nrow = (int)(rows - r0 < R ? rows - r0 : R);
  const int v8 = (int)(Kp / 8);  // 16-byte vectors per row
  for (int i = threadIdx.x; i < nrow * v8; i += blockDim.x) {
    const int r = i / v8, c = i - r * v8;
    __stcs(reinterpret_cast<uint4*>(op + (r0 + r) * ld_op) + c, reinterpret_cast<const uint4*>(tile + (int64_t)r * Kp)[c]);
  }
  dup = __syncthreads_or(dup);
  if (threadIdx.x == 0 && dup) atomicOr(&fs->overflow, 1);
}

// Wide integer fill into int64 scratch (COUNT: +1, SUM: +v), wrapping adds.
__global__ void k_fill_i64(const int32_t* __restrict__ kcode, const int32_t* __restrict__ rcode, ColDesc val,
                           int64_t n, unsigned long long* __restrict__ scr, int64_t ld) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t kc = kcode[i];
    if (kc < 0) continue;
    const long long v = val.data ? ld_int(val.data, val.type, i) : 1;
    atomicAdd(scr + (int64_t)rcode[i] * ld + kc, (unsigned long long)v);
  }
}

__global__ void k_fill_f32(const int32_t* __restrict__ kcode, const int32_t* __restrict__ rcode, ColDesc val,
                           int64_t n, float* __restrict__ scr, int64_t ld) {
  const int64_t stride = (int64_t)gridDim.x * T;
  const float* v = static_cast<const float*>(val.data);
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t kc = kcode[i];
    if (kc < 0) continue;
    atomicAdd(scr + (int64_t)rcode[i] * ld + kc, v ? __ldg(v + i) : 1.0f);
  }
}

__global__ void k_scratch_stats_i64(const long long* __restrict__ scr, int64_t count, FillStats* __restrict__ fs) {
  const int64_t stride = (int64_t)gridDim.x * T;
  unsigned long long mx = 0, nnz = 0;
  int neg = 0;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < count; i += stride) {
    const long long x = scr[i];
    const unsigned long long a = x < 0 ? (unsigned long long)(-(x + 1)) + 1ull : (unsigned long long)x;
    mx = max(mx, a);
    nnz += x != 0;
    neg |= x < 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  nnz = warp_sum(nnz);
  neg = __any_sync(0xffffffffu, neg);
  if (lane_id() == 0) {
    if (mx) atomicMax(&fs->max_abs, mx);
    if (nnz) atomicAdd(&fs->nnz, nnz);
    if (neg) atomicOr(&fs->neg, 1);
  }
}

// Digit planes from int64 scratch. Each thread handles 4 consecutive cells -> one u32 per plane.
__global__ void k_pack_planes(const long long* __restrict__ scr, int64_t count, int planes, int top_signed,
                              uint8_t* __restrict__ op, int64_t plane_stride) {
  const int64_t stride = (int64_t)gridDim.x * T;
  const int64_t n4 = count / 4;
  for (int64_t q = (int64_t)blockIdx.x * T + threadIdx.x; q < n4; q += stride) {
    const longlong2 a = reinterpret_cast<const longlong2*>(scr)[2 * q];
    const longlong2 b = reinterpret_cast<const longlong2*>(scr)[2 * q + 1];
    const long long x[4] = {a.x, a.y, b.x, b.y};
    for (int p = 0; p < planes; ++p) {
      uint32_t w = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t d = (p == planes - 1 && top_signed) ? (uint32_t)((x[j] >> (8 * p)) & 0xFF)  // s8 two's complement
                                                           : (uint32_t)(((unsigned long long)x[j] >> (8 * p)) & 0xFF);
        w |= d << (8 * j);
      }
      reinterpret_cast<uint32_t*>(op + p * plane_stride)[q] = w;
    }
  }
}

// Pattern plane: op[r][k] = 1 for every cell holding at least one tuple (plain
// idempotent byte stores, no atomics). Used for existence when SUM can cancel.
__global__ void k_fill_pattern_u8(const int32_t* __restrict__ kcode, const int32_t* __restrict__ rcode, int64_t n,
                                  uint8_t* __restrict__ op, int64_t ld) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t kc = kcode[i];
    if (kc >= 0) op[(int64_t)rcode[i] * ld + kc] = 1;
  }
}

// Symmetric simple-graph adjacency: op[u][v] = op[v][u] = 1 for u != v.
__global__ void k_fill_sym_pattern(const int32_t* __restrict__ u, const int32_t* __restrict__ v, int64_t n,
                                   uint8_t* __restrict__ op, int64_t ld) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t a = u[i], b = v[i];
    if (a < 0 || b < 0 || a == b) continue;
    op[(int64_t)a * ld + b] = 1;
    op[(int64_t)b * ld + a] = 1;
  }
}

__device__ __forceinline__ uint16_t bf16_bits(float x) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}
__device__ __forceinline__ float bf16_val(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

// fp32 scratch -> bf16 segments; 8 cells per thread step: the three-way split (hi, mid, lo)
// written into the K segments of the operand row by their roles (kernels.h kRoles*; kRolesHi:
// hi into segment 0 only); inexact = some cell is not bf16-exact (x - hi != 0)
__global__ void k_pack_bf16(const float* __restrict__ scr, int64_t rows, int64_t ld, uint16_t* __restrict__ op,
                            int64_t ld_op, int roles, FillStats* __restrict__ fs) {
  const int64_t per_row = ld / 8;
  const int64_t total = rows * per_row;
  const int64_t stride = (int64_t)gridDim.x * T;
  int inexact = 0;
  unsigned long long nnz = 0;
  for (int64_t q = (int64_t)blockIdx.x * T + threadIdx.x; q < total; q += stride) {
    const int64_t r = q / per_row, c8 = (q - r * per_row) * 8;
    const float4 a = *reinterpret_cast<const float4*>(scr + r * ld + c8);
    const float4 b = *reinterpret_cast<const float4*>(scr + r * ld + c8 + 4);
    const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      inexact |= (x[j] - bf16_val(bf16_bits(x[j]))) != 0.f;
      nnz += x[j] != 0.f;
    }
    store_split8<false>(op + r * ld_op + c8, ld, x, roles, kSplitSegs);
  }
  inexact = __any_sync(0xffffffffu, inexact);
  nnz = warp_sum(nnz);
  if (lane_id() == 0) {
    if (inexact) atomicOr(&fs->inexact, 1);
    if (nnz) atomicAdd(&fs->nnz, nnz);
  }
}

}  // namespace

cudaError_t launch_fill_count_u8(const int32_t* kcode, const int32_t* rcode, int64_t n, uint8_t* op, int64_t ld,
                                 FillStats* fs, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_fill_count_u8<<<grid_for(n), T, 0, s>>>(kcode, rcode, n, op, ld, fs);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fill_bf16_rows(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                                  uint16_t* op, int64_t ld_op, int32_t r0, int32_t r1, FillStats* fs, cudaStream_t s,
                                  int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_fill_bf16_rows<<<kNumSMs * 8, T, 0, s>>>(kcode, rcode, static_cast<const float*>(val.data), n, op, ld_op, r0, r1,
                                            fs);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_count_nonzero_u16(const uint16_t* op, int64_t ld_op, int64_t rows, int64_t cols,
                                     unsigned long long* out, cudaStream_t s, int64_t* launches) {
  if (rows <= 0 || cols <= 0 || cols % 8) return cols % 8 ? cudaErrorInvalidValue : cudaSuccess;
  k_count_nonzero_u16<<<kNumSMs * 8, T, 0, s>>>(op, ld_op, rows, cols, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fill_bf16_direct(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                                    uint16_t* op, int64_t ld_op, unsigned* occ, int64_t ld_occ, FillStats* fs,
                                    cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_fill_bf16_direct<<<grid_for(n), T, 0, s>>>(kcode, rcode, static_cast<const float*>(val.data), n, op, ld_op,
                                               occ, ld_occ, fs);
  if (launches) ++*launches;
  return cudaGetLastError();
}

namespace {
constexpr int kBinTileBytes = 64 * 1024;  // 3 tiles per SM
constexpr int kBinMaxBands = 8192;
constexpr int kBinBlocks = kNumSMs * 2;  // 1024-thread blocks, 2 per SM
constexpr int kBinTileThreads = 512;
struct BinPlan {
  int R = 0, P = 0, nband = 0, ncoarse = 0, nblk = 0;
  int64_t chunk = 0;
  size_t off_counts = 0, off_coffs = 0, off_btot = 0, off_boffs = 0, off_temp = 0, off_ent8 = 0, off_ent4 = 0,
         bytes = 0;
};
inline size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
BinPlan bin_plan(int64_t n, int64_t rows, int64_t Kp) {
  BinPlan p;
  if (n < (1 << 20) || Kp * 2 > kBinTileBytes || Kp % 32) return p;
  int R = 1;
  while (2 * R * Kp * 2 <= kBinTileBytes && R < rows) R *= 2;
  const int64_t nband = (rows + R - 1) / R;
  if (nband > kBinMaxBands) return p;
  int P = 1;
  while ((nband + P - 1) / P > kBinMaxCoarse) P *= 2;
  if (P > 64) return p;
  p.R = R;
  p.P = P;
  p.nband = (int)nband;
  p.ncoarse = (int)((nband + P - 1) / P);
  p.nblk = (int)std::min<int64_t>(kBinBlocks, (n + 8191) / 8192);
  p.chunk = ((n + p.nblk - 1) / p.nblk + 3) & ~int64_t(3);  // 16-byte aligned chunks
  const int64_t m = (int64_t)p.ncoarse * p.nblk;
  p.off_counts = 0;
  p.off_coffs = al256(m * 4);
  p.off_btot = p.off_coffs + al256((m + 1) * 8);
  p.off_boffs = p.off_btot + al256(nband * 4);
  p.off_temp = p.off_boffs + al256((nband + 1) * 8);
  p.off_ent8 = p.off_temp + al256(std::max(scan_temp_bytes(m), scan_temp_bytes(nband)));
  p.off_ent4 = p.off_ent8 + al256(n * 8);
  p.bytes = p.off_ent4 + al256(n * 4);
  return p;
}
}  // namespace

size_t fill_bf16_binned_ws(int64_t n, int64_t rows, int64_t Kp) { return bin_plan(n, rows, Kp).bytes; }

cudaError_t launch_fill_bf16_binned(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                                    int64_t rows, int64_t Kp, uint16_t* op, int64_t ld_op, FillStats* fs, void* ws,
                                    cudaStream_t s, int64_t* launches) {
  const BinPlan p = bin_plan(n, rows, Kp);
  if (!p.bytes) return cudaErrorInvalidValue;
  uint8_t* w = static_cast<uint8_t*>(ws);
  int32_t* counts = reinterpret_cast<int32_t*>(w + p.off_counts);
  int64_t* coffs = reinterpret_cast<int64_t*>(w + p.off_coffs);
  int32_t* btot = reinterpret_cast<int32_t*>(w + p.off_btot);
  int64_t* boffs = reinterpret_cast<int64_t*>(w + p.off_boffs);
  auto* ent8 = reinterpret_cast<unsigned long long*>(w + p.off_ent8);
  uint32_t* ent4 = reinterpret_cast<uint32_t*>(w + p.off_ent4);
  const int64_t m = (int64_t)p.ncoarse * p.nblk;
  cudaError_t e = cudaMemsetAsync(btot, 0, (size_t)p.nband * 4, s);
  if (e != cudaSuccess) return e;
  k_bin_hist<<<p.nblk, kBinThreads, p.nband * 4, s>>>(kcode, rcode, n, p.chunk, p.R, p.P, p.nband, p.ncoarse,
                                                      counts, btot);
  if ((e = exclusive_scan_i32(counts, coffs, m, coffs + m, w + p.off_temp, s, launches)) != cudaSuccess) return e;
  if ((e = exclusive_scan_i32(btot, boffs, p.nband, boffs + p.nband, w + p.off_temp, s, launches)) != cudaSuccess)
    return e;
  k_bin_scatter<<<p.nblk, kBinThreads, 0, s>>>(kcode, rcode, static_cast<const float*>(val.data), n, p.chunk, p.R,
                                               p.P, p.ncoarse, Kp, coffs, ent8, fs);
  k_bin_split<<<p.ncoarse, kBinThreads, 0, s>>>(ent8, coffs, p.nblk, p.P, p.nband, boffs, ent4);
  e = set_func_attr(k_bin_tile, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kBinTileBytes + kBinTileBytes / 16);
  if (e != cudaSuccess) return e;
  const int tile_smem = (int)(p.R * Kp * 2 + p.R * Kp / 8);
  k_bin_tile<<<p.nband, kBinTileThreads, tile_smem, s>>>(ent4, boffs, p.R, Kp, rows, op, ld_op, fs);
  if (launches) *launches += 4;
  return cudaGetLastError();
}

// ---- tiled bf16 direct fill (one binning level): the operand is cut into tiles of
// 65,536 cells (R rows x KW columns, KW = a power of two <= 8192); every tuple becomes a
// 4-byte entry (cell in tile << 16 | bf16 bits) binned by tile in ONE pass — large batches
// (16 K tuples per CTA) staged in shared memory so each tile's entries leave as runs — and
// one CTA per tile builds the tile in shared memory and writes it out coalesced, zeros
// included. Per tuple: 4-8 B (hist) + 12 B read + 4 B written (bin) + 4 B read + 2 B
// written (tile), vs the scattered 2-byte stores of the direct / row-range fills that
// are bound by L2's partial-sector store rate.
namespace {
constexpr int kT2Threads = 1024;     // hist / tile kernels
constexpr int kT2BinThreads = 1024;  // bin kernel, one CTA per SM (512 x 2 CTAs measured slower on
constexpr int kT2Batch = 16 * kT2BinThreads;  //   c4: 1.68 vs 1.56 ms — shorter runs per tile)
constexpr int kT2MaxTiles = 4096;
constexpr int kT2TileCells = 65536;
// SPLIT (values that are not bf16-exact): 8-byte entries (cell << 32 | fp32 bits), fp32 tiles of
// 32,768 cells, and the tile CTA writes bf16 hi / lo = bf16(x - hi) into the segments of the
// three-way split layout (kernels.h kRolesA / kRolesB) — no fp32 scratch, no atomics
template <bool SPLIT> struct T2 {
  using Ent = typename std::conditional<SPLIT, unsigned long long, uint32_t>::type;
  static constexpr int kCells = SPLIT ? 32768 : kT2TileCells;
  static constexpr int kBatch = SPLIT ? 8 * kT2BinThreads : kT2Batch;
};
struct T2Plan {
  int KW = 0, R = 0, nkt = 0, ntiles = 0, nblk = 0, kw_bits = 0;
  int64_t chunk = 0;
  size_t off_counts = 0, off_offs = 0, off_temp = 0, off_ent = 0, bytes = 0;
};
T2Plan t2_plan(int64_t n, int64_t rows, int64_t Kp, bool split = false) {
  T2Plan p;
  if (n < (1 << 20) || Kp % 8) return p;
  int KW = 128, kb = 7;
  while (KW < Kp && KW < 8192) { KW *= 2; ++kb; }
  const int R = (split ? 32768 : kT2TileCells) / KW;
  const int64_t nkt = (Kp + KW - 1) / KW, nrt = (rows + R - 1) / R;
  if (nkt * nrt > kT2MaxTiles) return p;
  p.KW = KW; p.kw_bits = kb; p.R = R; p.nkt = (int)nkt; p.ntiles = (int)(nkt * nrt);
  const int batch = split ? 8 * kT2BinThreads : kT2Batch;
  p.nblk = (int)std::min<int64_t>(kNumSMs, (n + batch - 1) / batch);
  p.chunk = ((n + p.nblk - 1) / p.nblk + 3) & ~int64_t(3);  // 16-byte aligned chunks
  const int64_t m = (int64_t)p.ntiles * p.nblk;
  p.off_counts = 0;
  p.off_offs = al256(m * 4);
  p.off_temp = p.off_offs + al256((m + 1) * 8);
  p.off_ent = p.off_temp + al256(scan_temp_bytes(m));
  p.bytes = p.off_ent + al256(n * (split ? 8 : 4));
  return p;
}

TCUDB_DEV int t2_tile(int r, int kc, int R, int kw_bits, int nkt) { return (r / R) * nkt + (kc >> kw_bits); }

// per-(tile, block) counts, tile-major (the scan gives each block its run per tile)
__global__ void __launch_bounds__(kT2Threads) k_t2_hist(const int32_t* __restrict__ kcode,
                                                        const int32_t* __restrict__ rcode, int64_t n, int64_t chunk,
                                                        int R, int kw_bits, int nkt, int ntiles,
                                                        int32_t* __restrict__ counts) {
  __shared__ int hist[kT2MaxTiles];
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) hist[t] = 0;
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = max(lo, min(n, lo + chunk));
  auto one = [&](int kc, int r) { if (kc >= 0) atomicAdd(&hist[t2_tile(r, kc, R, kw_bits, nkt)], 1); };
  const int64_t v1 = hi / 4;
  for (int64_t v = lo / 4 + threadIdx.x; v < v1; v += blockDim.x) {
    const int4 k = __ldcs(reinterpret_cast<const int4*>(kcode) + v);
    const int4 r = __ldcs(reinterpret_cast<const int4*>(rcode) + v);
    one(k.x, r.x); one(k.y, r.y); one(k.z, r.z); one(k.w, r.w);
  }
  for (int64_t i = v1 * 4 + threadIdx.x; i < hi; i += blockDim.x) one(kcode[i], rcode[i]);
  __syncthreads();
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) counts[(int64_t)t * gridDim.x + blockIdx.x] = hist[t];
}

template <bool SPLIT>
__global__ void __launch_bounds__(kT2BinThreads, 1) k_t2_bin(const int32_t* __restrict__ kcode,
                                                         const int32_t* __restrict__ rcode,
                                                         const float* __restrict__ val, int64_t n, int64_t chunk,
                                                         int R, int KW, int kw_bits, int nkt, int ntiles,
                                                         const int64_t* __restrict__ offs,
                                                         typename T2<SPLIT>::Ent* __restrict__ ent,
                                                         FillStats* __restrict__ fs) {
  using Ent = typename T2<SPLIT>::Ent;
  constexpr int kBatch = T2<SPLIT>::kBatch;
  extern __shared__ __align__(16) uint8_t smem[];
  Ent* stage = reinterpret_cast<Ent*>(smem);                                 // [kBatch]
  uint16_t* stile = reinterpret_cast<uint16_t*>(stage + kBatch);             // [kBatch]
  int64_t* gcur = reinterpret_cast<int64_t*>(stile + kBatch);               // [ntiles]
  int* cnt = reinterpret_cast<int*>(gcur + ntiles);                          // [ntiles]
  int* bstart = cnt + ntiles;                                                // [ntiles]
  __shared__ int wsum[kT2BinThreads / 32];
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    gcur[t] = offs[(int64_t)t * gridDim.x + blockIdx.x];
    cnt[t] = 0;
  }
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = max(lo, min(n, lo + chunk));
  const bool vec_val = val && (reinterpret_cast<uintptr_t>(val) & 15) == 0;
  const int per = (ntiles + kT2BinThreads - 1) / kT2BinThreads;  // counters per thread in the scan
  int inexact = 0;
  for (int64_t b0 = lo; b0 < hi; b0 += kBatch) {
    constexpr int U = kBatch / kT2BinThreads / 4;  // int4 vectors per thread per column
    Ent e[4 * U];
    int tl[4 * U], rk[4 * U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = b0 + ((int64_t)u * kT2BinThreads + threadIdx.x) * 4;
      int kc[4] = {-1, -1, -1, -1}, r[4] = {0, 0, 0, 0};
      uint32_t bv[4] = {0x3F800000u, 0x3F800000u, 0x3F800000u, 0x3F800000u};  // absent value = 1.0
      if (i + 3 < hi) {
        const int4 k4 = __ldcs(reinterpret_cast<const int4*>(kcode + i));
        const int4 r4 = __ldcs(reinterpret_cast<const int4*>(rcode + i));
        kc[0] = k4.x; kc[1] = k4.y; kc[2] = k4.z; kc[3] = k4.w;
        r[0] = r4.x; r[1] = r4.y; r[2] = r4.z; r[3] = r4.w;
        if (vec_val) {
          const uint4 b4 = __ldcs(reinterpret_cast<const uint4*>(val + i));
          bv[0] = b4.x; bv[1] = b4.y; bv[2] = b4.z; bv[3] = b4.w;
        } else if (val) {
#pragma unroll
          for (int q = 0; q < 4; ++q) bv[q] = __float_as_uint(val[i + q]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (i + q < hi) {
            kc[q] = kcode[i + q];
            r[q] = rcode[i + q];
            if (val) bv[q] = __float_as_uint(val[i + q]);
          }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int x = 4 * u + q;
        tl[x] = -1;
        if (kc[q] < 0) continue;
        inexact |= (bv[q] & 0xFFFFu) != 0u;
        tl[x] = t2_tile(r[q], kc[q], R, kw_bits, nkt);
        const uint32_t cell = (uint32_t)((r[q] % R) * KW + (kc[q] & (KW - 1)));  // < tile cells
        if constexpr (SPLIT) e[x] = ((unsigned long long)cell << 32) | bv[q];
        else e[x] = (cell << 16) | (bv[q] >> 16);
        rk[x] = atomicAdd(&cnt[tl[x]], 1);
      }
    }
    __syncthreads();
    // exclusive scan of the ntiles counts: each thread a contiguous run of `per`
    {
      const int t0 = threadIdx.x * per;
      int run = 0;
      for (int q = 0; q < per; ++q) run += t0 + q < ntiles ? cnt[t0 + q] : 0;
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane_id() >= o) incl += t;
      }
      if (lane_id() == 31) wsum[warp_id()] = incl;
      __syncthreads();
      if (warp_id() == 0) {
        const int w = lane_id() < kT2BinThreads / 32 ? wsum[lane_id()] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, wi, o);
          if (lane_id() >= o) wi += t;
        }
        if (lane_id() < kT2BinThreads / 32) wsum[lane_id()] = wi - w;
      }
      __syncthreads();
      int x = wsum[warp_id()] + incl - run;
      for (int q = 0; q < per; ++q)
        if (t0 + q < ntiles) { bstart[t0 + q] = x; x += cnt[t0 + q]; }
    }
    __syncthreads();
#pragma unroll
    for (int x = 0; x < 4 * U; ++x)
      if (tl[x] >= 0) {
        const int j = bstart[tl[x]] + rk[x];
        stage[j] = e[x];
        stile[j] = (uint16_t)tl[x];
      }
    __syncthreads();
    const int total = bstart[ntiles - 1] + cnt[ntiles - 1];
    for (int j = threadIdx.x; j < total; j += blockDim.x) {
      const int t = stile[j];
      __stcg(ent + gcur[t] + (j - bstart[t]), stage[j]);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
      gcur[t] += cnt[t];
      cnt[t] = 0;
    }
    __syncthreads();
  }
  inexact = __syncthreads_or(inexact);
  if (threadIdx.x == 0 && inexact) atomicOr(&fs->inexact, 1);
}

// one CTA per tile: R x KW bf16 cells (SPLIT: fp32 cells, written as the three-way bf16 split
// into the segments of the split layout by their roles, segment stride Kp) + occupancy bits
template <bool SPLIT>
__global__ void __launch_bounds__(kT2Threads, 1) k_t2_tile(const typename T2<SPLIT>::Ent* __restrict__ ent,
                                                          const int64_t* __restrict__ offs, int nblk, int R, int KW,
                                                          int nkt, int64_t rows, int64_t Kp,
                                                          uint16_t* __restrict__ op, int64_t ld_op, int roles,
                                                          FillStats* __restrict__ fs) {
  using Ent = typename T2<SPLIT>::Ent;
  constexpr int kCells = T2<SPLIT>::kCells;
  using Cell = typename std::conditional<SPLIT, uint32_t, uint16_t>::type;
  extern __shared__ __align__(16) uint8_t smem[];
  Cell* tile = reinterpret_cast<Cell*>(smem);
  unsigned* occ = reinterpret_cast<unsigned*>(smem + (size_t)kCells * sizeof(Cell));
  for (int i = threadIdx.x; i < kCells * (int)sizeof(Cell) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(tile)[i] = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < kCells / 32; i += blockDim.x) occ[i] = 0;
  __syncthreads();
  const int t = blockIdx.x;
  const int64_t lo = offs[(int64_t)t * nblk], hi = offs[(int64_t)(t + 1) * nblk];
  int dup = 0;
  constexpr int U = 4;
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (int64_t)U * blockDim.x) {
    Ent e[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      e[u] = i < hi ? __ldcs(ent + i) : (Ent)0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + (int64_t)u * blockDim.x >= hi) continue;
      const uint32_t c = SPLIT ? (uint32_t)((unsigned long long)e[u] >> 32) : (uint32_t)e[u] >> 16;
      tile[c] = SPLIT ? (Cell)((unsigned long long)e[u] & 0xFFFFFFFFull) : (Cell)((uint32_t)e[u] & 0xFFFFu);
      dup |= (int)((atomicOr(&occ[c >> 5], 1u << (c & 31)) >> (c & 31)) & 1u);
    }
  }
  __syncthreads();
  const int64_t r0 = (int64_t)(t / nkt) * R, c0 = (int64_t)(t % nkt) * KW;
  const int nrow = (int)min((int64_t)R, rows - r0);
  const int ncol = (int)min((int64_t)KW, Kp - c0);  // multiple of 8
  const int v8 = ncol / 8;
  for (int i = threadIdx.x; i < nrow * v8; i += blockDim.x) {
    const int r = i / v8, c = i - r * v8;
    if constexpr (!SPLIT) {
      __stcs(reinterpret_cast<uint4*>(op + (r0 + r) * ld_op + c0) + c,
             reinterpret_cast<const uint4*>(tile + (int64_t)r * KW)[c]);
    } else {
      const float4 a = reinterpret_cast<const float4*>(tile + (int64_t)r * KW)[2 * c];
      const float4 b = reinterpret_cast<const float4*>(tile + (int64_t)r * KW)[2 * c + 1];
      const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      store_split8<true>(op + (r0 + r) * ld_op + c0 + (int64_t)c * 8, Kp, x, roles, kSplitSegs);
    }
  }
  dup = __syncthreads_or(dup);
  if (threadIdx.x == 0 && dup) atomicOr(&fs->overflow, 1);
}
}  // namespace

size_t fill_bf16_tiled_ws(int64_t n, int64_t rows, int64_t Kp, bool split) {
  return t2_plan(n, rows, Kp, split).bytes;
}

template <bool SPLIT>
static cudaError_t run_t2(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n, int64_t rows,
                          int64_t Kp, uint16_t* op, int64_t ld_op, int roles, FillStats* fs, void* ws,
                          cudaStream_t s, int64_t* launches) {
  using Ent = typename T2<SPLIT>::Ent;
  const T2Plan p = t2_plan(n, rows, Kp, SPLIT);
  if (!p.bytes) return cudaErrorInvalidValue;
  uint8_t* w = static_cast<uint8_t*>(ws);
  int32_t* counts = reinterpret_cast<int32_t*>(w + p.off_counts);
  int64_t* offs = reinterpret_cast<int64_t*>(w + p.off_offs);
  Ent* ent = reinterpret_cast<Ent*>(w + p.off_ent);
  const int64_t m = (int64_t)p.ntiles * p.nblk;
  k_t2_hist<<<p.nblk, kT2Threads, 0, s>>>(kcode, rcode, n, p.chunk, p.R, p.kw_bits, p.nkt, p.ntiles, counts);
  cudaError_t e = exclusive_scan_i32(counts, offs, m, offs + m, w + p.off_temp, s, launches);
  if (e != cudaSuccess) return e;
  const int bin_smem = T2<SPLIT>::kBatch * (int)(sizeof(Ent) + 2) + p.ntiles * 16;
  if ((e = set_func_attr(k_t2_bin<SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, bin_smem)) != cudaSuccess)
    return e;
  k_t2_bin<SPLIT><<<p.nblk, kT2BinThreads, bin_smem, s>>>(kcode, rcode, static_cast<const float*>(val.data), n,
                                                          p.chunk, p.R, p.KW, p.kw_bits, p.nkt, p.ntiles, offs, ent,
                                                          fs);
  const int tile_smem = T2<SPLIT>::kCells * (SPLIT ? 4 : 2) + T2<SPLIT>::kCells / 8;
  if ((e = set_func_attr(k_t2_tile<SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem)) != cudaSuccess)
    return e;
  k_t2_tile<SPLIT><<<p.ntiles, kT2Threads, tile_smem, s>>>(ent, offs, p.nblk, p.R, p.KW, p.nkt, rows, Kp, op, ld_op,
                                                           roles, fs);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_fill_bf16_tiled(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                                   int64_t rows, int64_t Kp, uint16_t* op, int64_t ld_op, FillStats* fs, void* ws,
                                   cudaStream_t s, int64_t* launches) {
  return run_t2<false>(kcode, rcode, val, n, rows, Kp, op, ld_op, kRolesHi, fs, ws, s, launches);
}

cudaError_t launch_fill_bf16_split_tiled(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                                         int64_t rows, int64_t Kp, uint16_t* op, int64_t ld_op, int roles,
                                         FillStats* fs, void* ws, cudaStream_t s, int64_t* launches) {
  return run_t2<true>(kcode, rcode, val, n, rows, Kp, op, ld_op, roles, fs, ws, s, launches);
}

cudaError_t launch_fill_count_fp4(const int32_t* kcode, const int32_t* rcode, int64_t n, uint8_t* op,
                                  int64_t ld_elems, FillStats* fs, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_fill_count_fp4<<<grid_for(n), T, 0, s>>>(kcode, rcode, n, op, ld_elems, fs);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fill_pattern_u8(const int32_t* kcode, const int32_t* rcode, int64_t n, uint8_t* op, int64_t ld,
                                   cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_fill_pattern_u8<<<grid_for(n), T, 0, s>>>(kcode, rcode, n, op, ld);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fill_sym_pattern(const int32_t* u, const int32_t* v, int64_t n, uint8_t* op, int64_t ld,
                                    cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_fill_sym_pattern<<<grid_for(n), T, 0, s>>>(u, v, n, op, ld);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fill_i64(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                            long long* scr, int64_t ld, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_fill_i64<<<grid_for(n), T, 0, s>>>(kcode, rcode, val, n, reinterpret_cast<unsigned long long*>(scr), ld);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fill_f32(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n, float* scr,
                            int64_t ld, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_fill_f32<<<grid_for(n), T, 0, s>>>(kcode, rcode, val, n, scr, ld);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_scratch_stats_i64(const long long* scr, int64_t count, FillStats* fs, cudaStream_t s,
                                     int64_t* launches) {
  if (count <= 0) return cudaSuccess;
  k_scratch_stats_i64<<<grid_for(count, T * 8), T, 0, s>>>(scr, count, fs);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_pack_planes(const long long* scr, int64_t count, int planes, int top_signed, uint8_t* op,
                               int64_t plane_stride, cudaStream_t s, int64_t* launches) {
  if (count <= 0) return cudaSuccess;
  k_pack_planes<<<grid_for(count / 4, T * 4), T, 0, s>>>(scr, count, planes,
                                                         top_signed, op, plane_stride);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_pack_bf16(const float* scr, int64_t rows, int64_t ld, uint16_t* op, int64_t ld_op, int roles,
                             FillStats* fs, cudaStream_t s, int64_t* launches) {
  if (rows <= 0) return cudaSuccess;
  k_pack_bf16<<<grid_for(rows * (ld / 8), T * 4), T, 0, s>>>(scr, rows, ld, op, ld_op, roles, fs);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
