// sparse.cu — step a7: the sparse-operand path for low-density key domains.
//
// PAPER.md §4.2.4: below a density threshold a dense TCU product
// wastes work on zero tiles; TCUDB's TCU-SpMM skipped all-zero 16x16 tiles. On
// B200 with random keys at ~0.1% density nearly every MMA-sized tile is
// non-empty, so instead each joined pair is expanded once (J = sum_k
// cntA(k)·cntB(k) updates, the "output size of the join"):
//   1. bucket B by join-key code (CSC-by-key): offsets = scan(cntB), entries (h, w);
//   2. compact the A tuples that have work (kcode >= 0, cntB(kcode) > 0);
//   3. load-balanced expand: each 256-thread block owns 2048 consecutive updates of
//      the global update sequence (merge-path on the prefix of per-tuple work), so
//      skewed buckets (Zipf hubs) split evenly across blocks; every update is an
//      atomic C[g][h] += v·w (int32 / int64 wrapping / fp64) plus an optional
//      COUNT plane for existence (reading R3).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

constexpr int T = 256;
constexpr int UPB = 2048;           // updates per block
constexpr int UPT = UPB / T;        // updates per thread (strided by T)

inline int grid_for(int64_t n, int per_block = T * 4) {
  int64_t g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > kNumSMs * 16) g = kNumSMs * 16;
  return (int)g;
}

__global__ void k_bucket_fill(const int32_t* __restrict__ kcode, const int32_t* __restrict__ hcode, ColDesc w,
                              int64_t n, const int64_t* __restrict__ bstart, int32_t* __restrict__ cursor,
                              int32_t* __restrict__ b_h, void* __restrict__ b_w, int w_kind) {
  constexpr int U = 4;  // independent tuples per thread per step (latency-bound gathers)
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i0 = (int64_t)blockIdx.x * T + threadIdx.x; i0 < n; i0 += U * stride) {
    int32_t kc[U], hc[U];
    int64_t pos[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      kc[u] = i < n ? __ldcs(kcode + i) : -1;
      hc[u] = i < n ? __ldcs(hcode + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) pos[u] = kc[u] >= 0 ? __ldg(bstart + kc[u]) + atomicAdd(cursor + kc[u], 1) : -1;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (pos[u] < 0) continue;
      const int64_t i = i0 + u * stride;
      b_h[pos[u]] = hc[u];
      if (w_kind == 1) static_cast<long long*>(b_w)[pos[u]] = ld_int(w.data, w.type, i);
      else if (w_kind == 2) static_cast<float*>(b_w)[pos[u]] = __ldg(static_cast<const float*>(w.data) + i);
    }
  }
}

__global__ void k_work(const int32_t* __restrict__ kcode, int64_t n, const int32_t* __restrict__ cnt_b,
                       int32_t* __restrict__ work) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t kc = kcode[i];
    work[i] = kc >= 0 ? cnt_b[kc] : 0;
  }
}

// pos = exclusive scan of (work > 0) computed by the caller as a scan over flags;
// here flags are recomputed from work.
__global__ void k_compact_active(const int32_t* __restrict__ work, const int64_t* __restrict__ pos, int64_t n,
                                 int32_t* __restrict__ act_a, int32_t* __restrict__ act_w) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t wk = work[i];
    if (wk > 0) { act_a[pos[i]] = (int32_t)i; act_w[pos[i]] = wk; }
  }
}

// Active A tuples (kcode >= 0 and cntB(kcode) > 0) grouped by their row g (a counting
// sort): consecutive updates of the expand then land in a narrow window of C rows,
// which stays L2-resident instead of scattering atomics over the whole matrix.
__global__ void __launch_bounds__(1024) k_active_g_count(const int32_t* __restrict__ kcode,
                                                         const int32_t* __restrict__ gcode,
                                                         const int32_t* __restrict__ cnt_b, int64_t n, int G, int R,
                                                         int32_t* __restrict__ gcnt, int use_smem) {
  extern __shared__ int32_t s_cnt[];
  if (use_smem) {
    for (int i = threadIdx.x; i < G; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int32_t kc = kcode[i];
    if (kc < 0 || cnt_b[kc] == 0) continue;
    atomicAdd((use_smem ? s_cnt : gcnt) + gcode[i] / R, 1);
  }
  if (use_smem) {
    __syncthreads();
    for (int i = threadIdx.x; i < G; i += blockDim.x)
      if (s_cnt[i]) atomicAdd(gcnt + i, s_cnt[i]);
  }
}

__global__ void k_active_g_scatter(const int32_t* __restrict__ kcode, const int32_t* __restrict__ gcode,
                                   const int32_t* __restrict__ cnt_b, int64_t n, int R, const int64_t* __restrict__ goff,
                                   int32_t* __restrict__ gcur, int32_t* __restrict__ act_a,
                                   int32_t* __restrict__ act_w, const int64_t* __restrict__ bstart,
                                   int64_t* __restrict__ act_b, int32_t* __restrict__ act_g) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t kc = kcode[i];
    if (kc < 0) continue;
    const int32_t w = cnt_b[kc];
    if (w == 0) continue;
    const int32_t g = gcode[i];
    const int64_t pos = goff[g / R] + atomicAdd(gcur + g / R, 1);
    act_a[pos] = (int32_t)i;
    act_w[pos] = w;
    if (bstart) {
      act_b[pos] = bstart[kc];
      act_g[pos] = g;
    }
  }
}

// Same output as k_active_g_scatter for small G, without same-address contention on
// gcur[g] (c5: 16M tuples over 4,096 rows): each CTA counts its chunk per g in shared
// memory, reserves each g's range with one global atomic, then places its tuples with
// shared-memory cursors (a second read of the chunk, from L2).
__global__ void __launch_bounds__(1024) k_active_g_scatter_smem(
    const int32_t* __restrict__ kcode, const int32_t* __restrict__ gcode, const int32_t* __restrict__ cnt_b,
    int64_t n, int64_t chunk, int G, int R, const int64_t* __restrict__ goff, int32_t* __restrict__ gcur,
    int32_t* __restrict__ act_a, int32_t* __restrict__ act_w, const int64_t* __restrict__ bstart,
    int64_t* __restrict__ act_b, int32_t* __restrict__ act_g) {
  extern __shared__ int64_t s_base[];
  int32_t* s_cnt = reinterpret_cast<int32_t*>(s_base + G);
  for (int g = threadIdx.x; g < G; g += blockDim.x) s_cnt[g] = 0;
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
  // U tuples per thread per step: their loads and the dependent cnt_b gathers overlap
  constexpr int U = 4;
  const int64_t step = (int64_t)U * blockDim.x;
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += step) {
    int32_t kc[U], gc[U], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      kc[u] = i < hi ? __ldcs(kcode + i) : -1;
      gc[u] = i < hi ? __ldcs(gcode + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) w[u] = kc[u] >= 0 ? __ldg(cnt_b + kc[u]) : 0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (w[u] > 0) atomicAdd(s_cnt + gc[u] / R, 1);
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    const int c = s_cnt[g];
    s_base[g] = c ? goff[g] + atomicAdd(gcur + g, c) : 0;
    s_cnt[g] = 0;
  }
  __syncthreads();
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += step) {
    int32_t kc[U], gc[U], w[U];
    int64_t bs[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + (int64_t)u * blockDim.x;
      kc[u] = i < hi ? __ldcs(kcode + i) : -1;
      gc[u] = i < hi ? __ldcs(gcode + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      w[u] = kc[u] >= 0 ? __ldg(cnt_b + kc[u]) : 0;
      bs[u] = (bstart && kc[u] >= 0) ? __ldg(bstart + kc[u]) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (w[u] <= 0) continue;
      const int64_t pos = s_base[gc[u] / R] + atomicAdd(s_cnt + gc[u] / R, 1);
      act_a[pos] = (int32_t)(i0 + (int64_t)u * blockDim.x);
      act_w[pos] = w[u];
      if (bstart) {
        act_b[pos] = bs[u];
        act_g[pos] = gc[u];
      }
    }
  }
}

__global__ void k_flags_from_work(const int32_t* __restrict__ work, int64_t n, int32_t* __restrict__ flags) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) flags[i] = work[i] > 0;
}

__global__ void __launch_bounds__(T) k_expand(const ExpandArgs a) {
  __shared__ int64_t s_off[UPB + 2];
  __shared__ int64_t s_a0;
  __shared__ int s_cnt;
  const int64_t u0 = (int64_t)blockIdx.x * UPB;
  const int64_t u1 = min(u0 + UPB, a.J);
  if (threadIdx.x == 0) {
    // last active index whose offset <= u0
    int64_t lo = 0, hi = a.n_act - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (a.act_off[mid] <= u0) lo = mid; else hi = mid - 1;
    }
    s_a0 = lo;
    // number of active tuples overlapping [u0, u1): at most UPB + 1
    int64_t lo2 = lo, hi2 = a.n_act - 1;
    while (lo2 < hi2) {
      const int64_t mid = (lo2 + hi2 + 1) >> 1;
      if (a.act_off[mid] < u1) lo2 = mid; else hi2 = mid - 1;
    }
    s_cnt = (int)(lo2 - lo + 1);
  }
  __syncthreads();
  const int64_t a0 = s_a0;
  const int cnt = s_cnt;
  for (int i = threadIdx.x; i < cnt; i += T) s_off[i] = a.act_off[a0 + i];
  __syncthreads();
#pragma unroll 2
  for (int j = 0; j < UPT; ++j) {
    const int64_t u = u0 + (int64_t)j * T + threadIdx.x;
    if (u >= u1) break;
    // largest local index l with s_off[l] <= u
    int lo = 0, hi = cnt - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= u) lo = mid; else hi = mid - 1;
    }
    const int32_t ai = a.act_a[a0 + lo];
    const int32_t kc = a.kcodeA[ai];
    const int32_t g = a.gcodeA[ai];
    const int64_t pos = a.bstart[kc] + (u - s_off[lo]);
    const int32_t h = a.b_h[pos];
    const int64_t cell = (int64_t)g * a.ldc + h;
    switch (a.acc_kind) {
      case 4: {  // COUNT in packed u16 pairs; a carry out of a half is detected from the return value
        const int sh = 16 * (int)(cell & 1);
        const unsigned old = atomicAdd(static_cast<unsigned*>(a.C) + (cell >> 1), 1u << sh);
        if (((old >> sh) & 0xFFFFu) == 0xFFFFu) *a.ovf = 1;
        break;
      }
      case 0: atomicAdd(static_cast<int*>(a.C) + cell, 1); break;
      case 1: atomicAdd(static_cast<unsigned long long*>(a.C) + cell, 1ull); break;
      case 2: {
        const long long v = a.va.data ? ld_int(a.va.data, a.va.type, ai) : 1;
        const long long w = a.w_kind == 1 ? static_cast<const long long*>(a.b_w)[pos] : 1;
        atomicAdd(static_cast<unsigned long long*>(a.C) + cell, (unsigned long long)v * (unsigned long long)w);
        break;
      }
      default: {
        const double v = a.va.data ? (double)__ldg(static_cast<const float*>(a.va.data) + ai) : 1.0;
        const double w = a.w_kind == 2 ? (double)static_cast<const float*>(a.b_w)[pos] : 1.0;
        atomicAdd(static_cast<double*>(a.C) + cell, v * w);
      }
    }
    if (a.cnt) atomicAdd(a.cnt + cell, 1);
  }
}

}  // namespace

cudaError_t launch_bucket_fill(const int32_t* kcode, const int32_t* hcode, const ColDesc& w, int64_t n,
                               const int64_t* bstart, int32_t* cursor, int32_t* b_h, void* b_w, int w_kind,
                               cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_bucket_fill<<<grid_for(n), T, 0, s>>>(kcode, hcode, w, n, bstart, cursor, b_h, b_w, w_kind);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_active_by_g(const int32_t* kcode, const int32_t* gcode, const int32_t* cnt_b, int64_t n, int G,
                               int R, int32_t* gcnt, int64_t* goff, int32_t* gcur, int32_t* act_a, int32_t* act_w,
                               const int64_t* bstart, int64_t* act_b, int32_t* act_g,
                               void* scan_tmp, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  const int nb = (G + R - 1) / R;  // bands
  const bool smem = (int64_t)nb * 4 <= 160 * 1024;
  set_func_attr(k_active_g_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  int64_t blocks = n / std::max<int64_t>(4096, nb / 2);
  if (blocks > kNumSMs) blocks = kNumSMs;
  if (blocks < 1) blocks = 1;
  k_active_g_count<<<(int)blocks, 1024, smem ? (size_t)nb * 4 : 0, s>>>(kcode, gcode, cnt_b, n, nb, R, gcnt, smem);
  if (launches) ++*launches;
  cudaError_t e = exclusive_scan_i32(gcnt, goff, nb, goff + nb, scan_tmp, s, launches);
  if (e != cudaSuccess) return e;
  // few bands (<= 1024) and many tuples: per-CTA reservation (one global atomic per CTA and
  // band; the CTA's run per band is long enough to fill whole sectors); else one global
  // atomic per tuple (many bands: little contention)
  if (nb <= 1024 && n >= (1 << 20)) {
    set_func_attr(k_active_g_scatter_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 * 12);
    const int64_t nblk = std::min<int64_t>(2 * kNumSMs, (n + 16383) / 16384);
    const int64_t chunk = (n + nblk - 1) / nblk;
    k_active_g_scatter_smem<<<(int)nblk, 1024, (size_t)nb * 12, s>>>(kcode, gcode, cnt_b, n, chunk, nb, R, goff,
                                                                    gcur, act_a, act_w, bstart, act_b, act_g);
  } else {
    k_active_g_scatter<<<grid_for(n), T, 0, s>>>(kcode, gcode, cnt_b, n, R, goff, gcur, act_a, act_w, bstart, act_b,
                                                  act_g);
  }
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_work(const int32_t* kcode, int64_t n, const int32_t* cnt_b, int32_t* work, cudaStream_t s,
                        int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_work<<<grid_for(n), T, 0, s>>>(kcode, n, cnt_b, work);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_compact_active(const int32_t* work, const int64_t* pos, int64_t n, int32_t* act_a,
                                  int32_t* act_w, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_compact_active<<<grid_for(n), T, 0, s>>>(work, pos, n, act_a, act_w);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_flags_from_work(const int32_t* work, int64_t n, int32_t* flags, cudaStream_t s,
                                   int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_flags_from_work<<<grid_for(n), T, 0, s>>>(work, n, flags);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_expand(const ExpandArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.J <= 0 || a.n_act <= 0) return cudaSuccess;
  const int64_t nb = (a.J + UPB - 1) / UPB;
  if (nb > 0x7fffffffLL) return cudaErrorInvalidValue;
  k_expand<<<(unsigned)nb, T, 0, s>>>(a);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
