// reduce.cu — §8(f) f2: aggregates whose GROUP BY leaves one side ungrouped.
//
// PAPER.md §3.3 evaluates
//   Q3  SELECT SUM(A.Val), B.Val FROM A, B WHERE A.ID = B.ID GROUP BY B.Val
//       as 1^{1×n} × mat(A) × mat(B)^T
//   Q4  SELECT SUM(A.Val * B.Val) FROM A, B WHERE A.ID = B.ID
//       as mat(A) × mat(B)^T × 1^{m×1} reduced by 1^{1×n}
//   AVG = SUM / COUNT
// With A ungrouped the product collapses to a vector: SA(k) = Σ_{a.k=k} a.v is
// 1^{1×n} × mat(A) (one entry per join key), and group h receives
// Σ_{b.h=h} b.w · SA(b.k). That is a segmented reduction over B's tuples — HBM-
// bound, so it runs as two streaming passes with shared-memory privatized
// accumulators instead of a padded 1-row tensor-core GEMM (which would move the
// same bytes and waste 127 of 128 MMA rows). Existence is COUNT > 0 (reading R3):
// the count Σ_{b.h=h} cntA(b.k) is accumulated alongside.
// Integer sums wrap mod 2^64 (exact whenever the result fits; the guard a3 has
// proved it does); float sums accumulate fp64 products of fp32 inputs.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

constexpr int T = 256;
constexpr int kSmemGroups = 2048;  // privatized accumulators: 16 B x 2048 per block

// sum_k[k] += v (per-key sums of one side's values): kind 1 int64 (wrapping), 2 fp64
__global__ void k_key_sum(const int32_t* __restrict__ kcode, ColDesc v, int64_t n, int kind, void* __restrict__ sum_k) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t k = kcode[i];
    if (k < 0) continue;
    if (kind == 1) atomicAdd(static_cast<unsigned long long*>(sum_k) + k, (unsigned long long)ld_int(v.data, v.type, i));
    else atomicAdd(static_cast<double*>(sum_k) + k, (double)__ldg(static_cast<const float*>(v.data) + i));
  }
}

// cnt_g[g] += cnt_o[k]; sum_g[g] += w_i · S_o(k) over this side's tuples i (key k, group g).
// S_o(k) = sum_o[k] when the other side has values, else cnt_o[k]; w_i = 1 without values.
// kind: 0 COUNT, 1 int SUM, 2 float SUM.
template <bool SMEM>
__global__ void k_side_agg(const int32_t* __restrict__ kcode, const int32_t* __restrict__ gcode, ColDesc w,
                           int64_t n, const int32_t* __restrict__ cnt_o, const void* __restrict__ sum_o, int kind,
                           int NG, unsigned long long* __restrict__ cnt_g, void* __restrict__ sum_g) {
  __shared__ unsigned long long s_cnt[SMEM ? kSmemGroups : 1];
  __shared__ unsigned long long s_sum[SMEM ? kSmemGroups : 1];  // u64 bits (int) or fp64 bits
  if (SMEM) {
    for (int i = threadIdx.x; i < NG; i += T) { s_cnt[i] = 0; s_sum[i] = 0; }
    __syncthreads();
  }
  unsigned long long* cg = SMEM ? s_cnt : cnt_g;
  unsigned long long* sg = SMEM ? s_sum : static_cast<unsigned long long*>(sum_g);
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t k = kcode[i];
    if (k < 0) continue;
    const int32_t c = __ldg(cnt_o + k);
    if (c == 0) continue;
    const int32_t g = gcode[i];
    atomicAdd(cg + g, (unsigned long long)c);
    if (kind == 1) {
      const unsigned long long so = sum_o ? __ldg(static_cast<const unsigned long long*>(sum_o) + k)
                                          : (unsigned long long)c;
      const unsigned long long wi = w.data ? (unsigned long long)ld_int(w.data, w.type, i) : 1ull;
      atomicAdd(sg + g, so * wi);  // wrapping product and sum
    } else if (kind == 2) {
      const double so = sum_o ? __ldg(static_cast<const double*>(sum_o) + k) : (double)c;
      const double wi = w.data ? (double)__ldg(static_cast<const float*>(w.data) + i) : 1.0;
      atomicAdd(reinterpret_cast<double*>(sg) + g, so * wi);
    }
  }
  if (SMEM) {
    __syncthreads();
    for (int i = threadIdx.x; i < NG; i += T) {
      if (!s_cnt[i]) continue;
      atomicAdd(cnt_g + i, s_cnt[i]);
      if (kind == 1) atomicAdd(static_cast<unsigned long long*>(sum_g) + i, s_sum[i]);
      else if (kind == 2) atomicAdd(static_cast<double*>(sum_g) + i, __longlong_as_double((long long)s_sum[i]));
    }
  }
}

__global__ void k_side_flags(const unsigned long long* __restrict__ cnt_g, int64_t NG, int32_t* __restrict__ flags) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < NG; i += stride) flags[i] = cnt_g[i] != 0;
}

// Result rows for the groups with COUNT > 0, in ascending group order (codes are ranks).
// The grouped side's values come from dict_grp[code]; the ungrouped side's output column
// (if present at all) is its single value, const_val.
__global__ void k_side_write(const unsigned long long* __restrict__ cnt_g, const void* __restrict__ sum_g,
                             const int64_t* __restrict__ pos, int64_t NG, int agg_kind, SideOut o) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < NG; i += stride) {
    const unsigned long long c = cnt_g[i];
    if (!c) continue;
    const int64_t p = pos[i];
    const long long gv = o.dict_grp[i];
    if (o.grp_out) {
      if (o.grp_type) static_cast<long long*>(o.grp_out)[p] = gv;
      else static_cast<int*>(o.grp_out)[p] = (int)gv;
    }
    if (o.const_out) {
      if (o.const_type) static_cast<long long*>(o.const_out)[p] = o.const_val;
      else static_cast<int*>(o.const_out)[p] = (int)o.const_val;
    }
    switch (agg_kind) {
      case 0: static_cast<long long*>(o.agg)[p] = (long long)c; break;                          // COUNT
      case 1: static_cast<long long*>(o.agg)[p] = static_cast<const long long*>(sum_g)[i]; break;  // int SUM
      case 2: static_cast<double*>(o.agg)[p] = static_cast<const double*>(sum_g)[i]; break;        // float SUM
      case 3: static_cast<double*>(o.agg)[p] = (double)static_cast<const long long*>(sum_g)[i] / (double)c; break;
      default: static_cast<double*>(o.agg)[p] = static_cast<const double*>(sum_g)[i] / (double)c;  // AVG float
    }
  }
}

// AVG of two aligned results (same groups, same order): avg[i] = sum[i] / cnt[i] in fp64.
__global__ void k_avg_div(void* __restrict__ sum_inout, int sum_is_float, const long long* __restrict__ cnt, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const double s = sum_is_float ? static_cast<const double*>(sum_inout)[i]
                                  : (double)static_cast<const long long*>(sum_inout)[i];
    static_cast<double*>(sum_inout)[i] = s / (double)cnt[i];
  }
}

inline int grid_for(int64_t n) {
  int64_t g = (n + T * 4 - 1) / (T * 4);
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, kNumSMs * 16));
}

}  // namespace

cudaError_t launch_key_sum(const int32_t* kcode, const ColDesc& v, int64_t n, int kind, void* sum_k, cudaStream_t s,
                           int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_key_sum<<<grid_for(n), T, 0, s>>>(kcode, v, n, kind, sum_k);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_side_agg(const int32_t* kcode, const int32_t* gcode, const ColDesc& w, int64_t n,
                            const int32_t* cnt_o, const void* sum_o, int kind, int64_t NG,
                            unsigned long long* cnt_g, void* sum_g, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  if (NG <= kSmemGroups) {
    // enough tuples per block to amortize the per-block flush of NG accumulators
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(2 * kNumSMs, n / std::max<int64_t>(2048, 4 * NG)));
    k_side_agg<true><<<(int)blocks, T, 0, s>>>(kcode, gcode, w, n, cnt_o, sum_o, kind, (int)NG, cnt_g, sum_g);
  } else {
    k_side_agg<false><<<grid_for(n), T, 0, s>>>(kcode, gcode, w, n, cnt_o, sum_o, kind, (int)NG, cnt_g, sum_g);
  }
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_side_flags(const unsigned long long* cnt_g, int64_t NG, int32_t* flags, cudaStream_t s,
                              int64_t* launches) {
  if (NG <= 0) return cudaSuccess;
  k_side_flags<<<grid_for(NG), T, 0, s>>>(cnt_g, NG, flags);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_side_write(const unsigned long long* cnt_g, const void* sum_g, const int64_t* pos, int64_t NG,
                              int agg_kind, const SideOut& o, cudaStream_t s, int64_t* launches) {
  if (NG <= 0) return cudaSuccess;
  k_side_write<<<grid_for(NG), T, 0, s>>>(cnt_g, sum_g, pos, NG, agg_kind, o);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_avg_div(void* sum_inout, int sum_is_float, const long long* cnt, int64_t n, cudaStream_t s,
                           int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_avg_div<<<grid_for(n), T, 0, s>>>(sum_inout, sum_is_float, cnt, n);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
