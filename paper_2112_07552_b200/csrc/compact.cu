// compact.cu — step a8: nonzero compaction + decode of the result matrix.
//
// PAPER.md §3.2: nonzero(M) = {(i,j) | M_ij > 0} turns the result
// matrix back into a table on the GPU; §3.1 a pair is in the join
// iff C_ij > 0; Lemma Q3 (read as M_{1,j} per reading R4).
// Existence is decided on a COUNT plane (or on C itself when the guard proved
// that C != 0 <=> COUNT > 0; reading R3), so SUM = 0 groups are kept.
//
// Two passes over the G x H region (row-major tiles of 4096 columns per
// 256-thread block, 16 consecutive cells per thread): count -> scan -> write.
// Codes are ascending dense ranks, so row-major order is (g, h) order and the
// ORDER BY comes for free (§3.4). Decode: g = dict_g[i], h = dict_h[j].
#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

constexpr int T = 256;
constexpr int PER = 16;
constexpr int TW = T * PER;  // columns per block tile

__device__ __forceinline__ void load16(const void* base, int kind, int64_t ld, int64_t row, int64_t col0,
                                       int64_t H, double* out, bool* nz) {
  // Reads 16 consecutive cells (col0 .. col0+15) of one row; cells >= H are zero.
  const bool full = col0 + PER <= H;
  if (kind == 0 || kind == 2) {
    const uint32_t* p = static_cast<const uint32_t*>(base) + row * ld + col0;
    uint32_t v[PER];
    if (full) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 x = reinterpret_cast<const uint4*>(p)[q];
        v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < PER; ++j) v[j] = (col0 + j < H) ? p[j] : 0u;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (kind == 0) { out[j] = (double)(int)v[j]; nz[j] = v[j] != 0u; }
      else { const float f = __uint_as_float(v[j]); out[j] = (double)f; nz[j] = f != 0.f; }
    }
  } else {
    const unsigned long long* p = static_cast<const unsigned long long*>(base) + row * ld + col0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const unsigned long long v = (col0 + j < H) ? p[j] : 0ull;
      if (kind == 1) { out[j] = 0; nz[j] = v != 0ull; }
      else { const double d = __longlong_as_double((long long)v); out[j] = d; nz[j] = d != 0.0; }
    }
  }
}

__device__ __forceinline__ int exist16(const CompactArgs& a, int64_t row, int64_t col0, bool* nz) {
  double tmp[PER];
  load16(a.E, a.e_kind, a.lde, row, col0, a.H, tmp, nz);
  int c = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) c += nz[j];
  return c;
}

__global__ void __launch_bounds__(T) k_compact_count(const CompactArgs a, int64_t tiles_per_row,
                                                     int32_t* __restrict__ cnt) {
  const int64_t b = blockIdx.x;
  const int64_t row = b / tiles_per_row;
  const int64_t col0 = (b - row * tiles_per_row) * TW + (int64_t)threadIdx.x * PER;
  bool nz[PER];
  int c = col0 < a.H ? exist16(a, row, col0, nz) : 0;
  c = warp_sum(c);
  __shared__ int s[T / 32];
  if (lane_id() == 0) s[warp_id()] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < T / 32; ++w) t += s[w];
    cnt[b] = t;
  }
}

__global__ void __launch_bounds__(T) k_compact_write(const CompactArgs a, int64_t tiles_per_row,
                                                     const int64_t* __restrict__ off) {
  const int64_t b = blockIdx.x;
  const int64_t row = b / tiles_per_row;
  const int64_t col0 = (b - row * tiles_per_row) * TW + (int64_t)threadIdx.x * PER;
  bool nz[PER];
  int c = 0;
  if (col0 < a.H) c = exist16(a, row, col0, nz);
  else {
#pragma unroll
    for (int j = 0; j < PER; ++j) nz[j] = false;
  }
  int x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o); if (lane_id() >= o) x += y; }
  __shared__ int wt[T / 32];
  if (lane_id() == 31) wt[warp_id()] = x;
  __syncthreads();
  if (c == 0) return;
  int wp = 0;
  for (int w = 0; w < warp_id(); ++w) wp += wt[w];
  int64_t pos = off[b] + wp + x - c;
  double val[PER];
  bool dummy[PER];
  if (a.v_kind != 1) load16(a.V, a.v_kind, a.ldv, row, col0, a.H, val, dummy);
  const long long gval = a.dict_g[row];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (!nz[j]) continue;
    const long long hval = a.dict_h[col0 + j];
    if (a.g_out_type == 1) static_cast<long long*>(a.out_g)[pos] = gval;
    else static_cast<int*>(a.out_g)[pos] = (int)gval;
    if (a.h_out_type == 1) static_cast<long long*>(a.out_h)[pos] = hval;
    else static_cast<int*>(a.out_h)[pos] = (int)hval;
    if (a.agg_out == 0) {
      long long v;
      if (a.v_kind == 1) v = static_cast<const long long*>(a.V)[row * a.ldv + col0 + j];
      else v = (long long)val[j];  // int32 / f32 paths are exact in double
      static_cast<long long*>(a.out_agg)[pos] = v;
    } else {
      static_cast<double*>(a.out_agg)[pos] = val[j];
    }
    ++pos;
  }
}

}  // namespace

size_t compact_temp_bytes(int64_t G, int64_t H) {
  const int64_t tpr = (H + TW - 1) / TW;
  const int64_t nb = G * tpr;
  return ((size_t)nb * 4 + 15) / 16 * 16 + (size_t)nb * 8 + scan_temp_bytes(nb) + 64;
}

cudaError_t launch_compact_count(const CompactArgs& a, int64_t* nnz_dev, void* temp, cudaStream_t s,
                                 int64_t* launches) {
  const int64_t tpr = (a.H + TW - 1) / TW;
  const int64_t nb = a.G * tpr;
  int32_t* cnt = static_cast<int32_t*>(temp);
  int64_t* off = reinterpret_cast<int64_t*>(static_cast<char*>(temp) + ((size_t)nb * 4 + 15) / 16 * 16);
  if (nb <= 0) return exclusive_scan_i32(nullptr, nullptr, 0, nnz_dev, off, s, launches);
  if (nb > 0x7fffffffLL) return cudaErrorInvalidValue;
  k_compact_count<<<(unsigned)nb, T, 0, s>>>(a, tpr, cnt);
  if (launches) ++*launches;
  return exclusive_scan_i32(cnt, off, nb, nnz_dev, off + nb, s, launches);
}

cudaError_t launch_compact_write(const CompactArgs& a, void* temp, cudaStream_t s, int64_t* launches) {
  const int64_t tpr = (a.H + TW - 1) / TW;
  const int64_t nb = a.G * tpr;
  if (nb <= 0) return cudaSuccess;
  const int64_t* off = reinterpret_cast<const int64_t*>(static_cast<char*>(temp) + ((size_t)nb * 4 + 15) / 16 * 16);
  k_compact_write<<<(unsigned)nb, T, 0, s>>>(a, tpr, off);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
