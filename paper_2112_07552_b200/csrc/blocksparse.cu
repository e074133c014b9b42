// blocksparse.cu — §8(f) f4: the block-sparse tensor-core path, the B200 form of the
// paper's TCU-SpMM (§4.2.4: operands in CSR, 16x16 tiles, all-zero
// submatrices skipped). Here the operands stay dense tcgen05 operands and the GEMM skips
// every (tile, K-block) product whose A or B block holds no tuple:
//   1. key reordering: each join key gets the smallest A row (group code) that uses it;
//      keys are re-coded in that order, so keys used by the same rows become neighbours
//      and block structure in the data (entity-matching blocks, communities) becomes
//      contiguous K-blocks;
//   2. base occupancy bitmaps at 16-row x 64-key granularity, straight from the tuples;
//   3. per GEMM launch, tile bitmaps (128-row A tiles / BN-row B tiles x the launch's
//      K-block width) OR-reduced from the base ones; the GEMM kernel iterates only the
//      K-blocks set in both (gemm_tc.cu for_active_kb) and writes all-zero tiles without
//      an accumulator;
//   4. the selector's dense cost is scaled by the active fraction of the products.
// The bitmaps are a superset of the nonzero structure (a cell with tuples summing to 0
// keeps its bit), so the result is the dense product's, bit for bit on the integer paths.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

constexpr int T = 256;

inline int grid_for(int64_t n) {
  int64_t g = (n + T * 4 - 1) / (T * 4);
  if (g < 1) g = 1;
  if (g > kNumSMs * 16) g = kNumSMs * 16;
  return (int)g;
}

__global__ void k_bs_minrow(const int32_t* __restrict__ kcode, const int32_t* __restrict__ rcode, int64_t n,
                            int32_t* __restrict__ minrow) {
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += (int64_t)gridDim.x * T) {
    const int32_t k = kcode[i];
    if (k < 0) continue;
    const int32_t r = rcode[i];
    if (r < __ldg(minrow + k)) atomicMin(minrow + k, r);
  }
}

// sort keys by minrow (the radix sort is stable: ties keep ascending codes)
__global__ void k_bs_sortkeys(const int32_t* __restrict__ minrow, int64_t K, unsigned long long* __restrict__ keys,
                              uint32_t* __restrict__ vals) {
  for (int64_t k = (int64_t)blockIdx.x * T + threadIdx.x; k < K; k += (int64_t)gridDim.x * T) {
    keys[k] = (unsigned long long)(uint32_t)minrow[k];
    vals[k] = (uint32_t)k;
  }
}

__global__ void k_bs_clamp(unsigned long long* __restrict__ keys, int64_t K, unsigned long long G) {
  for (int64_t k = (int64_t)blockIdx.x * T + threadIdx.x; k < K; k += (int64_t)gridDim.x * T)
    if (keys[k] > G) keys[k] = G;
}

__global__ void k_bs_invert(const uint32_t* __restrict__ sorted_vals, int64_t K, int32_t* __restrict__ perm) {
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < K; i += (int64_t)gridDim.x * T)
    perm[sorted_vals[i]] = (int32_t)i;
}

__global__ void k_bs_permute_cnt(const int32_t* __restrict__ in, const int32_t* __restrict__ perm, int64_t K,
                                 int32_t* __restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * T + threadIdx.x; k < K; k += (int64_t)gridDim.x * T) out[perm[k]] = in[k];
}

// base bitmap: word (r / 16) * W + (k / 64) / 64, bit (k / 64) % 64
__global__ void k_bs_mark(const int32_t* __restrict__ kcode, const int32_t* __restrict__ rcode, int64_t n, int W,
                          unsigned long long* __restrict__ bm) {
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += (int64_t)gridDim.x * T) {
    const int32_t k = kcode[i];
    if (k < 0) continue;
    const int32_t r = rcode[i];
    const int kg = k >> 6;
    unsigned long long* w = bm + (int64_t)(r >> 4) * W + (kg >> 6);
    const unsigned long long bit = 1ull << (kg & 63);
    if (!(__ldcg(w) & bit)) atomicOr(w, bit);
  }
}

// tile bitmaps: tile t covers base row groups [t * rpt, (t + 1) * rpt) (clipped), bit kb of
// the launch's K-block space <- key groups [(kb mod period) * f, + f). One thread per
// (tile, K-block); a warp's 32 bits leave as one 32-bit half of a bitmap word.
__global__ void k_bs_derive(const unsigned long long* __restrict__ base, int base_rows, int W, int rpt, int f,
                            int64_t period_kb, int64_t total_kb, int ntiles, int Wout,
                            unsigned* __restrict__ out32) {
  const int64_t per_tile = (int64_t)Wout * 64;  // K-block slots per tile (padded to whole words)
  const int64_t nthr = (int64_t)ntiles * per_tile;
  for (int64_t x = (int64_t)blockIdx.x * T + threadIdx.x; x < nthr; x += (int64_t)gridDim.x * T) {
    const int t = (int)(x / per_tile);
    const int64_t kb = x - (int64_t)t * per_tile;
    bool any = false;
    if (kb < total_kb) {
      const int g0 = t * rpt, g1 = min(base_rows, g0 + rpt);
      const int64_t kg0 = (kb % period_kb) * f;
      for (int g = g0; g < g1 && !any; ++g) {
        const unsigned long long* row = base + (int64_t)g * W;
        for (int q = 0; q < f; ++q) {
          const int64_t kg = kg0 + q;
          if ((__ldg(row + (kg >> 6)) >> (kg & 63)) & 1ull) { any = true; break; }
        }
      }
    }
    const unsigned bits = __ballot_sync(0xffffffffu, any);  // per_tile % 64 == 0: warps never straddle tiles
    if (lane_id() == 0) out32[x >> 5] = bits;
  }
}

__global__ void k_bs_active(const unsigned long long* __restrict__ a, const unsigned long long* __restrict__ b,
                            int tiles_m, int tiles_n, int Wt, unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  const int64_t np = (int64_t)tiles_m * tiles_n;
  for (int64_t x = (int64_t)blockIdx.x * T + threadIdx.x; x < np; x += (int64_t)gridDim.x * T) {
    const int m = (int)(x / tiles_n), nn = (int)(x - (int64_t)m * tiles_n);
    for (int w = 0; w < Wt; ++w) c += __popcll(a[(int64_t)m * Wt + w] & b[(int64_t)nn * Wt + w]);
  }
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(out, c);
}

}  // namespace

size_t bs_reorder_temp_bytes(int64_t K) {
  return (size_t)K * (4 + 8 + 8 + 4 + 4 + 4) + radix_temp_bytes(K) + 1024;
}

cudaError_t launch_bs_reorder(int32_t* kA, const int32_t* gA, int64_t nA, int32_t* kB, int64_t nB, int32_t* cntA,
                              int32_t* cntB, int64_t K, int64_t G, void* temp, cudaStream_t s, int64_t* launches) {
  if (K <= 0) return cudaSuccess;
  char* t = static_cast<char*>(temp);
  auto take = [&](size_t bytes) { char* p = t; t += (bytes + 255) / 256 * 256; return p; };
  int32_t* minrow = reinterpret_cast<int32_t*>(take((size_t)K * 4));
  auto* k0 = reinterpret_cast<unsigned long long*>(take((size_t)K * 8));
  auto* k1 = reinterpret_cast<unsigned long long*>(take((size_t)K * 8));
  auto* v0 = reinterpret_cast<uint32_t*>(take((size_t)K * 4));
  auto* v1 = reinterpret_cast<uint32_t*>(take((size_t)K * 4));
  int32_t* perm = reinterpret_cast<int32_t*>(take((size_t)K * 4));
  void* rtmp = take(radix_temp_bytes(K));
  cudaError_t e = cudaMemsetAsync(minrow, 0x7F, (size_t)K * 4, s);  // 0x7F7F7F7F: after every row
  if (e != cudaSuccess) return e;
  k_bs_minrow<<<grid_for(nA), T, 0, s>>>(kA, gA, nA, minrow);
  k_bs_sortkeys<<<grid_for(K), T, 0, s>>>(minrow, K, k0, v0);
  bool alt = false;
  // minrow < G, or the "no A row" marker 0x7F7F7F7F: sort only the bits that can differ
  int bits = 32;
  if (G < (1ll << 24)) {
    // keys without an A tuple sort last either way: clamp their marker to G
    bits = 8;
    while (bits < 32 && ((int64_t)1 << bits) <= G) bits += 8;
    k_bs_clamp<<<grid_for(K), T, 0, s>>>(k0, K, (unsigned long long)G);
  }
  if ((e = radix_sort_pairs(k0, v0, k1, v1, K, bits, rtmp, s, launches, &alt)) != cudaSuccess) return e;
  k_bs_invert<<<grid_for(K), T, 0, s>>>(alt ? v1 : v0, K, perm);
  if ((e = launch_remap_codes(kA, nA, perm, s, launches)) != cudaSuccess) return e;
  if ((e = launch_remap_codes(kB, nB, perm, s, launches)) != cudaSuccess) return e;
  // per-key counts follow their keys (minrow is free again: scratch for the copy)
  k_bs_permute_cnt<<<grid_for(K), T, 0, s>>>(cntA, perm, K, minrow);
  cudaMemcpyAsync(cntA, minrow, (size_t)K * 4, cudaMemcpyDeviceToDevice, s);
  k_bs_permute_cnt<<<grid_for(K), T, 0, s>>>(cntB, perm, K, minrow);
  cudaMemcpyAsync(cntB, minrow, (size_t)K * 4, cudaMemcpyDeviceToDevice, s);
  if (launches) *launches += 5;
  return cudaGetLastError();
}

cudaError_t launch_bs_mark(const int32_t* kcode, const int32_t* rcode, int64_t n, int W, unsigned long long* bm,
                           cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_bs_mark<<<grid_for(n), T, 0, s>>>(kcode, rcode, n, W, bm);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_bs_derive(const unsigned long long* base, int base_rows, int W, int rows_per_tile, int f,
                             int64_t period_kb, int64_t total_kb, int ntiles, int Wout, unsigned long long* out,
                             cudaStream_t s, int64_t* launches) {
  if (rows_per_tile % 16) return cudaErrorInvalidValue;
  // one thread per (tile, K-block slot): the grid covers whole warps (ntiles * Wout * 64 threads)
  const int64_t nthr = (int64_t)ntiles * Wout * 64;
  const int grid = (int)std::min<int64_t>((nthr + T - 1) / T, (int64_t)kNumSMs * 32);
  k_bs_derive<<<grid, T, 0, s>>>(base, base_rows, W, rows_per_tile / 16, f, period_kb, total_kb, ntiles, Wout,
                                 reinterpret_cast<unsigned*>(out));
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_bs_active(const unsigned long long* a, const unsigned long long* b, int tiles_m, int tiles_n,
                             int Wt, unsigned long long* out, cudaStream_t s, int64_t* launches) {
  k_bs_active<<<grid_for((int64_t)tiles_m * tiles_n), T, 0, s>>>(a, b, tiles_m, tiles_n, Wt, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
