// scan_sort.cu — device-wide exclusive scan and LSD radix sort (key u64 + u32
// payload) used by the encoder (a2), the compaction (a8) and the sparse path (a7).
#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace tcudb {
namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;  // 4096

template <typename T>
__device__ __forceinline__ int64_t ld_as_i64(const T* p, int64_t i) { return (int64_t)p[i]; }

// Block-wide exclusive scan of one int64 per thread; returns the block total.
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t& excl) {
  __shared__ int64_t warp_tot[SCAN_THREADS / 32];
  const int lane = lane_id(), w = warp_id();
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  int64_t wpre = 0, tot = 0;
#pragma unroll
  for (int i = 0; i < SCAN_THREADS / 32; ++i) {
    const int64_t t = warp_tot[i];
    if (i < w) wpre += t;
    tot += t;
  }
  __syncthreads();
  excl = wpre + x - v;
  return tot;
}

template <typename T>
__global__ void k_tile_reduce(const T* __restrict__ in, int64_t n, int64_t* __restrict__ partial) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    const int64_t idx = base + (int64_t)i * SCAN_THREADS + threadIdx.x;
    if (idx < n) s += ld_as_i64(in, idx);
  }
  int64_t ex;
  const int64_t tot = block_exclusive_scan(s, ex);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// Exclusive scan of one tile with a carry-in; the thread owns SCAN_ITEMS consecutive items.
template <typename T>
__global__ void k_tile_scan(const T* __restrict__ in, int64_t* __restrict__ out, int64_t n,
                            const int64_t* __restrict__ carry, int64_t* __restrict__ total) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    const int64_t idx = base + i;
    v[i] = idx < n ? ld_as_i64(in, idx) : 0;
    s += v[i];
  }
  int64_t ex;
  const int64_t tot = block_exclusive_scan(s, ex);
  const int64_t c = carry ? carry[blockIdx.x] : 0;
  int64_t run = c + ex;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    const int64_t idx = base + i;
    if (idx < n) out[idx] = run;
    run += v[i];
  }
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *total = c + tot;
}

__global__ void k_set_zero(int64_t* p) { *p = 0; }

template <typename T>
cudaError_t scan_impl(const T* in, int64_t* out, int64_t n, int64_t* total, int64_t* temp, cudaStream_t s,
                      int64_t* launches) {
  if (n <= 0) {
    if (total) { k_set_zero<<<1, 1, 0, s>>>(total); if (launches) ++*launches; }
    return cudaGetLastError();
  }
  const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (nb == 1) {
    k_tile_scan<T><<<1, SCAN_THREADS, 0, s>>>(in, out, n, nullptr, total);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  int64_t* partial = temp;
  k_tile_reduce<T><<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, n, partial);
  if (launches) ++*launches;
  cudaError_t e = scan_impl<int64_t>(partial, partial, nb, nullptr, temp + nb, s, launches);
  if (e != cudaSuccess) return e;
  k_tile_scan<T><<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, out, n, partial, total);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------ radix sort
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 4096; warp w owns items [w*512, (w+1)*512)

__global__ void k_radix_hist(const uint64_t* __restrict__ keys, int64_t n, int shift, int32_t* __restrict__ hist,
                             int nblocks) {
  __shared__ int32_t h[256];
  for (int i = threadIdx.x; i < 256; i += RS_THREADS) h[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
  for (int i = threadIdx.x; i < RS_TILE; i += RS_THREADS) {
    const int64_t idx = base + i;
    if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 0xFF], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += RS_THREADS) hist[(int64_t)d * nblocks + blockIdx.x] = h[d];
}

__global__ void k_radix_scatter(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t n,
                                int shift, const int64_t* __restrict__ offs, int nblocks,
                                uint64_t* __restrict__ okeys, uint32_t* __restrict__ ovals) {
  __shared__ int32_t wcnt[RS_WARPS][256];
  __shared__ int64_t boff[256];
  const int w = warp_id(), lane = lane_id();
  for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&wcnt[0][0])[i] = 0;
  for (int d = threadIdx.x; d < 256; d += RS_THREADS) boff[d] = offs[(int64_t)d * nblocks + blockIdx.x];
  __syncthreads();
  const int64_t wbase = (int64_t)blockIdx.x * RS_TILE + (int64_t)w * (RS_TILE / RS_WARPS);
  // pass 1: per-warp digit counts
  for (int r = 0; r < RS_TILE / RS_WARPS / 32; ++r) {
    const int64_t idx = wbase + r * 32 + lane;
    const bool ok = idx < n;
    const uint32_t d = ok ? (uint32_t)((keys[idx] >> shift) & 0xFF) : 0x100u + lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (ok && (peers >> lane) == 1u) wcnt[w][d] += __popc(peers);  // highest peer lane adds
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan across warps per digit -> warp base offsets (in place)
  for (int d = threadIdx.x; d < 256; d += RS_THREADS) {
    int32_t run = 0;
    for (int ww = 0; ww < RS_WARPS; ++ww) { const int32_t c = wcnt[ww][d]; wcnt[ww][d] = run; run += c; }
  }
  __syncthreads();
  // pass 2: stable scatter
  for (int r = 0; r < RS_TILE / RS_WARPS / 32; ++r) {
    const int64_t idx = wbase + r * 32 + lane;
    const bool ok = idx < n;
    const uint64_t k = ok ? keys[idx] : 0;
    const uint32_t d = ok ? (uint32_t)((k >> shift) & 0xFF) : 0x100u + lane;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (ok) {
      const int32_t rank = wcnt[w][d] + __popc(peers & lanemask_lt());
      const int64_t pos = boff[d] + rank;
      okeys[pos] = k;
      ovals[pos] = vals[idx];
    }
    __syncwarp();
    if (ok && (peers >> lane) == 1u) wcnt[w][d] += __popc(peers);
    __syncwarp();
  }
}

}  // namespace

size_t scan_temp_bytes(int64_t n) {
  size_t total = 0;
  int64_t m = n;
  while (m > SCAN_TILE) { m = (m + SCAN_TILE - 1) / SCAN_TILE; total += (size_t)m; }
  return (total + 8) * sizeof(int64_t);
}

cudaError_t exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total, void* temp,
                               cudaStream_t s, int64_t* launches) {
  return scan_impl<int64_t>(in, out, n, total, static_cast<int64_t*>(temp), s, launches);
}
cudaError_t exclusive_scan_i32(const int32_t* in, int64_t* out, int64_t n, int64_t* total, void* temp,
                               cudaStream_t s, int64_t* launches) {
  return scan_impl<int32_t>(in, out, n, total, static_cast<int64_t*>(temp), s, launches);
}

size_t radix_temp_bytes(int64_t n) {
  const int64_t nb = (n + RS_TILE - 1) / RS_TILE;
  const int64_t h = nb * 256;
  return (size_t)h * sizeof(int32_t) + (size_t)h * sizeof(int64_t) + scan_temp_bytes(h) + 256;
}

cudaError_t radix_sort_pairs(unsigned long long* keys_, uint32_t* vals, unsigned long long* keys_alt_,
                             uint32_t* vals_alt, int64_t n, int bits, void* temp, cudaStream_t s, int64_t* launches,
                             bool* result_in_alt) {
  uint64_t* keys = reinterpret_cast<uint64_t*>(keys_);
  uint64_t* keys_alt = reinterpret_cast<uint64_t*>(keys_alt_);
  *result_in_alt = false;
  if (n <= 1) return cudaSuccess;
  const int nb = (int)((n + RS_TILE - 1) / RS_TILE);
  const int64_t h = (int64_t)nb * 256;
  int32_t* hist = static_cast<int32_t*>(temp);
  int64_t* offs = reinterpret_cast<int64_t*>(static_cast<char*>(temp) + ((h * sizeof(int32_t) + 15) & ~size_t(15)));
  void* stemp = reinterpret_cast<char*>(offs) + h * sizeof(int64_t);
  uint64_t *ki = keys, *ko = keys_alt;
  uint32_t *vi = vals, *vo = vals_alt;
  for (int shift = 0; shift < bits; shift += 8) {
    k_radix_hist<<<nb, RS_THREADS, 0, s>>>(ki, n, shift, hist, nb);
    if (launches) ++*launches;
    cudaError_t e = exclusive_scan_i32(hist, offs, h, nullptr, stemp, s, launches);
    if (e != cudaSuccess) return e;
    k_radix_scatter<<<nb, RS_THREADS, 0, s>>>(ki, vi, n, shift, offs, nb, ko, vo);
    if (launches) ++*launches;
    std::swap(ki, ko);
    std::swap(vi, vo);
    *result_in_alt = !*result_in_alt;
  }
  return cudaGetLastError();
}

}  // namespace tcudb
