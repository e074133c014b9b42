// partition.cu — multi-GPU row sharding: route the tuples of a
// table to P ranks by ranges of its group column — or, for the key-partitioned path
// (§8(f) f4), by a hash of its join key. Count pass (per-block smem histograms, one
// global atomic per destination per block), host exclusive scan of the P counts, scatter
// pass (warp-aggregated cursors) copying key, group and value columns.
#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

constexpr int T = 256;
constexpr int MAXP = 1024;

__device__ __forceinline__ int dest_of(long long g, const long long* bounds, int nb) {
  int lo = 0, hi = nb;  // number of bounds <= g
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (bounds[mid] <= g) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// destination of row i: the group range it falls in, or (by_key) a hash of its join key
// (fmix64, scaled to [0, P) by its high 32 bits)
__device__ __forceinline__ int dest_row(const ColDesc& key, const ColDesc& grp, int64_t i, const long long* sb, int P,
                                        int by_key) {
  if (by_key) {
    unsigned long long x = (unsigned long long)ld_int(key.data, key.type, i);
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return (int)(((x >> 32) * (unsigned long long)P) >> 32);
  }
  return dest_of(ld_int(grp.data, grp.type, i), sb, P - 1);
}

__global__ void k_part_count(ColDesc key, ColDesc grp, const long long* __restrict__ bounds, int P, int by_key,
                             unsigned long long* __restrict__ counts) {
  __shared__ long long sb[MAXP];
  __shared__ unsigned int sc[MAXP];
  for (int i = threadIdx.x; i < P; i += T) { sc[i] = 0; if (i < P - 1 && !by_key) sb[i] = bounds[i]; }
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < key.n; i += stride)
    atomicAdd(&sc[dest_row(key, grp, i, sb, P, by_key)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < P; i += T)
    if (sc[i]) atomicAdd(counts + i, (unsigned long long)sc[i]);
}

__global__ void k_part_scatter(ColDesc key, ColDesc grp, ColDesc val, const long long* __restrict__ bounds, int P,
                               int by_key, unsigned long long* __restrict__ cursor, void* __restrict__ ok,
                               void* __restrict__ og, void* __restrict__ ov) {
  __shared__ long long sb[MAXP];
  for (int i = threadIdx.x; i < P - 1 && !by_key; i += T) sb[i] = bounds[i];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * T;
  const int64_t n_round = (key.n + 31) & ~int64_t(31);
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n_round; i += stride) {
    const bool ok_ = i < key.n;
    const int d = ok_ ? dest_row(key, grp, i, sb, P, by_key) : -1 - lane_id();
    const unsigned act = __ballot_sync(0xffffffffu, ok_);
    const unsigned peers = __match_any_sync(0xffffffffu, d) & act;
    unsigned long long base = 0;
    const int leader = __ffs(peers) - 1;
    if (ok_ && leader == lane_id()) base = atomicAdd(cursor + d, (unsigned long long)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader < 0 ? 0 : leader);
    if (!ok_) continue;
    const int64_t pos = (int64_t)base + __popc(peers & lanemask_lt());
    if (key.type == 1) static_cast<long long*>(ok)[pos] = static_cast<const long long*>(key.data)[i];
    else static_cast<int*>(ok)[pos] = static_cast<const int*>(key.data)[i];
    if (grp.data) {
      if (grp.type == 1) static_cast<long long*>(og)[pos] = static_cast<const long long*>(grp.data)[i];
      else static_cast<int*>(og)[pos] = static_cast<const int*>(grp.data)[i];
    }
    if (val.data) {
      if (val.type == 1) static_cast<long long*>(ov)[pos] = static_cast<const long long*>(val.data)[i];
      else static_cast<int*>(ov)[pos] = static_cast<const int*>(val.data)[i];  // I32 or F32 bits
    }
  }
}

inline int grid_for(int64_t n) {
  int64_t g = (n + T * 4 - 1) / (T * 4);
  if (g < 1) g = 1;
  if (g > kNumSMs * 8) g = kNumSMs * 8;
  return (int)g;
}

}  // namespace

cudaError_t launch_part_count(const ColDesc& key, const ColDesc& grp, const long long* bounds, int P, int by_key,
                              unsigned long long* counts, cudaStream_t s, int64_t* launches) {
  if (P > MAXP) return cudaErrorInvalidValue;
  if (key.n <= 0) return cudaSuccess;
  k_part_count<<<grid_for(key.n), T, 0, s>>>(key, grp, bounds, P, by_key, counts);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_part_scatter(const ColDesc& key, const ColDesc& grp, const ColDesc& val, const long long* bounds,
                                int P, int by_key, unsigned long long* cursor, void* ok, void* og, void* ov,
                                cudaStream_t s, int64_t* launches) {
  if (P > MAXP) return cudaErrorInvalidValue;
  if (key.n <= 0) return cudaSuccess;
  k_part_scatter<<<grid_for(key.n), T, 0, s>>>(key, grp, val, bounds, P, by_key, cursor, ok, og, ov);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
