// tri_sparse.cu — §8(f) f3: the sparse triangle path (wedge check) for step a9.
//
// PAPER.md §3.2's chain exception evaluates the triangle query as a
// matrix product chain, T = trace(A³) / 6 on the symmetrised 0/1 adjacency; the
// dense form (gemm_tc.cu EPI_TRI) costs 2·V³ operations — 5.6e14 at c3's 65,536
// vertex ids, while the graph has only ~1 M edges. Here the same count is taken
// on the sparse graph (reading R15: simple undirected graph):
//   1. canonical undirected edges (min, max) of the coded endpoints, self-loops
//      dropped, sorted (LSD radix) and de-duplicated;
//   2. degrees; every edge is oriented from the endpoint with the smaller
//      (degree, id) to the larger, so each triangle is found exactly once and
//      every out-list has at most sqrt(2m) entries;
//   3. out-lists in CSR (counting sort by source);
//   4. one CTA per vertex u (ticket-scheduled): the bits of N+(u) in a shared-memory
//      bitmap over all V vertices, then every wedge u -> v -> w with v in N+(u)
//      tests bit w; the bits are cleared again after the count.
// T = number of hits (each triangle counted once through its lowest-ranked vertex).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

constexpr int T = 256;

inline int grid_for(int64_t n) {
  int64_t g = (n + T * 4 - 1) / (T * 4);
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, kNumSMs * 16));
}

// canonical key (min << bits | max) of the coded endpoints; self-loops get the all-ones
// sentinel (sorted last; a real edge cannot equal it because min < max)
__global__ void k_tri_keys(const int32_t* __restrict__ cu, const int32_t* __restrict__ cv, int64_t n, int bits,
                           unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t stride = (int64_t)gridDim.x * T;
  const unsigned long long sentinel = (1ull << (2 * bits)) - 1ull;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const unsigned a = (unsigned)cu[i], b = (unsigned)cv[i];
    keys[i] = a == b ? sentinel : ((unsigned long long)min(a, b) << bits) | max(a, b);
    vals[i] = 0;
  }
}

// unique edges (first of each run of equal sorted keys, self-loops excluded): flag
__global__ void k_tri_unique_flags(const unsigned long long* __restrict__ k, int64_t n, int bits,
                                   int32_t* __restrict__ flag) {
  const int64_t stride = (int64_t)gridDim.x * T;
  const unsigned long long sentinel = (1ull << (2 * bits)) - 1ull;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride)
    flag[i] = k[i] != sentinel && (i == 0 || k[i] != k[i - 1]);
}

__global__ void k_tri_compact_deg(const unsigned long long* __restrict__ k, const int32_t* __restrict__ flag,
                                  const int64_t* __restrict__ pos, int64_t n, int bits, int32_t* __restrict__ eu,
                                  int32_t* __restrict__ ev, int32_t* __restrict__ deg) {
  const int64_t stride = (int64_t)gridDim.x * T;
  const unsigned long long lo = (1ull << bits) - 1ull;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    if (!flag[i]) continue;
    const int32_t a = (int32_t)(k[i] >> bits), b = (int32_t)(k[i] & lo);
    eu[pos[i]] = a;
    ev[pos[i]] = b;
    atomicAdd(deg + a, 1);
    atomicAdd(deg + b, 1);
  }
}

__device__ __forceinline__ bool tri_before(int32_t a, int32_t b, const int32_t* __restrict__ deg) {
  const int32_t da = deg[a], db = deg[b];
  return da < db || (da == db && a < b);
}

// orient each unique edge; count out-degrees (pass 0) or place into CSR (pass 1)
__global__ void k_tri_orient(const int32_t* __restrict__ eu, const int32_t* __restrict__ ev, int64_t m,
                             const int32_t* __restrict__ deg, int32_t* __restrict__ odeg,
                             const int64_t* __restrict__ ooff, int32_t* __restrict__ ocur,
                             int32_t* __restrict__ adj, int pass) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < m; i += stride) {
    int32_t a = eu[i], b = ev[i];
    if (!tri_before(a, b, deg)) { const int32_t t = a; a = b; b = t; }
    if (pass == 0) atomicAdd(odeg + a, 1);
    else adj[ooff[a] + atomicAdd(ocur + a, 1)] = b;
  }
}

// one CTA per vertex (ticket order): bitmap of N+(u), wedge checks u -> v -> w
__global__ void __launch_bounds__(512) k_tri_count(const int64_t* __restrict__ ooff, const int32_t* __restrict__ adj,
                                                   int64_t V, unsigned long long* __restrict__ ticket,
                                                   unsigned long long* __restrict__ out) {
  extern __shared__ unsigned bm[];
  __shared__ int64_t s_u;
  const int64_t words = (V + 31) / 32;
  for (int64_t i = threadIdx.x; i < words; i += blockDim.x) bm[i] = 0u;
  unsigned long long cnt = 0;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_u = (int64_t)atomicAdd(ticket, 1ull);
    __syncthreads();
    const int64_t u = s_u;
    if (u >= V) break;
    const int64_t b0 = ooff[u], b1 = ooff[u + 1];
    if (b1 - b0 < 2) continue;  // a triangle needs two out-neighbours
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      const int32_t v = adj[i];
      atomicOr(bm + (v >> 5), 1u << (v & 31));
    }
    __syncthreads();
    // warps take the out-neighbours v; lanes walk N+(v)
    const int wid = warp_id(), nw = (int)(blockDim.x >> 5), lane = lane_id();
    for (int64_t i = b0 + wid; i < b1; i += nw) {
      const int32_t v = adj[i];
      const int64_t c0 = ooff[v], c1 = ooff[v + 1];
      for (int64_t j = c0 + lane; j < c1; j += 32) {
        const int32_t w = __ldg(adj + j);
        cnt += (bm[w >> 5] >> (w & 31)) & 1u;
      }
    }
    __syncthreads();
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
      const int32_t v = adj[i];
      bm[v >> 5] = 0u;
    }
  }
  cnt = warp_sum(cnt);
  if (lane_id() == 0 && cnt) atomicAdd(out, cnt);
}

}  // namespace

size_t tri_sparse_temp_bytes(int64_t n, int64_t V) {
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  return 2 * al(n * 8) + 2 * al(n * 4) + al(radix_temp_bytes(n)) + al(n * 4) + al((n + 1) * 8) +
         al(scan_temp_bytes(std::max<int64_t>(n, V + 1))) + 2 * al(n * 4) + 3 * al((V + 1) * 4) + al((V + 1) * 8) +
         al(n * 4) + 256;
}

size_t tri_sparse_smem(int64_t V) { return (size_t)((V + 31) / 32) * 4; }

cudaError_t launch_tri_sparse(const int32_t* cu, const int32_t* cv, int64_t n, int64_t V, void* temp,
                              unsigned long long* out, cudaStream_t s, int64_t* launches) {
  if (n <= 0 || V <= 0) return cudaSuccess;
  const size_t smem = tri_sparse_smem(V);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  char* t = static_cast<char*>(temp);
  auto take = [&](size_t bytes) { char* p = t; t += al(bytes); return p; };
  auto* k0 = reinterpret_cast<unsigned long long*>(take(n * 8));
  auto* k1 = reinterpret_cast<unsigned long long*>(take(n * 8));
  auto* v0 = reinterpret_cast<uint32_t*>(take(n * 4));
  auto* v1 = reinterpret_cast<uint32_t*>(take(n * 4));
  void* rtmp = take(radix_temp_bytes(n));
  auto* flag = reinterpret_cast<int32_t*>(take(n * 4));
  auto* pos = reinterpret_cast<int64_t*>(take((n + 1) * 8));
  void* stmp = take(scan_temp_bytes(std::max<int64_t>(n, V + 1)));
  auto* eu = reinterpret_cast<int32_t*>(take(n * 4));
  auto* ev = reinterpret_cast<int32_t*>(take(n * 4));
  auto* deg = reinterpret_cast<int32_t*>(take((V + 1) * 4));
  auto* odeg = reinterpret_cast<int32_t*>(take((V + 1) * 4));
  auto* ocur = reinterpret_cast<int32_t*>(take((V + 1) * 4));
  auto* ooff = reinterpret_cast<int64_t*>(take((V + 1) * 8));
  auto* adj = reinterpret_cast<int32_t*>(take(n * 4));
  cudaError_t e;
  int bits = 1;
  while ((1ll << bits) < V) ++bits;  // bits per endpoint code
  k_tri_keys<<<grid_for(n), T, 0, s>>>(cu, cv, n, bits, k0, v0);
  bool alt = false;
  if ((e = radix_sort_pairs(k0, v0, k1, v1, n, (2 * bits + 7) / 8 * 8, rtmp, s, launches, &alt)) != cudaSuccess)
    return e;
  const unsigned long long* ks = alt ? k1 : k0;
  k_tri_unique_flags<<<grid_for(n), T, 0, s>>>(ks, n, bits, flag);
  if ((e = exclusive_scan_i32(flag, pos, n, pos + n, stmp, s, launches)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(deg, 0, (V + 1) * 4, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(odeg, 0, (V + 1) * 4, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(ocur, 0, (V + 1) * 4, s)) != cudaSuccess) return e;
  k_tri_compact_deg<<<grid_for(n), T, 0, s>>>(ks, flag, pos, n, bits, eu, ev, deg);
  int64_t m = 0;  // unique undirected edges
  if ((e = cudaMemcpyAsync(&m, pos + n, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  if (m > 0) {
    k_tri_orient<<<grid_for(m), T, 0, s>>>(eu, ev, m, deg, odeg, nullptr, nullptr, nullptr, 0);
    if ((e = exclusive_scan_i32(odeg, ooff, V, ooff + V, stmp, s, launches)) != cudaSuccess) return e;
    k_tri_orient<<<grid_for(m), T, 0, s>>>(eu, ev, m, deg, nullptr, ooff, ocur, adj, 1);
    if ((e = set_func_attr(k_tri_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)) !=
        cudaSuccess)
      return e;
    unsigned long long* ticket = reinterpret_cast<unsigned long long*>(ocur);  // reused: 8 bytes, zeroed below
    if ((e = cudaMemsetAsync(ticket, 0, 8, s)) != cudaSuccess) return e;
    const int per_sm = smem <= 48 * 1024 ? 4 : smem <= 100 * 1024 ? 2 : 1;
    k_tri_count<<<(unsigned)std::min<int64_t>(V, (int64_t)per_sm * kNumSMs), 512, smem, s>>>(ooff, adj, V, ticket, out);
  }
  if (launches) *launches += 7;
  return cudaGetLastError();
}

}  // namespace tcudb
