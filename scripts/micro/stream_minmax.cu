// Micro-benchmark: streaming min/max over 6 x 67M int32 columns, several load schedules.
#include <cstdio>
#include <cstdint>
#include <climits>
#include <cuda_runtime.h>
__device__ long long g_out[16];
__device__ __forceinline__ int4 ldv(const int4* p) {
  int4 v;
  asm volatile("ld.global.cs.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
template <int U>
__global__ void k_mm(const int4* const* cols, int64_t n4) {
  const int4* p = cols[blockIdx.y];
  int mn = INT_MAX, mx = INT_MIN;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += U * stride) {
    int4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = ldv(p + min(i0 + u * stride, n4 - 1));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      mn = min(mn, min(min(x[u].x, x[u].y), min(x[u].z, x[u].w)));
      mx = max(mx, max(max(x[u].x, x[u].y), max(x[u].z, x[u].w)));
    }
  }
  for (int o = 16; o; o >>= 1) { mn = min(mn, __shfl_xor_sync(~0u, mn, o)); mx = max(mx, __shfl_xor_sync(~0u, mx, o)); }
  if ((threadIdx.x & 31) == 0) { atomicMin(&g_out[0], (long long)mn); atomicMax(&g_out[1], (long long)mx); }
}
// contiguous chunk per block (each block streams its own contiguous range)
template <int U>
__global__ void k_mm_chunk(const int4* const* cols, int64_t n4, int64_t chunk) {
  const int4* p = cols[blockIdx.y];
  int mn = INT_MAX, mx = INT_MIN;
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(n4, lo + chunk);
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += U * blockDim.x) {
    int4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = ldv(p + min(i0 + u * (int64_t)blockDim.x, hi - 1));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      mn = min(mn, min(min(x[u].x, x[u].y), min(x[u].z, x[u].w)));
      mx = max(mx, max(max(x[u].x, x[u].y), max(x[u].z, x[u].w)));
    }
  }
  for (int o = 16; o; o >>= 1) { mn = min(mn, __shfl_xor_sync(~0u, mn, o)); mx = max(mx, __shfl_xor_sync(~0u, mx, o)); }
  if ((threadIdx.x & 31) == 0) { atomicMin(&g_out[0], (long long)mn); atomicMax(&g_out[1], (long long)mx); }
}
int main() {
  const int64_t n = 8192LL * 8192, n4 = n / 4;
  int4* cols_h[6];
  for (int c = 0; c < 6; ++c) { cudaMalloc(&cols_h[c], n * 4); cudaMemset(cols_h[c], c, n * 4); }
  int4** cols_d; cudaMalloc(&cols_d, sizeof(cols_h)); cudaMemcpy(cols_d, cols_h, sizeof(cols_h), cudaMemcpyHostToDevice);
  void* flush; cudaMalloc(&flush, 512 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemset(flush, r, 512 << 20);
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("%-40s %.3f ms  %.0f GB/s  %s\n", name, best, 6.0 * n * 4 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  for (int tpb : {256, 512, 1024})
    for (int bps : {2, 4, 8, 16}) {
      int64_t gx = 148LL * bps * 256 / tpb; if (gx < 1) gx = 1;
      char nm[64];
      snprintf(nm, 64, "stride U4 tpb%d gx%lld", tpb, (long long)gx);
      run(nm, [&] { k_mm<4><<<dim3(gx, 6), tpb>>>(cols_d, n4); });
      snprintf(nm, 64, "stride U8 tpb%d gx%lld", tpb, (long long)gx);
      run(nm, [&] { k_mm<8><<<dim3(gx, 6), tpb>>>(cols_d, n4); });
      snprintf(nm, 64, "chunk U4 tpb%d gx%lld", tpb, (long long)gx);
      int64_t chunk = (n4 + gx - 1) / gx;
      run(nm, [&] { k_mm_chunk<4><<<dim3(gx, 6), tpb>>>(cols_d, n4, chunk); });
    }
  run("big grid U1 tpb256", [&] { k_mm<1><<<dim3((n4 + 255) / 256, 6), 256>>>(cols_d, n4); });
  run("grid 2368 U4 tpb256 (current)", [&] { k_mm<4><<<dim3(2368, 6), 256>>>(cols_d, n4); });
  return 0;
}
