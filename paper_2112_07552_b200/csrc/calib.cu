// calib.cu — device-side helpers of the one-time selector calibration at tcudb_create
// (SURVEY §8(b) "runs calibration (A19)"; §4.2.2 P:1186-1195 and the sampling
// of P:1511-1527: the cost model's constants are measured on the device, not assumed).
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// k[i] uniform over [0, keys), g[i] uniform over [0, groups) (counter-based, seeded)
__global__ void k_gen_cols(int32_t* __restrict__ k, int32_t* __restrict__ g, int64_t n, uint32_t keys,
                           uint32_t groups, uint32_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t a = mix32((uint32_t)i * 2u + seed), b = mix32((uint32_t)i * 2u + 1u + seed * 0x9E3779B9u);
    k[i] = (int32_t)(((uint64_t)a * keys) >> 32);
    g[i] = (int32_t)(((uint64_t)b * groups) >> 32);
  }
}

}  // namespace

cudaError_t launch_gen_cols(int32_t* k, int32_t* g, int64_t n, uint32_t keys, uint32_t groups, uint32_t seed,
                            cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_gen_cols<<<kNumSMs * 4, 256, 0, s>>>(k, g, n, keys, groups, seed);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
