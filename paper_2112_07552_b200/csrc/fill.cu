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

// fp32 scratch -> bf16 hi (and optionally lo) segments; 8 cells per thread step.
__global__ void k_pack_bf16(const float* __restrict__ scr, int64_t rows, int64_t ld, uint16_t* __restrict__ op,
                            int64_t ld_op, int seg_hi, int seg_lo, FillStats* __restrict__ fs) {
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
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint16_t h0 = bf16_bits(x[2 * j]), h1 = bf16_bits(x[2 * j + 1]);
      const float r0 = x[2 * j] - bf16_val(h0), r1 = x[2 * j + 1] - bf16_val(h1);
      inexact |= (r0 != 0.f) | (r1 != 0.f);
      nnz += (x[2 * j] != 0.f) + (x[2 * j + 1] != 0.f);
      hi[j] = (uint32_t)h0 | ((uint32_t)h1 << 16);
      lo[j] = (uint32_t)bf16_bits(r0) | ((uint32_t)bf16_bits(r1) << 16);
    }
    uint16_t* row = op + r * ld_op;
    *reinterpret_cast<uint4*>(row + (int64_t)seg_hi * ld + c8) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    if (seg_lo >= 0) *reinterpret_cast<uint4*>(row + (int64_t)seg_lo * ld + c8) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
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

cudaError_t launch_fill_bf16_direct(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                                    uint16_t* op, int64_t ld_op, unsigned* occ, int64_t ld_occ, FillStats* fs,
                                    cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_fill_bf16_direct<<<grid_for(n), T, 0, s>>>(kcode, rcode, static_cast<const float*>(val.data), n, op, ld_op,
                                               occ, ld_occ, fs);
  if (launches) ++*launches;
  return cudaGetLastError();
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

cudaError_t launch_pack_bf16(const float* scr, int64_t rows, int64_t ld, uint16_t* op, int64_t ld_op, int seg_hi,
                             int seg_lo, FillStats* fs, cudaStream_t s, int64_t* launches) {
  if (rows <= 0) return cudaSuccess;
  k_pack_bf16<<<grid_for(rows * (ld / 8), T * 4), T, 0, s>>>(scr, rows, ld, op, ld_op, seg_hi, seg_lo, fs);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
