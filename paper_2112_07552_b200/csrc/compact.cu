// compact.cu — step a8: nonzero compaction + decode of the result matrix.
//
// PAPER.md §3.2: nonzero(M) = {(i,j) | M_ij > 0} turns the result
// matrix back into a table on the GPU; §3.1 a pair is in the join
// iff C_ij > 0; Lemma Q3 (read as M_{1,j} per reading R4).
// Existence is decided on a COUNT plane (or on C itself when the guard proved
// that C != 0 <=> COUNT > 0; reading R3), so SUM = 0 groups are kept.
//
// Work unit: a segment = one row x 256 consecutive columns (the GEMM's N tile).
//   count:  per-segment nonzero counts — produced by the GEMM epilogue for free
//           on the dense path, or by k_seg_count (one warp per segment);
//   scan:   exclusive prefix over G x nseg counts (row-major);
//   write:  one warp per segment, 8 chunks of 32 columns; __ballot_sync +
//           popc gives each nonzero its slot, so reads of C and dict_h and the
//           writes of (g, h, agg) are all 32-wide contiguous (coalesced).
// Codes are ascending dense ranks, so row-major order is (g, h) order and the
// ORDER BY comes for free (§3.4). Decode: g = dict_g[i], h = dict_h[j].
#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

constexpr int T = 256;
constexpr int WPB = T / 32;

__device__ __forceinline__ bool nz_at(const void* base, int kind, int64_t idx) {
  switch (kind) {
    case 0: return static_cast<const int*>(base)[idx] != 0;
    case 1: return static_cast<const long long*>(base)[idx] != 0;
    case 2: return static_cast<const float*>(base)[idx] != 0.f;
    default: return static_cast<const double*>(base)[idx] != 0.0;
  }
}

__global__ void __launch_bounds__(T) k_seg_count(const CompactArgs a, int32_t* __restrict__ cnt) {
  const int64_t nsegs = a.G * a.nseg;
  const int lane = lane_id();
  for (int64_t s = (int64_t)blockIdx.x * WPB + warp_id(); s < nsegs; s += (int64_t)gridDim.x * WPB) {
    const int64_t row = s / a.nseg;
    const int64_t col0 = (s - row * a.nseg) * 256;
    int c = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t col = col0 + j * 32 + lane;
      c += (col < a.H && nz_at(a.E, a.e_kind, row * a.lde + col)) ? 1 : 0;
    }
    c = warp_sum(c);
    if (lane == 0) cnt[s] = c;
  }
}

__global__ void __launch_bounds__(T) k_seg_write(const CompactArgs a, const int64_t* __restrict__ off) {
  const int64_t nsegs = a.G * a.nseg;
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt();
  for (int64_t s = (int64_t)blockIdx.x * WPB + warp_id(); s < nsegs; s += (int64_t)gridDim.x * WPB) {
    const int64_t row = s / a.nseg;
    const int64_t col0 = (s - row * a.nseg) * 256;
    if (col0 >= a.H) continue;
    int64_t base = off[s];
    const long long gval = a.dict_g[row];
#pragma unroll 2
    for (int j = 0; j < 8; ++j) {
      const int64_t col = col0 + j * 32 + lane;
      const bool in = col < a.H;
      const bool e = in && nz_at(a.E, a.e_kind, row * a.lde + col);
      const uint32_t m = __ballot_sync(0xffffffffu, e);
      if (e) {
        const int64_t pos = base + __popc(m & lt);
        const long long hval = a.dict_h[col];
        if (a.g_out_type == 1) static_cast<long long*>(a.out_g)[pos] = gval;
        else static_cast<int*>(a.out_g)[pos] = (int)gval;
        if (a.h_out_type == 1) static_cast<long long*>(a.out_h)[pos] = hval;
        else static_cast<int*>(a.out_h)[pos] = (int)hval;
        const int64_t vi = row * a.ldv + col;
        if (a.agg_out == 0) {
          long long v;
          switch (a.v_kind) {
            case 0: v = static_cast<const int*>(a.V)[vi]; break;
            case 1: v = static_cast<const long long*>(a.V)[vi]; break;
            default: v = (long long)static_cast<const float*>(a.V)[vi];
          }
          static_cast<long long*>(a.out_agg)[pos] = v;
        } else {
          const double v = a.v_kind == 2 ? (double)static_cast<const float*>(a.V)[vi]
                                         : static_cast<const double*>(a.V)[vi];
          static_cast<double*>(a.out_agg)[pos] = v;
        }
      }
      base += __popc(m);
    }
  }
}

inline int grid_for_segs(int64_t nsegs) {
  int64_t g = (nsegs + WPB - 1) / WPB;
  if (g < 1) g = 1;
  if (g > kNumSMs * 32) g = kNumSMs * 32;
  return (int)g;
}

}  // namespace

size_t compact_temp_bytes(int64_t G, int64_t nseg) {
  const int64_t n = G * nseg;
  return ((size_t)n * 4 + 15) / 16 * 16 + (size_t)n * 8 + scan_temp_bytes(n) + 64;
}

// counts: if `precounted` != NULL the per-segment counts already exist (GEMM epilogue);
// otherwise they are computed into the temp buffer.
cudaError_t launch_compact_count(const CompactArgs& a, const int32_t* precounted, int64_t* nnz_dev, void* temp,
                                 cudaStream_t s, int64_t* launches) {
  const int64_t n = a.G * a.nseg;
  int32_t* cnt = static_cast<int32_t*>(temp);
  int64_t* off = reinterpret_cast<int64_t*>(static_cast<char*>(temp) + ((size_t)n * 4 + 15) / 16 * 16);
  if (n <= 0) return exclusive_scan_i32(nullptr, nullptr, 0, nnz_dev, off, s, launches);
  const int32_t* src = precounted;
  if (!src) {
    k_seg_count<<<grid_for_segs(n), T, 0, s>>>(a, cnt);
    if (launches) ++*launches;
    src = cnt;
  }
  return exclusive_scan_i32(src, off, n, nnz_dev, off + n, s, launches);
}

cudaError_t launch_compact_write(const CompactArgs& a, void* temp, cudaStream_t s, int64_t* launches) {
  const int64_t n = a.G * a.nseg;
  if (n <= 0) return cudaSuccess;
  const int64_t* off = reinterpret_cast<const int64_t*>(static_cast<char*>(temp) + ((size_t)n * 4 + 15) / 16 * 16);
  k_seg_write<<<grid_for_segs(n), T, 0, s>>>(a, off);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
