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
#include <algorithm>
#include <cstdint>
#include <cstdlib>

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
    case 4: return static_cast<const unsigned short*>(base)[idx] != 0;
    default: return static_cast<const double*>(base)[idx] != 0.0;
  }
}

__global__ void __launch_bounds__(T) k_seg_count(const CompactArgs a, int32_t* __restrict__ cnt) {
  const int64_t nsegs = a.G * a.nseg;
  const int lane = lane_id();
  for (int64_t s = (int64_t)blockIdx.x * WPB + warp_id(); s < nsegs; s += (int64_t)gridDim.x * WPB) {
    const int64_t row = s / a.nseg;
    const int64_t col0 = (s - row * a.nseg) * a.seg_w;
    const int64_t lim = min(a.H, col0 + a.seg_w);
    int c = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t col = col0 + j * 32 + lane;
      c += (col < lim && nz_at(a.E, a.e_kind, row * a.lde + col)) ? 1 : 0;
    }
    c = warp_sum(c);
    if (lane == 0) cnt[s] = c;
  }
}

template <int K>
struct Cell;
template <> struct Cell<0> { using T = int;       static __device__ bool nz(T x) { return x != 0; } };
template <> struct Cell<1> { using T = long long; static __device__ bool nz(T x) { return x != 0; } };
template <> struct Cell<2> { using T = float;     static __device__ bool nz(T x) { return x != 0.f; } };
template <> struct Cell<3> { using T = double;    static __device__ bool nz(T x) { return x != 0.0; } };
template <> struct Cell<4> { using T = unsigned short; static __device__ bool nz(T x) { return x != 0; } };

// One warp per 256-column segment: all 8 chunk loads are issued before the
// ballots (8 loads in flight per lane); when V is E the value comes from the
// same load. Output slots: base + popc(ballot & lanemask_lt) -> contiguous stores.
template <int EK, int VK, bool SAME, int GT, int HT>
__global__ void __launch_bounds__(T) k_seg_write(const CompactArgs a, const int64_t* __restrict__ off) {
  using ET = typename Cell<EK>::T;
  using VT = typename Cell<VK>::T;
  const int64_t nsegs = a.G * a.nseg;
  const int lane = lane_id();
  const uint32_t lt = lanemask_lt();
  const ET* __restrict__ E = static_cast<const ET*>(a.E);
  const VT* __restrict__ V = static_cast<const VT*>(a.V);
  // Two segments per warp iteration: all 16 cell loads and 16 dict_h loads are in
  // flight before the first ballot (the kernel is load-latency bound otherwise).
  constexpr int P = 2;
  const int64_t stride = (int64_t)gridDim.x * WPB;
  for (int64_t s0 = (int64_t)blockIdx.x * WPB + warp_id(); s0 < nsegs; s0 += P * stride) {
    ET e[P][8];
    VT v[P][8];
    long long hv[P][8];
    int64_t row[P], col0[P], lim[P];
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const int64_t s = s0 + q * stride;
      row[q] = s < nsegs ? s / a.nseg : 0;
      col0[q] = (s - row[q] * a.nseg) * a.seg_w;
      // a segment without nonzeros (off[s + 1] == off[s]) is not read at all: block-sparse
      // products leave whole tiles zero
      lim[q] = (s < nsegs && off[s + 1] > off[s]) ? min(a.H, col0[q] + a.seg_w) : 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t col = col0[q] + j * 32 + lane;
        const bool in = col < lim[q];
        e[q][j] = in ? __ldcs(E + row[q] * a.lde + col) : ET(0);
        hv[q][j] = !in ? 0 : a.h_affine ? a.h_base + col : __ldg(a.dict_h + col);
      }
    }
#pragma unroll
    for (int q = 0; q < P; ++q) {
      const int64_t s = s0 + q * stride;
      if (s >= nsegs || col0[q] >= a.H || lim[q] == 0) continue;
    if (!SAME) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t col = col0[q] + j * 32 + lane;
        v[q][j] = (col < lim[q] && Cell<EK>::nz(e[q][j])) ? __ldcs(V + row[q] * a.ldv + col) : VT(0);
      }
    }
    int64_t base = off[s];
    const long long gval = GT < 2 ? a.dict_g[row[q]] : 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const bool nz = Cell<EK>::nz(e[q][j]);
      const uint32_t m = __ballot_sync(0xffffffffu, nz);
      if (nz) {
        const int64_t pos = base + __popc(m & lt);
        const long long hval = hv[q][j];
        // streaming (evict-first) stores: the result tuples are not re-read by the GPU
        // (GT 2 / 3: the g column is written by k_fill_g, one vectorised run per row)
        if (GT == 1) __stcs(static_cast<long long*>(a.out_g) + pos, gval);
        else if (GT == 0) __stcs(static_cast<int*>(a.out_g) + pos, (int)gval);
        if (HT == 1) __stcs(static_cast<long long*>(a.out_h) + pos, hval);
        else __stcs(static_cast<int*>(a.out_h) + pos, (int)hval);
        const VT x = SAME ? (VT)e[q][j] : v[q][j];
        if (VK == 2 || VK == 3) __stcs(static_cast<double*>(a.out_agg) + pos, (double)x);
        else __stcs(static_cast<long long*>(a.out_agg) + pos, (long long)x);
      }
      base += __popc(m);
    }
    }
  }
}

// The g column of the result is constant along each row: row r's tuples occupy
// [off[r * nseg], off[(r + 1) * nseg]) and all carry dict_g[r]. One warp per row writes that
// run with aligned 16-byte stores (scalar head / tail), so the ordered write pass above stores
// only h and agg.
template <typename GV>
__global__ void __launch_bounds__(T) k_fill_g(const CompactArgs a, const int64_t* __restrict__ off) {
  constexpr int PER16 = 16 / sizeof(GV);
  const int lane = lane_id();
  GV* out = static_cast<GV*>(a.out_g);
  for (int64_t r = (int64_t)blockIdx.x * WPB + warp_id(); r < a.G; r += (int64_t)gridDim.x * WPB) {
    const int64_t b = off[r * a.nseg], e = off[(r + 1) * a.nseg];
    if (b >= e) continue;
    const GV g = (GV)a.dict_g[r];
    // head up to 16-byte alignment, aligned body, tail
    const int64_t mis = (int64_t)((reinterpret_cast<uintptr_t>(out + b) & 15) / sizeof(GV));
    const int64_t b16 = min(e, b + (mis ? PER16 - mis : 0));
    if (b + lane < b16) __stcs(out + b + lane, g);
    const int64_t nv = (e - b16) / PER16;
    uint4 w;
    if (sizeof(GV) == 4) w = make_uint4((unsigned)g, (unsigned)g, (unsigned)g, (unsigned)g);
    else w = make_uint4((unsigned)(long long)g, (unsigned)((unsigned long long)(long long)g >> 32),
                        (unsigned)(long long)g, (unsigned)((unsigned long long)(long long)g >> 32));
    uint4* o4 = reinterpret_cast<uint4*>(out + b16);
    for (int64_t i = lane; i < nv; i += 32) __stcs(o4 + i, w);
    for (int64_t i = b16 + nv * PER16 + lane; i < e; i += 32) __stcs(out + i, g);
  }
}

template <int EK, int VK, bool SAME>
int launch_write_t(const CompactArgs& a, const int64_t* off, int grid, cudaStream_t s) {
  // g in its own pass for the dense e2m1 COUNT results (u16 cells, long rows): aligned vector
  // runs instead of a 4 / 8-byte store per tuple (c2: compaction 0.378 -> 0.370 ms; on c4 / c5
  // measured within noise, so only here — scripts/gpu_fillg.sh)
  static const bool no_fg = getenv("TCUDB_NO_FILL_G") && getenv("TCUDB_NO_FILL_G")[0] == '1';
  const bool fill_g = !no_fg && EK == 4 && a.nseg >= 8;
  const int sel = (fill_g ? 4 : 0) + a.g_out_type * 2 + a.h_out_type;
  switch (sel) {
    case 0: k_seg_write<EK, VK, SAME, 0, 0><<<grid, T, 0, s>>>(a, off); break;
    case 1: k_seg_write<EK, VK, SAME, 0, 1><<<grid, T, 0, s>>>(a, off); break;
    case 2: k_seg_write<EK, VK, SAME, 1, 0><<<grid, T, 0, s>>>(a, off); break;
    case 3: k_seg_write<EK, VK, SAME, 1, 1><<<grid, T, 0, s>>>(a, off); break;
    case 4: k_seg_write<EK, VK, SAME, 2, 0><<<grid, T, 0, s>>>(a, off); break;
    case 5: k_seg_write<EK, VK, SAME, 2, 1><<<grid, T, 0, s>>>(a, off); break;
    case 6: k_seg_write<EK, VK, SAME, 3, 0><<<grid, T, 0, s>>>(a, off); break;
    default: k_seg_write<EK, VK, SAME, 3, 1><<<grid, T, 0, s>>>(a, off); break;
  }
  if (fill_g) {
    const int gg = (int)std::min<int64_t>((a.G + WPB - 1) / WPB, (int64_t)kNumSMs * 8);
    if (a.g_out_type) k_fill_g<long long><<<std::max(gg, 1), T, 0, s>>>(a, off);
    else k_fill_g<int><<<std::max(gg, 1), T, 0, s>>>(a, off);
  }
  return fill_g ? 2 : 1;  // kernels launched
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
  return ((size_t)n * 4 + 15) / 16 * 16 + (size_t)(n + 1) * 8 + scan_temp_bytes(n) + 64;
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
  // off[n] = the total as well (the write pass reads off[s + 1] - off[s] per segment)
  const cudaError_t e = exclusive_scan_i32(src, off, n, nnz_dev, off + n + 1, s, launches);
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(off + n, nnz_dev, 8, cudaMemcpyDeviceToDevice, s);
}

cudaError_t launch_compact_write(const CompactArgs& a, void* temp, cudaStream_t s, int64_t* launches) {
  const int64_t n = a.G * a.nseg;
  if (n <= 0) return cudaSuccess;
  const int64_t* off = reinterpret_cast<const int64_t*>(static_cast<char*>(temp) + ((size_t)n * 4 + 15) / 16 * 16);
  const int grid = grid_for_segs(n);
  const bool same = a.E == a.V && a.e_kind == a.v_kind && a.lde == a.ldv;
  int nk = 1;
  if (same) {
    switch (a.e_kind) {
      case 0: nk = launch_write_t<0, 0, true>(a, off, grid, s); break;
      case 1: nk = launch_write_t<1, 1, true>(a, off, grid, s); break;
      case 2: nk = launch_write_t<2, 2, true>(a, off, grid, s); break;
      case 4: nk = launch_write_t<4, 4, true>(a, off, grid, s); break;
      default: nk = launch_write_t<3, 3, true>(a, off, grid, s);
    }
  } else {
    // separate existence planes: int32 counts (u8 pattern GEMM) or u16 (e2m1 pattern GEMM)
    if (a.e_kind == 0) {
      switch (a.v_kind) {
        case 0: nk = launch_write_t<0, 0, false>(a, off, grid, s); break;
        case 1: nk = launch_write_t<0, 1, false>(a, off, grid, s); break;
        case 2: nk = launch_write_t<0, 2, false>(a, off, grid, s); break;
        default: nk = launch_write_t<0, 3, false>(a, off, grid, s);
      }
    } else if (a.e_kind == 4) {
      switch (a.v_kind) {
        case 0: nk = launch_write_t<4, 0, false>(a, off, grid, s); break;
        case 1: nk = launch_write_t<4, 1, false>(a, off, grid, s); break;
        case 2: nk = launch_write_t<4, 2, false>(a, off, grid, s); break;
        default: nk = launch_write_t<4, 3, false>(a, off, grid, s);
      }
    } else {
      return cudaErrorInvalidValue;
    }
  }
  if (launches) *launches += nk;
  return cudaGetLastError();
}

}  // namespace tcudb
