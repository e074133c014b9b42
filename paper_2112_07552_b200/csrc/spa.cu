// spa.cu — step a7 + a8 fused for the sparse path: row-wise expansion into
// shared-memory accumulators (a sparse accumulator, "SPA", per result row) and
// direct compaction from shared memory.
//
// PAPER.md §4.2.4 sends low-density joins to a sparse product; the
// result matrix is then turned back into a table by nonzero() (§3.2).
// Materializing C = G x H in HBM (zeroing it, scattering J atomics into it, and
// reading it twice for count + write) dominates that path when G x H is large
// (c3: 40k x 40k). Here no C exists:
//   A tuples are ordered by group code g (counting sort, sparse.cu), so the
//   updates of result rows [g0, g1) are one contiguous range of the update
//   sequence (update u of active tuple t hits bucket entry bstart[k_t] + u - off_t).
//   count pass: one CTA per band of rows; a presence bitmap per row in shared
//               memory (atomicOr), then popcounts -> row_nnz[g];
//   scan:       row_out = exclusive scan of row_nnz (the result allocation is
//               exact: n_result = total);
//   write pass: one CTA per (smaller) band; value cells + bitmap in shared
//               memory (shared-memory atomics), then each row is written in h
//               order straight to (g, h, agg) at row_out[g] — codes are ranks, so
//               the output is in (g, h) order like the dense path's.
// Both passes split each band's updates evenly over the CTA's warps; a warp maps 32
// consecutive updates to their tuples with one ballot + one OR-reduction (spa_expand).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

constexpr int NT = 1024;
constexpr size_t kSmemMax = 216 * 1024;  // dynamic; + ~8.5 KB static (write pass) <= 227 KB

__device__ __forceinline__ int64_t shfl64(int64_t v, int src) {
  return (int64_t)__shfl_sync(0xffffffffu, (long long)v, src);
}

// Largest t in [lo, hi) with off[t] <= u (off ascending, off[lo] <= u): 32-way search,
// one coalesced probe round per factor of 32.
__device__ __forceinline__ int64_t warp_find(const int64_t* __restrict__ off, int64_t lo, int64_t hi, int64_t u) {
  const int lane = lane_id();
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + lane * step;
    const unsigned m = __ballot_sync(0xffffffffu, p < hi && off[p] <= u);
    lo = lo + (int64_t)(31 - __clz(m)) * step;
    hi = min(hi, lo + step);
  }
  const unsigned m = __ballot_sync(0xffffffffu, lo + lane < hi && off[lo + lane] <= u);
  return lo + (31 - __clz(m));
}

// Calls f(row_in_band, h, bucket_pos, a_index) for every update of the CTA's band of
// rows [g0, g0 + rows) (active tuples are grouped by band: goff[band]).
// The band's update range is split evenly over the CTA's warps; each warp then works
// alone (no CTA barriers) on windows of 32 consecutive active tuples, one per lane, each
// clamped to the warp's update range:
//   long tuples (>= 32 updates in range): the warp walks the tuple's bucket together,
//     32 consecutive bucket entries per step (coalesced, no per-update mapping);
//   short tuples: their updates are numbered by a warp prefix sum, and update j + lane is
//     located by a 5-step search over the lanes' prefixes.
// (c3's 2-hop tuples average ~420 updates, so nearly all updates take the first form.)
template <bool NEED_A, class F>
__device__ __forceinline__ void spa_expand(const SpaArgs& a, int64_t t_begin, int64_t t_end, int64_t g0, F f) {
  const int lane = lane_id(), wid = warp_id(), nw = (int)(blockDim.x >> 5);
  if (t_begin >= t_end) return;
  const int64_t U0 = a.act_off[t_begin], U1 = a.act_off[t_end];
  const int64_t per = (U1 - U0 + nw - 1) / nw;
  int64_t u = U0 + (int64_t)wid * per;
  const int64_t uend = min(U1, u + per);
  if (u >= uend) return;
  int64_t t = warp_find(a.act_off, t_begin, t_end, u);
  while (u < uend) {
    const int64_t tl = t + lane;
    const bool valid = tl < t_end;
    const int64_t o = valid ? a.act_off[tl] : LLONG_MAX;
    const int64_t b = valid ? a.act_b[tl] : 0;
    const int gr = valid ? a.act_g[tl] - (int)g0 : 0;
    const int ai = (NEED_A && valid) ? a.act_a[tl] : 0;
    const int64_t wend = min(uend, t + 32 < t_end ? a.act_off[t + 32] : U1);
    // this lane's tuple, clamped to [u, wend)
    int64_t onext = shfl64(o, (lane + 1) & 31);
    if (lane == 31) onext = wend;
    const int64_t lo = max(o, u), hi = min(onext, wend);
    const int len = (valid && hi > lo) ? (int)(hi - lo) : 0;
    // long tuples: the whole warp walks one bucket range at a time
    unsigned lm = __ballot_sync(0xffffffffu, len >= 32);
    while (lm) {
      const int l = __ffs(lm) - 1;
      lm &= lm - 1;
      const int64_t xlo = shfl64(lo, l), xhi = shfl64(hi, l);
      const int64_t delta = shfl64(b, l) - shfl64(o, l);  // bucket pos = update index + delta
      const int r = __shfl_sync(0xffffffffu, gr, l);
      const int aval = NEED_A ? __shfl_sync(0xffffffffu, ai, l) : 0;
      for (int64_t x0 = xlo; x0 < xhi; x0 += 128) {
        int hh[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t x = x0 + 32 * j + lane;
          hh[j] = x < xhi ? __ldg(a.b_h + x + delta) : 0;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t x = x0 + 32 * j + lane;
          if (x < xhi) f(r, hh[j], x + delta, aval);
        }
      }
    }
    // short tuples: prefix-numbered updates, 32 per step
    const int slen = len < 32 ? len : 0;
    int incl = slen;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    const int sp = incl - slen;
    const int S = __shfl_sync(0xffffffffu, incl, 31);
    for (int j = 0; j < S; j += 32) {
      const int k = j + lane;
      int l = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int sps = __shfl_sync(0xffffffffu, sp, l + step);
        if (sps <= k) l += step;
      }
      const int64_t xl = shfl64(lo, l), dl = shfl64(b, l) - shfl64(o, l);
      const int spl = __shfl_sync(0xffffffffu, sp, l);
      const int r = __shfl_sync(0xffffffffu, gr, l);
      const int aval = NEED_A ? __shfl_sync(0xffffffffu, ai, l) : 0;
      if (k < S) {
        const int64_t pos = xl + (k - spl) + dl;
        f(r, __ldg(a.b_h + pos), pos, aval);
      }
    }
    u = wend;
    t += 32;
  }
}

constexpr int NTC = 512;  // count pass: 2 CTAs per SM
__global__ void __launch_bounds__(NTC, 2) k_spa_count(const SpaArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  // count_bands consecutive bands per CTA (their tuples are contiguous), or one listed band
  const int64_t b0 = a.band_list ? (int64_t)a.band_list[blockIdx.x] : (int64_t)blockIdx.x * a.count_bands;
  const int64_t b1 = a.band_list ? b0 + 1 : min(a.nbands, b0 + a.count_bands);
  const int64_t g0 = b0 * a.rows;
  const int64_t g1 = min(a.G, b1 * a.rows);
  const int nr = (int)(g1 - g0);
  const int64_t W = a.words;
  unsigned* bits = reinterpret_cast<unsigned*>(smem);
  for (int i = threadIdx.x; i < nr * (int)W; i += NTC) bits[i] = 0u;
  __syncthreads();
  spa_expand<false>(a, a.goff[b0], a.goff[b1], g0, [&](int r, int h, int64_t, int32_t) {
    atomicOr(bits + r * W + (h >> 5), 1u << (h & 31));
  });
  __syncthreads();
  for (int r = warp_id(); r < nr; r += NTC / 32) {
    int c = 0;
    for (int64_t w = lane_id(); w < W; w += 32) c += __popc(bits[r * W + w]);
    c = warp_sum(c);
    if (lane_id() == 0) a.row_nnz[g0 + r] = c;
  }
}

template <int ACC>
struct AccT;
template <> struct AccT<0> { using T = int; };
template <> struct AccT<1> { using T = unsigned long long; };
template <> struct AccT<2> { using T = unsigned long long; };
template <> struct AccT<3> { using T = double; };

template <int ACC>
__global__ void __launch_bounds__(NT) k_spa_write(const SpaArgs a) {
  using T = typename AccT<ACC>::T;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int64_t s_base[NT / 32 + 1];
  __shared__ uint8_t s_stage[NT / 32][256];
  const int64_t g0 = (int64_t)blockIdx.x * a.rows;
  const int64_t g1 = min(a.G, g0 + a.rows);
  const int nr = (int)(g1 - g0);
  const int64_t W = a.words, ldc = W * 32;
  T* acc = reinterpret_cast<T*>(smem);
  unsigned* bits = reinterpret_cast<unsigned*>(acc + (size_t)a.rows * ldc);
  {  // zero the cells with 16-byte stores (a row is a multiple of 128 bytes)
    const int nv = (int)((size_t)nr * ldc * sizeof(T) / 16);
    for (int i = threadIdx.x; i < nv; i += NT) reinterpret_cast<uint4*>(acc)[i] = make_uint4(0, 0, 0, 0);
  }
  for (int i = threadIdx.x; i < nr * (int)W; i += NT) bits[i] = 0u;
  __syncthreads();
  spa_expand<(ACC >= 2)>(a, a.goff[blockIdx.x], a.goff[blockIdx.x + 1], g0, [&](int r, int h, int64_t pos, int32_t ai) {
    const int64_t cell = r * ldc + h;
    if constexpr (ACC == 0) {
      atomicAdd(acc + cell, 1);
      atomicOr(bits + r * W + (h >> 5), 1u << (h & 31));
    } else if constexpr (ACC == 1) {
      atomicAdd(acc + cell, 1ull);
      atomicOr(bits + r * W + (h >> 5), 1u << (h & 31));
    } else if constexpr (ACC == 2) {
      const long long v = a.va.data ? ld_int(a.va.data, a.va.type, ai) : 1;
      const long long w = a.w_kind == 1 ? static_cast<const long long*>(a.b_w)[pos] : 1;
      atomicAdd(acc + cell, (unsigned long long)v * (unsigned long long)w);  // wrapping, exact mod 2^64
      atomicOr(bits + r * W + (h >> 5), 1u << (h & 31));
    } else {
      const double v = a.va.data ? (double)__ldg(static_cast<const float*>(a.va.data) + ai) : 1.0;
      const double w = a.w_kind == 2 ? (double)static_cast<const float*>(a.b_w)[pos] : 1.0;
      atomicAdd(acc + cell, v * w);
      atomicOr(bits + r * W + (h >> 5), 1u << (h & 31));
    }
  });
  __syncthreads();
  // each row: warps own contiguous slices of 8-word (256-cell) groups. Per group, lane l
  // takes byte l of the group's bitmap, the warp prefix-sums the byte popcounts, the set
  // cells go to a per-warp staging list (u8 offsets), and the list is written out with
  // all 32 lanes active (coalesced (g, h, agg) stores, one dict_h gather per output).
  const int nw = NT / 32, wid = warp_id(), lane = lane_id();
  uint8_t* stage = s_stage[wid];
  const int ngrp = (int)((W + 7) / 8);
  const int per = (ngrp + nw - 1) / nw;
  const int q0 = min(ngrp, wid * per), q1 = min(ngrp, q0 + per);
  for (int r = 0; r < nr; ++r) {
    const int64_t g = g0 + r;
    const unsigned* rb = bits + r * W;
    const uint8_t* rbytes = reinterpret_cast<const uint8_t*>(rb);
    const int nbytes = (int)W * 4;
    int c = 0;
    for (int i = q0 * 32 + lane; i < q1 * 32 && i < nbytes; i += 32) c += __popc(rbytes[i]);
    c = warp_sum(c);
    if (lane == 0) s_base[wid] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t run = a.row_out[g];
      for (int i = 0; i < nw; ++i) { const int64_t x = s_base[i]; s_base[i] = run; run += x; }
    }
    __syncthreads();
    int64_t base = s_base[wid];
    const long long gv = a.dict_g[g];
    const T* arow = acc + (int64_t)r * ldc;
    for (int q = q0; q < q1; ++q) {
      const int bi = q * 32 + lane;
      unsigned m = bi < nbytes ? rbytes[bi] : 0u;
      const int cnt = __popc(m);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      if (total == 0) continue;
      int p = incl - cnt;
      while (m) {
        const int b = __ffs(m) - 1;
        stage[p++] = (uint8_t)(lane * 8 + b);
        m &= m - 1;
      }
      __syncwarp();
      const int64_t hq = (int64_t)q * 256;
      for (int j = lane; j < total; j += 32) {
        const int64_t h = hq + stage[j];
        const int64_t o = base + j;
        const long long hv = __ldg(a.dict_h + h);
        if (a.g_out_type) __stcs(static_cast<long long*>(a.out_g) + o, gv);
        else __stcs(static_cast<int*>(a.out_g) + o, (int)gv);
        if (a.h_out_type) __stcs(static_cast<long long*>(a.out_h) + o, hv);
        else __stcs(static_cast<int*>(a.out_h) + o, (int)hv);
        const T x = arow[h];
        if constexpr (ACC == 3) __stcs(static_cast<double*>(a.out_agg) + o, x);
        else __stcs(static_cast<long long*>(a.out_agg) + o, (long long)x);
      }
      __syncwarp();
      base += total;
    }
    __syncthreads();  // s_base reuse
  }
}

// ---------------------------------------------------------------------------
// One-pass variant: expansion, counting and writing of a band in ONE kernel.
// Persistent CTAs (NTF threads, 2 per SM) take bands in ascending order from a
// ticket counter; after expanding band b a CTA publishes its tuple count and finds
// its output offset by a decoupled look-back over the bands before it (every band
// with a smaller ticket is held by a running CTA, so the wait always ends). The
// result buffer is sized by the upper bound min(G·H, J) tuples, so no count pass
// and no second expansion are needed. Cells are zeroed as they are read, so shared
// memory is cleared once per CTA, not once per band.
// COUNT uses packed u16 cells (half the shared memory of int32, so twice the rows
// per band or two CTAs per SM on wide rows); a count reaching 65,535 raises *ovf and
// the caller reruns the kernel with int32 cells.
constexpr int NTF = 512;
constexpr size_t kSmemFused = 96 * 1024;  // + ~17 KB static (stages): 2 CTAs per SM

template <int ACC> struct FusedCell;
template <> struct FusedCell<0> { using T = uint16_t; };            // COUNT, packed u16
template <> struct FusedCell<1> { using T = int; };                 // COUNT int32
template <> struct FusedCell<2> { using T = unsigned long long; };  // integer SUM (wrapping)
template <> struct FusedCell<3> { using T = double; };              // float SUM

constexpr unsigned long long kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbVal = (1ull << 62) - 1;

template <int ACC>
__global__ void __launch_bounds__(NTF, 2) k_spa_fused(const SpaArgs a) {
  using T = typename FusedCell<ACC>::T;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int64_t s_base[NTF / 32 + 1];
  __shared__ uint16_t s_stage16[NTF / 32][16 * 32];
  __shared__ int64_t s_rowbase[64];
  __shared__ int s_rowcnt[64];
  __shared__ int64_t s_band;
  const int nw = NTF / 32, wid = warp_id(), lane = lane_id();
  const int64_t W = a.words, ldc = W * 32;
  T* acc = reinterpret_cast<T*>(smem);
  unsigned* bits = reinterpret_cast<unsigned*>(smem + ((size_t)a.rows * ldc * sizeof(T) + 15) / 16 * 16);
  {
    const int nv = (int)(((size_t)a.rows * ldc * sizeof(T) + 15) / 16);
    for (int i = threadIdx.x; i < nv; i += NTF) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < a.rows * (int)W; i += NTF) bits[i] = 0u;
  }
  volatile unsigned long long* state = reinterpret_cast<volatile unsigned long long*>(a.lb_state);
  bool ovf = false;
  // the next band's ticket is drawn one band ahead (thread 0), so the atomic's latency
  // overlaps the current band's expansion instead of stalling the whole CTA
  unsigned long long next_ticket = 0;
  if (threadIdx.x == 0) next_ticket = atomicAdd(a.ticket, 1ull);
  for (;;) {
    __syncthreads();  // smem clear / previous band finished before the ticket is replaced
    if (threadIdx.x == 0) {
      s_band = (int64_t)next_ticket;
      if ((int64_t)next_ticket < a.nbands) next_ticket = atomicAdd(a.ticket, 1ull);
    }
    __syncthreads();
    const int64_t b = s_band;
    if (b >= a.nbands) break;
    const int64_t g0 = b * a.rows;
    const int nr = (int)min((int64_t)a.rows, a.G - g0);
    // write pass: this band's row offsets, loaded now and consumed after the expansion
    int64_t rowoff0 = 0;
    if (a.row_out && threadIdx.x < nr) rowoff0 = a.row_out[g0 + threadIdx.x];
    // a u16 cell can only reach 65,535 in a band with >= 65,535 updates: lighter bands use
    // fire-and-forget reductions (the returning atomic's latency was ~15 % of the band
    // kernel's warp samples on c3)
    const bool check16 = ACC == 0 && a.act_off[a.goff[b + 1]] - a.act_off[a.goff[b]] >= 65535;
    spa_expand<(ACC >= 2)>(a, a.goff[b], a.goff[b + 1], g0, [&](int r, int h, int64_t pos, int32_t ai) {
      if constexpr (ACC == 0) {
        const int sh = (h & 1) * 16;
        unsigned* cell = reinterpret_cast<unsigned*>(acc) + ((r * ldc + h) >> 1);
        if (check16) {
          const unsigned old = atomicAdd(cell, 1u << sh);
          if (((old >> sh) & 0xFFFFu) == 0xFFFFu) ovf = true;
        } else {
          atomicAdd(cell, 1u << sh);  // result unused: a shared-memory reduction
        }
      } else if constexpr (ACC == 1) {
        atomicAdd(acc + r * ldc + h, 1);
      } else if constexpr (ACC == 2) {
        const long long v = a.va.data ? ld_int(a.va.data, a.va.type, ai) : 1;
        const long long w = a.w_kind == 1 ? static_cast<const long long*>(a.b_w)[pos] : 1;
        atomicAdd(acc + r * ldc + h, (unsigned long long)v * (unsigned long long)w);
      } else {
        const double v = a.va.data ? (double)__ldg(static_cast<const float*>(a.va.data) + ai) : 1.0;
        const double w = a.w_kind == 2 ? (double)static_cast<const float*>(a.b_w)[pos] : 1.0;
        atomicAdd(acc + r * ldc + h, v * w);
      }
      atomicOr(bits + r * W + (h >> 5), 1u << (h & 31));
    });
    __syncthreads();
    // tuples per row of the band
    for (int r = wid; r < nr && !a.row_out; r += nw) {
      int c = 0;
      for (int64_t w = lane; w < W; w += 32) c += __popc(bits[r * W + w]);
      c = warp_sum(c);
      if (lane == 0) s_rowcnt[r] = c;
    }
    __syncthreads();
    if (a.row_out) {
      // write pass of the two-pass schedule: offsets from the count pass
      if (threadIdx.x < nr) s_rowbase[threadIdx.x] = rowoff0;
    } else if (threadIdx.x == 0) {
      int64_t cnt = 0;
      for (int r = 0; r < nr; ++r) cnt += s_rowcnt[r];
      // decoupled look-back: publish the aggregate, sum predecessors back to an inclusive prefix
      int64_t prefix = 0;
      if (b == 0) {
        atomicExch(reinterpret_cast<unsigned long long*>(a.lb_state), kLbInc | (unsigned long long)cnt);
      } else {
        atomicExch(reinterpret_cast<unsigned long long*>(a.lb_state) + b, kLbAgg | (unsigned long long)cnt);
        for (int64_t j = b - 1; j >= 0;) {
          const unsigned long long v = state[j];
          if ((v & ~kLbVal) == 0) continue;  // predecessor still expanding
          prefix += (int64_t)(v & kLbVal);
          if ((v & ~kLbVal) == kLbInc) break;
          --j;
        }
        atomicExch(reinterpret_cast<unsigned long long*>(a.lb_state) + b, kLbInc | (unsigned long long)(prefix + cnt));
      }
      if (b == a.nbands - 1) *a.total = prefix + cnt;
      int64_t run = prefix;
      for (int r = 0; r < nr; ++r) { s_rowbase[r] = run; run += s_rowcnt[r]; }
    }
    __syncthreads();
    // write: per row, warps own contiguous slices of 16-word (512-cell) chunks; lanes 0-15
    // hold one bitmap word each, a warp scan numbers the chunk's tuples, each lane lists its
    // set bits into the warp's 512-entry stage, and the stage is written out 32 tuples per
    // step (coalesced (g, h, agg) stores)
    constexpr int CW = 16;
    const int nch = (int)((W + CW - 1) / CW);
    const int per = (nch + nw - 1) / nw;
    const int q0 = min(nch, wid * per), q1 = min(nch, q0 + per);
    uint16_t* stage = s_stage16[wid];
    for (int r = 0; r < nr; ++r) {
      const int64_t g = g0 + r;
      unsigned* rb = bits + r * W;
      int c = 0;
      for (int64_t wq = (int64_t)q0 * CW + lane; wq < (int64_t)q1 * CW && wq < W; wq += 32) c += __popc(rb[wq]);
      c = warp_sum(c);
      if (lane == 0) s_base[wid] = c;
      __syncthreads();
      if (threadIdx.x == 0) {
        int64_t run = s_rowbase[r];
        for (int i = 0; i < nw; ++i) { const int64_t x = s_base[i]; s_base[i] = run; run += x; }
      }
      __syncthreads();
      int64_t base = s_base[wid];
      const long long gv = a.dict_g[g];
      T* arow = acc + (int64_t)r * ldc;
      for (int q = q0; q < q1; ++q) {
        // lane l takes half-word l & 1 of word l >> 1: all 32 lanes list set bits, at most 16 each
        const int64_t wi = (int64_t)q * CW + (lane >> 1);
        unsigned m = wi < W ? rb[wi] : 0u;
        m = (lane & 1) ? (m >> 16) : (m & 0xFFFFu);
        const int cnt = __popc(m);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) continue;
        int p = incl - cnt;
        while (m) {
          const int bb = __ffs(m) - 1;
          stage[p++] = (uint16_t)(lane * 16 + bb);
          m &= m - 1;
        }
        if (!(lane & 1) && wi < W) rb[wi] = 0u;  // this word is consumed (both halves were read above)
        __syncwarp();
        const int64_t hq = (int64_t)q * CW * 32;
        // two tuples per lane per step: both dictionary gathers are in flight before the
        // stores that consume them (the h store stalled on its gather)
        for (int j0 = lane; j0 < total; j0 += 64) {
          const int j1 = j0 + 32;
          const bool v1 = j1 < total;
          const int64_t h0 = hq + stage[j0];
          const int64_t h1 = v1 ? hq + stage[j1] : h0;
          const long long hv0 = __ldg(a.dict_h + h0);
          const long long hv1 = __ldg(a.dict_h + h1);
          const T x0 = arow[h0];
          const T x1 = arow[h1];
          arow[h0] = (T)0;  // zero on read: the next band starts from a clear accumulator
          if (v1) arow[h1] = (T)0;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && !v1) break;
            const int64_t o = base + (u ? j1 : j0);
            const long long hv = u ? hv1 : hv0;
            const T x = u ? x1 : x0;
            if (a.g_out_type) __stcs(static_cast<long long*>(a.out_g) + o, gv);
            else __stcs(static_cast<int*>(a.out_g) + o, (int)gv);
            if (a.h_out_type) __stcs(static_cast<long long*>(a.out_h) + o, hv);
            else __stcs(static_cast<int*>(a.out_h) + o, (int)hv);
            if constexpr (ACC == 3) __stcs(static_cast<double*>(a.out_agg) + o, x);
            else __stcs(static_cast<long long*>(a.out_agg) + o, (long long)x);
          }
        }
        __syncwarp();
        base += total;
      }
      __syncthreads();  // s_base reuse
    }
  }
  if (ovf) *a.ovf = 1;
}

}  // namespace

__global__ void k_band_weight_max(const int64_t* __restrict__ goff, const int64_t* __restrict__ act_off,
                                  int64_t nbands, unsigned long long* __restrict__ out) {
  unsigned long long m = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbands; b += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)(act_off[goff[b + 1]] - act_off[goff[b]]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0 && m) atomicMax(out, m);
}

__global__ void k_hub_list(const int64_t* __restrict__ goff, const int64_t* __restrict__ act_off, int64_t nbands,
                           unsigned long long thr, int32_t* __restrict__ list, unsigned long long* __restrict__ n) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbands; b += (int64_t)gridDim.x * blockDim.x)
    if ((unsigned long long)(act_off[goff[b + 1]] - act_off[goff[b]]) > thr)
      list[atomicAdd(n, 1ull)] = (int32_t)b;
}

__global__ void k_hub_publish(const int32_t* __restrict__ list, int64_t n_list, const int32_t* __restrict__ row_nnz,
                              int rows, int64_t G, unsigned long long* __restrict__ lb_state) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_list; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = list[i], g0 = b * rows, g1 = min(G, g0 + rows);
    unsigned long long c = 0;
    for (int64_t g = g0; g < g1; ++g) c += (unsigned long long)row_nnz[g];
    lb_state[b] = kLbAgg | c;  // the band's aggregate, before any CTA takes a ticket
  }
}

cudaError_t launch_hub_list(const SpaArgs& a, unsigned long long thr, int32_t* list, unsigned long long* n_out,
                            cudaStream_t s, int64_t* launches) {
  if (a.nbands <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>(2 * kNumSMs, (a.nbands + 255) / 256);
  k_hub_list<<<(unsigned)blocks, 256, 0, s>>>(a.goff, a.act_off, a.nbands, thr, list, n_out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_hub_publish(const SpaArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.n_list <= 0) return cudaSuccess;
  k_hub_publish<<<(unsigned)std::min<int64_t>(kNumSMs, (a.n_list + 255) / 256), 256, 0, s>>>(
      a.band_list, a.n_list, a.row_nnz, a.rows, a.G, a.lb_state);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_band_weight_max(const SpaArgs& a, unsigned long long* out, cudaStream_t s, int64_t* launches) {
  if (a.nbands <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>(2 * kNumSMs, (a.nbands + 255) / 256);
  k_band_weight_max<<<(unsigned)blocks, 256, 0, s>>>(a.goff, a.act_off, a.nbands, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// Fused one-pass plan: rows per band so that 2 CTAs fit per SM and there are >= ~4
// bands per CTA for the ticket scheduler to balance. false: a row does not fit.
bool spa_fused_plan(SpaArgs& a) {
  a.words = (a.H + 31) / 32;
  const size_t cell = a.acc_kind == 4 ? 2 : (a.acc_kind == 0 ? 4 : 8);
  const size_t row_w = (size_t)a.words * 32 * cell + (size_t)a.words * 4;
  const int fit = (int)std::min<size_t>(64, (kSmemFused - 16) / row_w);
  if (fit < 1) return false;
  const int64_t grid = 2 * kNumSMs;
  const int64_t want = std::max<int64_t>(1, a.G / (4 * grid));
  a.rows = (int)std::min<int64_t>(want, fit);
  a.nbands = (a.G + a.rows - 1) / a.rows;
  return true;
}

static size_t fused_smem(const SpaArgs& a) {
  const size_t cell = a.acc_kind == 4 ? 2 : (a.acc_kind == 0 ? 4 : 8);
  return ((size_t)a.rows * a.words * 32 * cell + 15) / 16 * 16 + (size_t)a.rows * a.words * 4;
}

template <int ACC>
static cudaError_t launch_fused_t(const SpaArgs& a, cudaStream_t s) {
  const cudaError_t e = set_func_attr(k_spa_fused<ACC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kSmemFused);
  if (e != cudaSuccess) return e;
  const int64_t grid = std::min<int64_t>(a.nbands, 2 * kNumSMs);
  k_spa_fused<ACC><<<(unsigned)grid, NTF, fused_smem(a), s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_spa_fused(const SpaArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.G <= 0) return cudaSuccess;
  cudaError_t e;
  switch (a.acc_kind) {
    case 4: e = launch_fused_t<0>(a, s); break;
    case 0: e = launch_fused_t<1>(a, s); break;
    case 2: e = launch_fused_t<2>(a, s); break;
    case 3: e = launch_fused_t<3>(a, s); break;
    default: return cudaErrorInvalidValue;  // int64 COUNT cells: two-pass path
  }
  if (launches) ++*launches;
  return e;
}

bool spa_plan(SpaArgs& a) {
  a.words = (a.H + 31) / 32;
  const size_t row_bits = (size_t)a.words * 4;
  const size_t cell = a.acc_kind == 0 ? 4 : 8;
  const size_t row_w = (size_t)a.words * 32 * cell + row_bits;
  if (row_w + 1024 > kSmemMax) return false;
  // one band of rows per CTA in both passes: ~2 waves of 1-CTA-per-SM bands
  const int64_t want = std::max<int64_t>(1, (a.G + 2 * kNumSMs - 1) / (2 * kNumSMs));
  a.rows = (int)std::min<int64_t>(want, (int64_t)((kSmemMax - 1024) / row_w));
  if (a.rows < 1) return false;
  a.nbands = (a.G + a.rows - 1) / a.rows;
  // count pass: bitmaps only, so several bands per CTA (<= 48 KB, >= ~4 CTAs per SM of work)
  const int64_t by_smem = std::max<int64_t>(1, (int64_t)(48 * 1024 / (row_bits * a.rows)));
  const int64_t by_grid = std::max<int64_t>(1, a.nbands / (4 * kNumSMs));
  a.count_bands = (int)std::min(by_smem, by_grid);
  return true;
}

void spa_count_plan(SpaArgs& a) {
  const size_t row_bits = (size_t)a.words * 4;
  const int64_t by_smem = std::max<int64_t>(1, (int64_t)(48 * 1024 / (row_bits * a.rows)));
  const int64_t by_grid = std::max<int64_t>(1, a.nbands / (4 * kNumSMs));
  a.count_bands = (int)std::min(by_smem, by_grid);
}

static size_t count_smem(const SpaArgs& a) { return (size_t)a.count_bands * a.rows * a.words * 4; }
static size_t write_smem(const SpaArgs& a) {
  const size_t cell = a.acc_kind == 0 ? 4 : 8;
  return (size_t)a.rows * a.words * 32 * cell + (size_t)a.rows * a.words * 4;
}

cudaError_t launch_spa_count(const SpaArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.G <= 0) return cudaSuccess;
  const size_t sm = count_smem(a);
  const cudaError_t e = set_func_attr(k_spa_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
  if (e != cudaSuccess) return e;
  const int64_t grid = a.band_list ? a.n_list : (a.nbands + a.count_bands - 1) / a.count_bands;
  if (grid <= 0) return cudaSuccess;
  k_spa_count<<<(unsigned)grid, NTC, sm, s>>>(a);
  if (launches) ++*launches;
  return cudaGetLastError();
}

template <int ACC>
static cudaError_t launch_write_t(const SpaArgs& a, cudaStream_t s) {
  const cudaError_t e = set_func_attr(k_spa_write<ACC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kSmemMax);
  if (e != cudaSuccess) return e;
  k_spa_write<ACC><<<(unsigned)((a.G + a.rows - 1) / a.rows), NT, write_smem(a), s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_spa_write(const SpaArgs& a, cudaStream_t s, int64_t* launches) {
  if (a.G <= 0) return cudaSuccess;
  cudaError_t e;
  switch (a.acc_kind) {
    case 0: e = launch_write_t<0>(a, s); break;
    case 1: e = launch_write_t<1>(a, s); break;
    case 2: e = launch_write_t<2>(a, s); break;
    default: e = launch_write_t<3>(a, s);
  }
  if (launches) ++*launches;
  return e;
}

}  // namespace tcudb
