// encode.cu — steps a1/a2: column statistics and key-domain encoding.
//
// PAPER.md §3.1: dom(ID) = dom(A.ID) ∪ dom(B.ID) = {v_1..v_k},
// v_j ↦ column j; §4.2.1 per-column metadata (min, max,
// #distinct). Readings: codes are dense ranks (R2); the join-key
// domain keeps only keys present on BOTH sides (∩ ⊆ ∪ gives the same result —
// a key on one side only yields a zero column; R1).
//
// Two dictionary mechanisms, chosen per domain from the min/max statistics:
//   direct-offset (span <= 4n): presence flags over [min, max], codes = exclusive
//     scan of the flags (ascending by construction);
//   hash (otherwise): open-addressing table of 2^ceil(log2 2n) slots keyed by
//     (x - min); an insert reads the slot first (a present key costs no atomic)
//     and CASes only an empty slot; side flags, compaction by scan,
//     and — for the group domains — an LSD radix sort of the distinct values so
//     codes are ascending ranks (result order = (g,h) order).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "dict.cuh"

namespace tcudb {
namespace {

constexpr int T = 256;

// ------------------------------------------------------------------ a1: statistics
// Block-level reduction, then ONE set of atomics per block: same-address global
// atomics serialize in L2 (~1 ns each), so per-warp atomics from thousands of warps
// cost more than the column scan itself.
__device__ __forceinline__ void col_stats_finish(ColStats* s, long long mn, long long mx, long long mabs, int flags) {
  __shared__ long long smn[T / 32], smx[T / 32], sab[T / 32];
  __shared__ int sfl[T / 32];
  mn = warp_min_ll(mn); mx = warp_max_ll(mx); mabs = warp_min_ll(mabs);
  flags = (int)__reduce_or_sync(0xffffffffu, (unsigned)flags);  // every flag bit, not just "any"
  if (lane_id() == 0) { smn[warp_id()] = mn; smx[warp_id()] = mx; sab[warp_id()] = mabs; sfl[warp_id()] = flags; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < T / 32; ++w) {
      mn = min(mn, smn[w]); mx = max(mx, smx[w]); mabs = min(mabs, sab[w]); flags |= sfl[w];
    }
    atomicMin(&s->mn, mn);
    atomicMax(&s->mx, mx);
    atomicMin(&s->min_abs, mabs);
    if (flags) atomicOr(&s->flags, flags);
  }
}

// HyperLogLog register update (see k_hll): the same hash for int32 and int64 values
TCUDB_DEV void hll_add(unsigned* s_reg, long long x) {
  const unsigned long long h = fmix64((unsigned long long)x * 0x9E3779B97F4A7C15ull + 1);
  const unsigned idx = (unsigned)(h >> (64 - kHllP));
  const unsigned long long w = h << kHllP;
  const unsigned rho = w ? (unsigned)__clzll(w) + 1u : (unsigned)(64 - kHllP + 1);
  if (rho > s_reg[idx]) atomicMax(&s_reg[idx], rho);  // most updates stop at the read
}

// 32-bit variant for the sketches of int32 GROUP columns (each has its own sketch; the key
// columns share the union sketch and keep the 64-bit hash so int32 and int64 keys agree)
TCUDB_DEV void hll_add32(unsigned* s_reg, int x) {
  const unsigned h = fmix32((unsigned)x * 0x9E3779B1u + 1u);
  const unsigned idx = h >> (32 - kHllP);
  const unsigned w = h << kHllP;
  const unsigned rho = w ? (unsigned)__clz(w) + 1u : (unsigned)(32 - kHllP + 1);
  if (rho > s_reg[idx]) atomicMax(&s_reg[idx], rho);
}

// Sketch gate: 4,096 evenly spaced samples per int column (columns 0..3); a column is
// sketched in the statistics pass iff its sampled span already exceeds the direct-offset
// limit (max(4n, 65536): it will be a hash-mode domain). gate[c] = 1 / 0 (read back with
// the statistics; a hash domain whose samples missed its span falls back to k_hll).
__global__ void k_sketch_gate(ColDesc c0, ColDesc c1, ColDesc c2, ColDesc c3, int* __restrict__ gate) {
  const ColDesc c = blockIdx.x == 0 ? c0 : blockIdx.x == 1 ? c1 : blockIdx.x == 2 ? c2 : c3;
  __shared__ long long smn[32], smx[32];
  long long mn = LLONG_MAX, mx = LLONG_MIN;
  if (c.data && c.n > 0) {
    // n * i < 2^63 for n < 2^51: 64-bit index math (a 128-bit division per sample cost ~15 us)
    long long x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = threadIdx.x + u * (int)blockDim.x;
      x[u] = i < 4096 ? ld_int(c.data, c.type, (int64_t)(c.n < (1ll << 51) ? c.n * i / 4096
                                                                         : (int64_t)((__int128)c.n * i / 4096)))
                      : x[0];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) { mn = min(mn, x[u]); mx = max(mx, x[u]); }
  }
  mn = warp_min_ll(mn); mx = warp_max_ll(mx);
  if (lane_id() == 0) { smn[warp_id()] = mn; smx[warp_id()] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x / 32); ++w) { mn = min(mn, smn[w]); mx = max(mx, smx[w]); }
    // the key domain spans both key columns: n of the pair
    const int64_t n = blockIdx.x <= 1 ? c0.n + c1.n : c.n;
    const unsigned long long span = (unsigned long long)mx - (unsigned long long)mn;
    gate[blockIdx.x] = (mx >= mn && span + 1 > (unsigned long long)max((int64_t)4 * n, (int64_t)65536)) ? 1 : 0;
  }
}

// blockIdx.y = column id. Integer columns: min / max (int64). Float columns:
// min / max / min |x| (ordered-int encodings of fp32). HLL: the #distinct sketches of the
// key columns (0, 1 -> one union sketch), A.g (2) and B.h (3) are updated in the same pass
// (sketch regs[3][kHllM], zeroed by the caller) — the #distinct metadata of P:1005-1008.
template <bool HLL>
__global__ void k_col_stats(ColDesc c0, ColDesc c1, ColDesc c2, ColDesc c3, ColDesc c4, ColDesc c5,
                            ColStats* __restrict__ st, unsigned* __restrict__ hll, const int* __restrict__ gate) {
  __shared__ unsigned s_reg[HLL ? kHllM : 1];
  ColDesc c = blockIdx.y == 0 ? c0 : blockIdx.y == 1 ? c1 : blockIdx.y == 2 ? c2 : blockIdx.y == 3 ? c3
             : blockIdx.y == 4 ? c4 : c5;
  if (!c.data || c.n <= 0) return;
  // key columns 0/1 share the union sketch: sketched if either sample says hash mode
  const bool sk = HLL && blockIdx.y < 4 &&
                  (blockIdx.y <= 1 ? (gate[0] | gate[1]) != 0 : gate[blockIdx.y] != 0);
  if (sk) {
    for (int i = threadIdx.x; i < kHllM; i += T) s_reg[i] = 0;
    __syncthreads();
  }
  unsigned* gsk = sk ? hll + (blockIdx.y <= 1 ? 0 : (blockIdx.y - 1)) * kHllM : nullptr;
  auto flush = [&]() {
    if (!sk) return;
    __syncthreads();
    for (int i = threadIdx.x; i < kHllM; i += T)
      if (s_reg[i]) atomicMax(gsk + i, s_reg[i]);
  };
  ColStats* s = st + blockIdx.y;
  const int64_t stride = (int64_t)gridDim.x * T;
  const int64_t gtid = (int64_t)blockIdx.x * T + threadIdx.x;
  // 16-byte vector loads, two in flight per thread; the scalar tail (< 4 items) after
  const int64_t n4 = (reinterpret_cast<uintptr_t>(c.data) & 15) ? 0 : c.n / 4;
  if (c.type == 2) {  // fp32
    float mn = INFINITY, mx = -INFINITY, mabs = INFINITY;
    int nonfinite = 0;
    const float* p = static_cast<const float*>(c.data);
    const float4* p4 = static_cast<const float4*>(c.data);
    int inexact = 0;  // some value is not bf16-representable (flags bit 1)
    auto take = [&](float x) {
      if (!isfinite(x)) nonfinite = 1;
      inexact |= (__float_as_uint(x) & 0xFFFFu) != 0u;
      mn = fminf(mn, x); mx = fmaxf(mx, x); mabs = fminf(mabs, fabsf(x));
    };
    for (int64_t i0 = gtid; i0 < n4; i0 += 4 * stride) {
      float4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // clamped index: a repeat is harmless for min/max
        const int4 t = ld_stream_v4(p4 + min(i0 + u * stride, n4 - 1));
        x[u] = make_float4(__int_as_float(t.x), __int_as_float(t.y), __int_as_float(t.z), __int_as_float(t.w));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) { take(x[u].x); take(x[u].y); take(x[u].z); take(x[u].w); }
    }
    for (int64_t i = n4 * 4 + gtid; i < c.n; i += stride) take(__ldcs(p + i));
    // fp32 -> order-preserving int: flip for negatives
    auto ord = [](float f) { int b = __float_as_int(f); return b >= 0 ? (long long)b : (long long)(b ^ 0x7fffffff); };
    col_stats_finish(s, ord(mn), ord(mx), ord(mabs), nonfinite | (inexact << 1));
    return;
  }
  if (c.type == 0) {  // int32: 32-bit compares, widened once at the end
    int mn = INT_MAX, mx = INT_MIN;
    unsigned mabs = UINT_MAX;
    const int* p = static_cast<const int*>(c.data);
    const int4* p4 = static_cast<const int4*>(c.data);
    const bool key_col = blockIdx.y <= 1;
    auto take = [&](int x) {
      mn = min(mn, x); mx = max(mx, x);
      mabs = min(mabs, x < 0 ? 0u - (unsigned)x : (unsigned)x);
      if (sk) {
        if (key_col) hll_add(s_reg, (long long)x);
        else hll_add32(s_reg, x);
      }
    };
    for (int64_t i0 = gtid; i0 < n4; i0 += 4 * stride) {
      int4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = ld_stream_v4(p4 + min(i0 + u * stride, n4 - 1));  // clamped: a repeat is harmless
#pragma unroll
      for (int u = 0; u < 4; ++u) { take(x[u].x); take(x[u].y); take(x[u].z); take(x[u].w); }
    }
    for (int64_t i = n4 * 4 + gtid; i < c.n; i += stride) take(__ldcs(p + i));
    flush();
    col_stats_finish(s, (long long)mn, (long long)mx, (long long)mabs, 0);
    return;
  }
  long long mn = LLONG_MAX, mx = LLONG_MIN, mabs = LLONG_MAX;
  auto take64 = [&](long long x) {
    mn = min(mn, x); mx = max(mx, x);
    const long long a = x < 0 ? (x == LLONG_MIN ? LLONG_MAX : -x) : x;
    mabs = min(mabs, a);
    if (sk) hll_add(s_reg, x);
  };
  // 16-byte vectors (two values), four in flight per thread; the odd tail after
  const int64_t n2 = (reinterpret_cast<uintptr_t>(c.data) & 15) ? 0 : c.n / 2;
  const longlong2* p2 = static_cast<const longlong2*>(c.data);
  for (int64_t i0 = gtid; i0 < n2; i0 += 4 * stride) {
    longlong2 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // clamped index: a repeat is harmless for min / max / a sketch
      const int4 t = ld_stream_v4(p2 + min(i0 + u * stride, n2 - 1));
      x[u] = make_longlong2(((long long)(unsigned)t.y << 32) | (unsigned)t.x, ((long long)(unsigned)t.w << 32) | (unsigned)t.z);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) { take64(x[u].x); take64(x[u].y); }
  }
  for (int64_t i = n2 * 2 + gtid; i < c.n; i += stride) take64(__ldcs(static_cast<const long long*>(c.data) + i));
  flush();
  col_stats_finish(s, mn, mx, mabs, 0);
}

__global__ void k_init_stats(ColStats* st, int n) {
  const int i = threadIdx.x;
  if (i < n) { st[i].mn = LLONG_MAX; st[i].mx = LLONG_MIN; st[i].min_abs = LLONG_MAX; st[i].flags = 0; st[i].pad = 0; }
}

// ------------------------------------------------------------------ #distinct sketch
// PAPER.md §4.2.1 keeps "the number of distinct values" per column as
// metadata. For hash-mode domains it is estimated on the device with a HyperLogLog
// sketch (2^12 registers, ~1.6 % standard error) so the hash table is sized by the
// distinct count (L2-resident when small) instead of by the tuple count.
__global__ void __launch_bounds__(1024) k_hll(ColDesc c, unsigned* __restrict__ regs) {
  __shared__ unsigned s_reg[kHllM];
  for (int i = threadIdx.x; i < kHllM; i += blockDim.x) s_reg[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += stride) {
    const unsigned long long h = fmix64((unsigned long long)ld_int(c.data, c.type, i) * 0x9E3779B97F4A7C15ull + 1);
    const unsigned idx = (unsigned)(h >> (64 - kHllP));
    const unsigned long long w = h << kHllP;
    const unsigned rho = w ? (unsigned)__clzll(w) + 1u : (unsigned)(64 - kHllP + 1);
    if (rho > s_reg[idx]) atomicMax(&s_reg[idx], rho);  // most updates stop at the read
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kHllM; i += blockDim.x)
    if (s_reg[i]) atomicMax(regs + i, s_reg[i]);
}

// ------------------------------------------------------------------ direct-offset dictionary
__global__ void k_mark_direct(ColDesc c, long long minv, uint8_t* __restrict__ flags) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < c.n; i += stride)
    flags[(unsigned long long)ld_int(c.data, c.type, i) - (unsigned long long)minv] = 1;
}

// Small spans with many tuples per value (e.g. c4: 67 M tuples over 8,192 keys):
// mark a block-private copy of the flags in shared memory, then write each
// block's set flags once — global stores drop from n to (#blocks x span).
__global__ void __launch_bounds__(1024) k_mark_direct_smem(ColDesc c, long long minv, uint8_t* __restrict__ flags,
                                                          int span) {
  extern __shared__ uint8_t s_flag[];
  for (int i = threadIdx.x; i < span; i += blockDim.x) s_flag[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += stride)
    s_flag[(unsigned long long)ld_int(c.data, c.type, i) - (unsigned long long)minv] = 1;
  __syncthreads();
  for (int i = threadIdx.x; i < span; i += blockDim.x)
    if (s_flag[i]) flags[i] = 1;
}

// ------------------------------------------------------------------ hash dictionary
// Slot key = (x - min) as u64; EMPTY = ~0. Linear probing; equal keys in a warp
// are inserted once (warp aggregation). flags[slot] = 1 marks the side.
__global__ void k_hash_insert(ColDesc c, long long minv, unsigned long long* __restrict__ slots,
                              unsigned long long mask, uint8_t* __restrict__ flags, int* __restrict__ overflow,
                              int32_t* __restrict__ row_slot, int wide) {
  constexpr int U = 4;  // elements per thread per iteration: the first-probe loads overlap
  const int64_t stride = (int64_t)gridDim.x * T;
  const int64_t n_round = (c.n + 31) & ~int64_t(31);
  for (int64_t i0 = (int64_t)blockIdx.x * T + threadIdx.x; i0 < n_round; i0 += U * stride) {
    unsigned long long off[U], h[U], cur[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      ok[u] = i < c.n;
      off[u] = ok[u] ? (unsigned long long)ld_int(c.data, c.type, i) - (unsigned long long)minv
                     : ~0ull - 1 - lane_id();
      h[u] = slot_hash(off[u], wide) & mask;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = ok[u] ? __ldcg(slots + h[u]) : 0ull;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // no warp de-duplication (match.any on 64-bit values costs more than it saves):
      // equal keys in flight both find the slot by the plain read or by the CAS's return
      if (!ok[u]) continue;
      unsigned long long hh = h[u], cc = cur[u];
      bool placed = false;
      for (unsigned long long step = 0; step <= mask; ++step) {  // bounded: a full table is reported
        // plain read first: a key already present (the common case for hot keys) costs no atomic
        if (cc == off[u]) { placed = true; break; }
        if (cc == ~0ull) {
          const unsigned long long prev = atomicCAS(slots + hh, ~0ull, off[u]);
          if (prev == ~0ull || prev == off[u]) { placed = true; break; }
        }
        hh = (hh + 1) & mask;
        cc = __ldcg(slots + hh);
      }
      if (row_slot) row_slot[i0 + u * stride] = placed ? (int32_t)hh : -1;
      if (!placed) { *overflow = 1; continue; }
      if (!flags[hh]) flags[hh] = 1;
    }
  }
}

// Small int32 domains, dictionary only (no per-row slots; c5's group columns: 16.7 M values
// over 4,096 distinct): a sparse block-local set of 32-bit offsets (32,768 slots, stored as
// offset + 1, 0 = empty; load <= 1/8 for the <= 4 K keys a block may hold, so the longest
// probe among a warp's 32 lanes stays short — the linear-probing divergence of a half-full
// table cost ~150 instructions per tuple), 16-byte vector loads four in flight, then the
// block's distinct keys into the global table (same slots and flags as k_hash_insert).
constexpr int kSdThreads = 1024;
constexpr int kSdBits = 15;
__global__ void __launch_bounds__(kSdThreads) k_small_distinct(ColDesc c, long long minv,
                                                               unsigned long long* __restrict__ slots,
                                                               unsigned long long mask, uint8_t* __restrict__ flags,
                                                               int* __restrict__ overflow, int64_t chunk,
                                                               int64_t step) {
  extern __shared__ uint32_t s_set[];
  constexpr int TS = 1 << kSdBits;
  __shared__ int s_n, s_top;
  for (int i = threadIdx.x; i < TS; i += kSdThreads) s_set[i] = 0u;
  if (threadIdx.x == 0) { s_n = 0; s_top = 0; }
  __syncthreads();
  const uint32_t mn = (uint32_t)minv;
  auto ins = [&](int x) {
    const uint32_t k1 = ((uint32_t)x - mn) + 1u;  // offset + 1; offset 2^32 - 1 is kept aside
    if (k1 == 0u) { s_top = 1; return; }
    uint32_t h = (k1 * 0x9E3779B1u) >> (32 - kSdBits);
    while (true) {
      const uint32_t cur = s_set[h];
      if (cur == k1) return;
      if (cur == 0u) {
        const uint32_t prev = atomicCAS(s_set + h, 0u, k1);
        if (prev == 0u) { atomicAdd(&s_n, 1); return; }
        if (prev == k1) return;
      }
      h = (h + 1) & (TS - 1);
    }
  };
  const int32_t* col = static_cast<const int32_t*>(c.data);
  if (step > 1) {
    // sample: tuples 0, step, 2 step, ... (the caller checks every tuple against the result)
    const int64_t m = (c.n + step - 1) / step;
    const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(m, lo + chunk);
    constexpr int U = 8;
    // warp-uniform trip counts: the __syncwarp below needs every lane of the warp
    for (int64_t jw = lo + (threadIdx.x & ~31); jw < hi; jw += U * kSdThreads) {
      const int64_t j0 = jw + lane_id();
      int x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = j0 + u * kSdThreads < hi ? __ldcs(col + (j0 + u * kSdThreads) * step) : 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (j0 + u * kSdThreads < hi) ins(x[u]);
        __syncwarp();
      }
    }
  }
  const int64_t lo = step > 1 ? 0 : (int64_t)blockIdx.x * chunk, hi = step > 1 ? 0 : min(c.n, lo + chunk);  // chunk % 4 == 0
  const int4* c4 = reinterpret_cast<const int4*>(c.data);
  const int64_t v_lo = lo >> 2, v_hi = hi >> 2;
  constexpr int U = 4;
  for (int64_t vw = v_lo + (threadIdx.x & ~31); vw < v_hi; vw += U * kSdThreads) {  // warp-uniform trips
    const int64_t v0 = vw + lane_id();
    int4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = v0 + u * kSdThreads < v_hi ? __ldcs(c4 + v0 + u * kSdThreads) : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (v0 + u * kSdThreads < v_hi) { ins(x[u].x); ins(x[u].y); ins(x[u].z); ins(x[u].w); }
      // reconverge: lanes leaving the probe loops at different steps otherwise run the
      // following iterations in separate groups (measured ~11 of 32 lanes active)
      __syncwarp();
    }
    if (__any_sync(0xffffffffu, s_n > TS / 4)) break;  // > 8 K distinct values in a block: the caller rebuilds by n
  }
  for (int64_t i = (v_hi << 2) + threadIdx.x; i < hi; i += kSdThreads) ins(col[i]);
  __syncthreads();
  if (s_n > TS / 4) {
    if (threadIdx.x == 0) *overflow = 1;
    return;
  }
  for (int sidx = threadIdx.x; sidx <= TS; sidx += kSdThreads) {
    const uint32_t k1 = sidx < TS ? s_set[sidx] : (s_top ? 0u : 1u);  // sidx == TS: offset 2^32 - 1
    if (sidx < TS ? !k1 : k1) continue;
    const unsigned long long off = (unsigned long long)(uint32_t)(k1 - 1u);
    unsigned long long hh = slot_hash(off, 0) & mask;
    int32_t placed = -1;
    for (unsigned long long step = 0; step <= mask; ++step) {
      const unsigned long long cc = __ldcg(slots + hh);
      if (cc == off) { placed = (int32_t)hh; break; }
      if (cc == ~0ull) {
        const unsigned long long prev = atomicCAS(slots + hh, ~0ull, off);
        if (prev == ~0ull || prev == off) { placed = (int32_t)hh; break; }
      }
      hh = (hh + 1) & mask;
    }
    if (placed < 0) *overflow = 1;
    else if (!flags[placed]) flags[placed] = 1;
  }
}

// Small domains with many tuples per value (c5: 16.7 M group values over 4,096
// distinct): every tuple of k_hash_insert reads a slot of a tiny global table, and
// those L2 requests (not bytes) bound it. Here each block first de-duplicates its
// chunk in a shared-memory table (same key encoding and probing, capacity cap_s),
// inserts only its distinct keys into the global table, and maps its tuples to global
// slots from shared memory on a second read of the chunk. A block chunk with more
// than cap_s / 2 distinct keys reports overflow (the caller rebuilds sized by n).
__global__ void __launch_bounds__(1024) k_hash_insert_smem(ColDesc c, long long minv,
                                                          unsigned long long* __restrict__ slots,
                                                          unsigned long long mask, uint8_t* __restrict__ flags,
                                                          int* __restrict__ overflow, int32_t* __restrict__ row_slot,
                                                          int cap_s, int64_t chunk, int wide) {
  extern __shared__ unsigned long long s_key[];
  int32_t* s_map = reinterpret_cast<int32_t*>(s_key + cap_s);
  __shared__ int s_n, s_bad;
  const unsigned smask = (unsigned)cap_s - 1u;
  for (int i = threadIdx.x; i < cap_s; i += blockDim.x) s_key[i] = ~0ull;
  if (threadIdx.x == 0) { s_n = 0; s_bad = 0; }
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * chunk, hi = min(c.n, lo + chunk);
  auto sfind = [&](unsigned long long off, bool insert) -> int {
    unsigned h = (unsigned)slot_hash(off, wide) & smask;
    for (int step = 0; step < cap_s; ++step) {
      const unsigned long long cur = s_key[h];
      if (cur == off) return (int)h;
      if (cur == ~0ull) {
        if (!insert) return -1;
        const unsigned long long prev = atomicCAS(s_key + h, ~0ull, off);
        if (prev == ~0ull) { atomicAdd(&s_n, 1); return (int)h; }
        if (prev == off) return (int)h;
      }
      h = (h + 1) & smask;
    }
    return -1;
  };
  int64_t i_tail = lo;
  if (c.type == 0 && !(reinterpret_cast<uintptr_t>(c.data) & 15) && !(lo & 3)) {
    // int32 column: 16-byte vectors, four in flight per thread (one scalar load at a time
    // kept ~1 K loads in flight per SM: latency-bound at ~0.6 TB/s)
    const int4* c4 = reinterpret_cast<const int4*>(c.data);
    const int64_t v_lo = lo >> 2, v_hi = hi >> 2;
    constexpr int U = 4;
    for (int64_t vw = v_lo + (threadIdx.x & ~31); vw < v_hi; vw += U * blockDim.x) {  // warp-uniform trips
      const int64_t v0 = vw + lane_id();
      int4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = v0 + u * blockDim.x < v_hi ? __ldcs(c4 + v0 + u * blockDim.x) : make_int4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (v0 + u * blockDim.x < v_hi) {
          const int xs[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (sfind((unsigned long long)(long long)xs[q] - (unsigned long long)minv, true) < 0) s_bad = 1;
        }
        __syncwarp();  // reconverge after the probe loops
      }
    }
    i_tail = v_hi << 2;
  }
  for (int64_t i = i_tail + threadIdx.x; i < hi; i += blockDim.x) {
    const unsigned long long off = (unsigned long long)ld_int(c.data, c.type, i) - (unsigned long long)minv;
    if (sfind(off, true) < 0) s_bad = 1;
  }
  __syncthreads();
  if (s_bad || s_n > cap_s / 2 + cap_s / 4) {
    if (threadIdx.x == 0) *overflow = 1;
    return;
  }
  for (int sidx = threadIdx.x; sidx < cap_s; sidx += blockDim.x) {
    const unsigned long long off = s_key[sidx];
    if (off == ~0ull) continue;
    unsigned long long hh = slot_hash(off, wide) & mask;
    int32_t placed = -1;
    for (unsigned long long step = 0; step <= mask; ++step) {
      const unsigned long long cc = __ldcg(slots + hh);
      if (cc == off) { placed = (int32_t)hh; break; }
      if (cc == ~0ull) {
        const unsigned long long prev = atomicCAS(slots + hh, ~0ull, off);
        if (prev == ~0ull || prev == off) { placed = (int32_t)hh; break; }
      }
      hh = (hh + 1) & mask;
    }
    s_map[sidx] = placed;
    if (placed < 0) *overflow = 1;
    else if (!flags[placed]) flags[placed] = 1;
  }
  if (!row_slot) return;  // dictionary only: the caller looks values up itself
  __syncthreads();
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const unsigned long long off = (unsigned long long)ld_int(c.data, c.type, i) - (unsigned long long)minv;
    __stcs(row_slot + i, s_map[sfind(off, false)]);
  }
}

// ------------------------------------------------------------------ predicate scan -> codes
// pred(i) = fa[i] && (fb ? fb[i] : 1). Tile = 4096 flags per 256-thread block.
constexpr int PT = 4096;
__global__ void k_pred_count(const uint8_t* __restrict__ fa, const uint8_t* __restrict__ fb, int64_t n,
                             int32_t* __restrict__ tile_cnt, unsigned long long* __restrict__ union_cnt) {
  const int64_t base = (int64_t)blockIdx.x * PT + threadIdx.x * 16;
  int c = 0, u = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int64_t i = base + j;
    if (i < n) {
      const int a = fa[i], b = fb ? fb[i] : 1;
      c += a & b;
      if (fb) u += a | b;
    }
  }
  c = warp_sum(c); u = warp_sum(u);
  __shared__ int sc[T / 32], su[T / 32];
  if (lane_id() == 0) { sc[warp_id()] = c; su[warp_id()] = u; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int tc = 0, tu = 0;
    for (int w = 0; w < T / 32; ++w) { tc += sc[w]; tu += su[w]; }
    tile_cnt[blockIdx.x] = tc;
    if (union_cnt && tu) atomicAdd(union_cnt, (unsigned long long)tu);
  }
}

// Single-block variant for spans up to ~1 M flags (one launch instead of count +
// scan + codes): 1024 threads sweep the flags in 16 K chunks with a running offset;
// also writes the total, the ∪ count, and (direct group domains) dict[code] = min + x.
__device__ __forceinline__ void pred_codes_1blk_body(const uint8_t* __restrict__ fa,
                                                          const uint8_t* __restrict__ fb, int64_t n,
                                                          int32_t* __restrict__ code, int64_t* __restrict__ count,
                                                          unsigned long long* __restrict__ union_cnt,
                                                          long long* __restrict__ dict, long long minv) {
  __shared__ int wt[32];
  __shared__ long long s_run;
  if (threadIdx.x == 0) s_run = 0;
  long long u = 0;
  for (int64_t base0 = 0; base0 < n; base0 += 1024 * 16) {
    const int64_t base = base0 + (int64_t)threadIdx.x * 16;
    uint8_t p[16];
    int c = 0;
    if (base + 16 <= n) {  // 16 flags per thread as one 16-byte load (spans are 16-byte aligned allocations)
      const uint4 va = *reinterpret_cast<const uint4*>(fa + base);
      const uint4 vb = fb ? *reinterpret_cast<const uint4*>(fb + base) : make_uint4(~0u, ~0u, ~0u, ~0u);
      const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int a = (wa[j >> 2] >> (8 * (j & 3))) & 1, b = (wb[j >> 2] >> (8 * (j & 3))) & 1;
        p[j] = (uint8_t)(a & b);
        c += p[j];
        if (fb) u += a | b;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t i = base + j;
        const int a = i < n ? fa[i] : 0, b = (i < n) ? (fb ? fb[i] : 1) : 0;
        p[j] = (uint8_t)(a & b);
        c += p[j];
        if (fb) u += a | b;
      }
    }
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o); if (lane_id() >= o) x += y; }
    if (lane_id() == 31) wt[warp_id()] = x;
    __syncthreads();
    int wp = 0, tot = 0;
    for (int w = 0; w < 32; ++w) { const int t = wt[w]; if (w < warp_id()) wp += t; tot += t; }
    long long run = s_run + wp + x - c;
    int32_t cv[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int64_t i = base + j;
      cv[j] = p[j] ? (int32_t)run : -1;
      if (i < n && p[j] && dict) dict[run] = minv + (long long)i;
      run += p[j];
    }
    if (base + 16 <= n) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        reinterpret_cast<int4*>(code + base)[j] = make_int4(cv[4 * j], cv[4 * j + 1], cv[4 * j + 2], cv[4 * j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (base + j < n) code[base + j] = cv[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) s_run += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = s_run;
  if (union_cnt) {
    u = warp_sum(u);
    if (lane_id() == 0 && u) atomicAdd(union_cnt, (unsigned long long)u);
  }
}

__global__ void __launch_bounds__(1024) k_pred_codes_1blk(const uint8_t* __restrict__ fa,
                                                          const uint8_t* __restrict__ fb, int64_t n,
                                                          int32_t* __restrict__ code, int64_t* __restrict__ count,
                                                          unsigned long long* __restrict__ union_cnt,
                                                          long long* __restrict__ dict, long long minv) {
  pred_codes_1blk_body(fa, fb, n, code, count, union_cnt, dict, minv);
}

// up to three small dictionaries' codes in one launch (one block each: the key, A.g and B.h
// dictionaries of a query), instead of three dependent single-block launches
__global__ void __launch_bounds__(1024) k_pred_codes_1blk_multi(PredJob j0, PredJob j1, PredJob j2) {
  const PredJob& j = blockIdx.x == 0 ? j0 : blockIdx.x == 1 ? j1 : j2;
  pred_codes_1blk_body(j.fa, j.fb, j.n, j.code, j.count, j.union_cnt, j.dict, j.minv);
}

__global__ void k_pred_codes(const uint8_t* __restrict__ fa, const uint8_t* __restrict__ fb, int64_t n,
                             const int64_t* __restrict__ tile_off, int32_t* __restrict__ code,
                             long long* __restrict__ dict, long long minv) {
  const int64_t base = (int64_t)blockIdx.x * PT + threadIdx.x * 16;
  uint8_t p[16];
  int c = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int64_t i = base + j;
    p[j] = (i < n) ? (uint8_t)(fa[i] & (fb ? fb[i] : 1)) : 0;
    c += p[j];
  }
  // block exclusive scan of c
  int x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o); if (lane_id() >= o) x += y; }
  __shared__ int wt[T / 32];
  if (lane_id() == 31) wt[warp_id()] = x;
  __syncthreads();
  int wp = 0;
  for (int w = 0; w < warp_id(); ++w) wp += wt[w];
  int64_t run = tile_off[blockIdx.x] + wp + x - c;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int64_t i = base + j;
    if (i < n) {
      code[i] = p[j] ? (int32_t)run : -1;
      if (p[j] && dict) dict[run] = minv + (long long)i;
      run += p[j];
    }
  }
}

// ------------------------------------------------------------------ group dictionaries
// direct: dict[code[x]] = min + x
__global__ void k_direct_dict(const int32_t* __restrict__ code, int64_t range, long long minv,
                              long long* __restrict__ dict) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t x = (int64_t)blockIdx.x * T + threadIdx.x; x < range; x += stride) {
    const int32_t c = code[x];
    if (c >= 0) dict[c] = minv + (long long)x;
  }
}
// hash: gather (slot key, slot) pairs of occupied slots into compaction order
__global__ void k_gather_slots(const int32_t* __restrict__ tmp_code, const unsigned long long* __restrict__ slots,
                               int64_t cap, unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t s = (int64_t)blockIdx.x * T + threadIdx.x; s < cap; s += stride) {
    const int32_t c = tmp_code[s];
    if (c >= 0) { keys[c] = slots[s]; vals[c] = (uint32_t)s; }
  }
}
// hash: after sorting by key, rank i -> slot_code[slot] = i, dict[i] = min + key
// remap (optional): remap[old compaction-order code] = rank, for codes already handed out
__global__ void k_rank_write(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals,
                             int64_t n, long long minv, int32_t* __restrict__ slot_code,
                             long long* __restrict__ dict, int32_t* __restrict__ remap) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    if (remap) remap[slot_code[vals[i]]] = (int32_t)i;
    slot_code[vals[i]] = (int32_t)i;
    dict[i] = (long long)(keys[i] + (unsigned long long)minv);
  }
}

constexpr int SMALL_SORT = 4096;  // small hash-mode group domains: rank by counting

// Rank by counting for small domains (<= SMALL_SORT values): gather the distinct keys
// (code_in[slot] >= 0) into code order, then every value's rank = #{keys < it}, computed
// by many blocks against a shared-memory copy of all keys (keys are distinct).
__global__ void k_small_gather(const int32_t* __restrict__ code_in, const unsigned long long* __restrict__ slots,
                               int64_t cap, unsigned long long* __restrict__ keys, int32_t* __restrict__ slot_of) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < cap; s += stride) {
    const int32_t c = code_in[s];
    if (c >= 0) { keys[c] = slots[s]; slot_of[c] = (int32_t)s; }
  }
}

__global__ void __launch_bounds__(256) k_small_count_rank(const unsigned long long* __restrict__ keys,
                                                          const int32_t* __restrict__ slot_of, int count,
                                                          long long minv, int32_t* __restrict__ slot_code,
                                                          long long* __restrict__ dict, int32_t* __restrict__ remap) {
  // 32 keys per CTA (one per lane); warp w counts the smaller keys in the w-th eighth of
  // the array, the eighths are summed in shared memory (count / 32 CTAs spread the O(n^2)
  // comparisons over the SMs: 16 CTAs of one key per thread took 41 us at n = 4,096)
  __shared__ unsigned long long sk[SMALL_SORT];
  __shared__ int part[8][32];
  for (int i = threadIdx.x; i < count; i += blockDim.x) sk[i] = keys[i];
  __syncthreads();
  const int lane = lane_id(), w = warp_id();
  const int c = blockIdx.x * 32 + lane;
  const unsigned long long x = c < count ? sk[c] : 0ull;
  const int per = (count + 7) / 8, lo = w * per, hi = min(count, lo + per);
  int r = 0;
#pragma unroll 8
  for (int i = lo; i < hi; ++i) r += sk[i] < x;  // broadcast reads: no bank conflicts
  part[w][lane] = r;
  __syncthreads();
  if (w != 0 || c >= count) return;
  r = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) r += part[q][lane];
  if (remap) remap[c] = r;
  slot_code[slot_of[c]] = r;
  dict[r] = (long long)(x + (unsigned long long)minv);
}

__global__ void k_remap_codes(int32_t* __restrict__ codes, int64_t n, const int32_t* __restrict__ remap) {
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) {
    const int32_t c = codes[i];
    if (c >= 0) codes[i] = remap[c];
  }
}

// ------------------------------------------------------------------ probe (codes per tuple)
// Codes of rows i0 + u * stride: through the insert's per-row slots when present
// (code[row_slot[i]], one gather from an L2-sized table), else by value.
template <int U>
TCUDB_DEV void rows_lookup(const DictView& d, const long long* x, const bool* ok, int64_t i0, int64_t stride,
                           int32_t* out) {
  if (d.row_slot) {
    int32_t sl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) sl[u] = ok[u] ? __ldcs(d.row_slot + i0 + u * stride) : -1;
#pragma unroll
    for (int u = 0; u < U; ++u) out[u] = sl[u] >= 0 ? __ldg(d.code + sl[u]) : -1;
    return;
  }
  dict_lookup_batch<U>(d, x, ok, out);
}

// kcode / gcode per tuple; per-key counts (warp-aggregated); per-group tuple
// counts and sum |v| of tuples whose key survives the ∩ (guard bounds, a3).
// Variant with the per-key counters privatized in shared memory (small key
// domains with many tuples per key, e.g. c4: 8,192 keys x 8,192 tuples each):
// smem atomics, then one global atomic per key per block.
__global__ void __launch_bounds__(1024) k_probe_smem(ColDesc key, ColDesc grp, DictView kd, DictView gd,
                                                     int32_t* __restrict__ kcode, int32_t* __restrict__ gcode,
                                                     int32_t* __restrict__ cnt_k, int K) {
  extern __shared__ int32_t s_cnt[];
  for (int k = threadIdx.x; k < K; k += blockDim.x) s_cnt[k] = 0;
  __syncthreads();
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < key.n; i0 += U * stride) {
    long long xk[U], xg[U];
    bool ok[U];
    int32_t kc[U], gc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      ok[u] = i < key.n;
      xk[u] = ok[u] ? ld_int(key.data, key.type, i) : 0;
      xg[u] = ok[u] ? ld_int(grp.data, grp.type, i) : 0;
    }
    dict_lookup_batch<U>(kd, xk, ok, kc);
    dict_lookup_batch<U>(gd, xg, ok, gc);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) continue;
      const int64_t i = i0 + u * stride;
      kcode[i] = kc[u];
      gcode[i] = gc[u];
      if (kc[u] >= 0) atomicAdd(s_cnt + kc[u], 1);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    if (s_cnt[k]) atomicAdd(cnt_k + k, s_cnt[k]);
}

// Same result as k_probe_smem for int32 columns whose key and group dictionaries are
// both direct (code = table[x - min]) and small: the two code tables sit in shared
// memory next to the counters (a random gather from shared memory costs a few bank
// conflicts; from L1 it costs one wavefront per distinct 128-byte line), and each
// thread moves 16-byte vectors: 4 keys + 4 groups in, 4 + 4 codes out.
__global__ void __launch_bounds__(1024) k_probe_direct_smem(const int32_t* __restrict__ key,
                                                            const int32_t* __restrict__ grp, int64_t n,
                                                            DictView kd, DictView gd, int32_t* __restrict__ kcode,
                                                            int32_t* __restrict__ gcode,
                                                            int32_t* __restrict__ cnt_k, int K) {
  extern __shared__ int32_t s_cnt[];
  int32_t* s_kd = s_cnt + K;
  int32_t* s_gd = s_kd + kd.size;
  for (int k = threadIdx.x; k < K; k += blockDim.x) s_cnt[k] = 0;
  for (int i = threadIdx.x; i < (int)kd.size; i += blockDim.x) s_kd[i] = __ldg(kd.code + i);
  for (int i = threadIdx.x; i < (int)gd.size; i += blockDim.x) s_gd[i] = __ldg(gd.code + i);
  __syncthreads();
  const unsigned ks = (unsigned)kd.size, gs = (unsigned)gd.size;
  const int kmin = (int)kd.minv, gmin = (int)gd.minv;
  auto one = [&](int x, int y, int& kc, int& gc) {
    const unsigned ok = (unsigned)x - (unsigned)kmin, og = (unsigned)y - (unsigned)gmin;
    kc = ok < ks ? s_kd[ok] : -1;
    gc = og < gs ? s_gd[og] : -1;
    if (kc >= 0) atomicAdd(s_cnt + kc, 1);
  };
  const int64_t n4 = n / 4;
  const int4* k4 = reinterpret_cast<const int4*>(key);
  const int4* g4 = reinterpret_cast<const int4*>(grp);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n4; v += 2 * stride) {
    const bool two = v + stride < n4;
    const int4 xa = __ldcs(k4 + v), ya = __ldcs(g4 + v);
    int4 xb = xa, yb = ya;
    if (two) { xb = __ldcs(k4 + v + stride); yb = __ldcs(g4 + v + stride); }
    int4 ka, ga, kb, gb;
    one(xa.x, ya.x, ka.x, ga.x); one(xa.y, ya.y, ka.y, ga.y);
    one(xa.z, ya.z, ka.z, ga.z); one(xa.w, ya.w, ka.w, ga.w);
    reinterpret_cast<int4*>(kcode)[v] = ka;
    reinterpret_cast<int4*>(gcode)[v] = ga;
    if (two) {
      one(xb.x, yb.x, kb.x, gb.x); one(xb.y, yb.y, kb.y, gb.y);
      one(xb.z, yb.z, kb.z, gb.z); one(xb.w, yb.w, kb.w, gb.w);
      reinterpret_cast<int4*>(kcode)[v + stride] = kb;
      reinterpret_cast<int4*>(gcode)[v + stride] = gb;
    }
  }
  for (int64_t i = n4 * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    one(key[i], grp[i], kcode[i], gcode[i]);
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    if (s_cnt[k]) atomicAdd(cnt_k + k, s_cnt[k]);
}

__global__ void k_probe(ColDesc key, ColDesc grp, ColDesc val, DictView kd, DictView gd,
                        int32_t* __restrict__ kcode, int32_t* __restrict__ gcode, int32_t* __restrict__ cnt_k,
                        double* __restrict__ rowabs_g) {
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * T;
  const int64_t n_round = (key.n + 31) & ~int64_t(31);
  for (int64_t i0 = (int64_t)blockIdx.x * T + threadIdx.x; i0 < n_round; i0 += U * stride) {
  long long xk[U], xg[U];
  bool okv[U];
  int32_t kcv[U], gcv[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + u * stride;
    okv[u] = i < key.n;
    xk[u] = okv[u] && !kd.row_slot ? ld_int(key.data, key.type, i) : 0;
    xg[u] = okv[u] && !gd.row_slot ? ld_int(grp.data, grp.type, i) : 0;
  }
  rows_lookup<U>(kd, xk, okv, i0, stride, kcv);
  rows_lookup<U>(gd, xg, okv, i0, stride, gcv);
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + u * stride;
    if (i >= n_round) break;  // warp-uniform
    const bool ok = okv[u];
    const int32_t kc = ok ? kcv[u] : -1, gc = ok ? gcv[u] : -1;
    if (ok) { kcode[i] = kc; gcode[i] = gc; }
    const int32_t kk = (ok && kc >= 0) ? kc : -2 - lane_id();
    const unsigned peers = __match_any_sync(0xffffffffu, kk);
    if (ok && kc >= 0 && (__ffs(peers) - 1) == lane_id()) atomicAdd(cnt_k + kc, __popc(peers));
    if (ok && kc >= 0 && rowabs_g) {
      // sum |v| per group in fp64 (a bound only: no wrap-around, relative rounding ~1e-16 * n)
      double a = 1.0;
      if (val.data) {
        if (val.type == 2) a = 0.0;  // float: bound not needed
        else a = fabs((double)ld_int(val.data, val.type, i));
      }
      atomicAdd(rowabs_g + gc, a);
    }
  }
  }
}

// Group codes from a small finished hash dictionary (<= 16 K slots, offsets of 32 bits, int32
// column): each CTA copies the slots (as 32-bit offsets) and their codes into shared memory
// and maps 16-byte vectors of the column (a global-table probe per tuple was L2-latency-bound).
constexpr int kGcThreads = 1024;
constexpr int kGcMaxCap = 16384;
constexpr int kGcBits = 14;  // 16,384 shared slots: load <= 1/4 for <= 4 K groups
__global__ void __launch_bounds__(kGcThreads) k_group_codes_smem(ColDesc grp, DictView gd, int32_t* __restrict__ gcode,
                                                                 int* __restrict__ miss) {
  extern __shared__ __align__(16) unsigned long long s_gt[];  // (offset << 32 | code), ~0 = empty
  constexpr int TS = 1 << kGcBits;
  for (int i = threadIdx.x; i < TS; i += kGcThreads) s_gt[i] = ~0ull;
  __syncthreads();
  auto sh = [](uint32_t off) { return (off * 0x9E3779B1u) >> (32 - kGcBits); };
  const int cap = (int)gd.size + 1;  // hash mode: size = mask
  for (int i = threadIdx.x; i < cap; i += kGcThreads) {
    const unsigned long long k = __ldg(gd.slots + i);
    if (k == ~0ull) continue;
    const unsigned long long w = (k << 32) | (uint32_t)__ldg(gd.code + i);
    uint32_t h = sh((uint32_t)k);
    while (atomicCAS(s_gt + h, ~0ull, w) != ~0ull) h = (h + 1) & (TS - 1);
  }
  __syncthreads();
  const unsigned mn = (unsigned)gd.minv;
  int missed = 0;
  auto look = [&](int x) -> int32_t {
    const uint32_t off = (uint32_t)x - mn;
    uint32_t h = sh(off);
    while (true) {
      const unsigned long long w = s_gt[h];
      if ((uint32_t)(w >> 32) == off && w != ~0ull) return (int32_t)(uint32_t)w;
      if (w == ~0ull) { missed = 1; return -1; }
      h = (h + 1) & (TS - 1);
    }
  };
  const int64_t nv = grp.n / 4;
  const int4* g4 = reinterpret_cast<const int4*>(grp.data);
  int4* o4 = reinterpret_cast<int4*>(gcode);
  const int64_t stride = (int64_t)gridDim.x * kGcThreads;
  constexpr int U = 4;
  for (int64_t vw = (int64_t)blockIdx.x * kGcThreads + (threadIdx.x & ~31); vw < nv; vw += U * stride) {  // warp-uniform
    const int64_t v0 = vw + lane_id();
    int4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = v0 + u * stride < nv ? __ldcs(g4 + v0 + u * stride) : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (v0 + u * stride < nv) __stcg(o4 + v0 + u * stride, make_int4(look(x[u].x), look(x[u].y), look(x[u].z), look(x[u].w)));
      __syncwarp();  // reconverge after the probe loops
    }
  }
  for (int64_t i = nv * 4 + (int64_t)blockIdx.x * kGcThreads + threadIdx.x; i < grp.n; i += stride)
    gcode[i] = look(static_cast<const int32_t*>(grp.data)[i]);
  if (miss && __any_sync(0xffffffffu, missed) && lane_id() == 0) atomicOr(miss, 1);
}

// Group codes only (the hash-partitioned sparse path encodes the join key itself).
__global__ void k_group_codes(ColDesc grp, DictView gd, int32_t* __restrict__ gcode, int* __restrict__ miss) {
  int missed = 0;
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * T;
  for (int64_t i0 = (int64_t)blockIdx.x * T + threadIdx.x; i0 < grp.n; i0 += U * stride) {
    long long x[U];
    bool ok[U];
    int32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      ok[u] = i < grp.n;
      x[u] = ok[u] && !gd.row_slot ? ld_int(grp.data, grp.type, i) : 0;
    }
    rows_lookup<U>(gd, x, ok, i0, stride, c);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (ok[u]) { gcode[i0 + u * stride] = c[u]; missed |= c[u] < 0; }
  }
  if (miss && missed) atomicOr(miss, 1);
}

// J = sum_k cntA[k] * cntB[k] (join size, a4) and max per-key counts.
// out[0] = J = sum_k cntA[k]*cntB[k]; out[3] = sum cntA, out[4] = sum cntB (tuples with a
// key in the ∩ domain on each side)
__global__ void k_join_size(const int32_t* __restrict__ ca, const int32_t* __restrict__ cb, int64_t K,
                            unsigned long long* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * T;
  unsigned long long s = 0, sa = 0, sb = 0;
  for (int64_t k = (int64_t)blockIdx.x * T + threadIdx.x; k < K; k += stride) {
    const unsigned long long a = (unsigned)ca[k], b = (unsigned)cb[k];
    s += a * b;
    if (b) sa += a;
    if (a) sb += b;
  }
  s = warp_sum(s); sa = warp_sum(sa); sb = warp_sum(sb);
  if (lane_id() == 0) {
    if (s) atomicAdd(out, s);
    if (sa) atomicAdd(out + 3, sa);
    if (sb) atomicAdd(out + 4, sb);
  }
}

// number of set bits of (w & mask) over n words (occupancy maps, fp4 nibble maps)
__global__ void k_popcount(const unsigned* __restrict__ w, int64_t n, unsigned mask,
                           unsigned long long* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * T;
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) c += __popc(__ldcs(w + i) & mask);
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(out, c);
}

__global__ void k_max_u64(const unsigned long long* __restrict__ x, int64_t n, unsigned long long* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * T;
  unsigned long long m = 0;
  for (int64_t i = (int64_t)blockIdx.x * T + threadIdx.x; i < n; i += stride) m = max(m, x[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0 && m) atomicMax(out, m);
}

inline int grid_for(int64_t n, int per_block = T * 4) {
  int64_t g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > kNumSMs * 16) g = kNumSMs * 16;
  return (int)g;
}

}  // namespace

// ------------------------------------------------------------------ launchers
cudaError_t launch_col_stats(const ColDesc* cols, ColStats* st, cudaStream_t s, int64_t* launches, unsigned* hll,
                             int* gate) {
  k_init_stats<<<1, 32, 0, s>>>(st, 6);
  int64_t nmax = 1;
  for (int i = 0; i < 6; ++i) if (cols[i].data && cols[i].n > nmax) nmax = cols[i].n;
  dim3 grid((unsigned)std::min<int64_t>(2 * kNumSMs, (nmax + T * 16 - 1) / (T * 16)), 6);
  if (hll) {
    k_sketch_gate<<<4, 1024, 0, s>>>(cols[0], cols[1], cols[2], cols[3], gate);
    k_col_stats<true><<<grid, T, 0, s>>>(cols[0], cols[1], cols[2], cols[3], cols[4], cols[5], st, hll, gate);
    if (launches) ++*launches;
  } else {
    k_col_stats<false><<<grid, T, 0, s>>>(cols[0], cols[1], cols[2], cols[3], cols[4], cols[5], st, nullptr,
                                          nullptr);
  }
  if (launches) *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_hll(const ColDesc& c, unsigned* regs, cudaStream_t s, int64_t* launches) {
  if (c.n <= 0) return cudaSuccess;
  int64_t blocks = (c.n + 16 * 1024 - 1) / (16 * 1024);
  if (blocks > kNumSMs) blocks = kNumSMs;
  k_hll<<<(int)blocks, 1024, 0, s>>>(c, regs);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_mark_direct(const ColDesc& c, long long minv, uint8_t* flags, int64_t span, cudaStream_t s,
                               int64_t* launches) {
  if (c.n <= 0) return cudaSuccess;
  // Same-address global stores serialize in L2 (a Zipf-hot key written by thousands of
  // threads): mark in shared memory instead whenever the span fits, so each block
  // stores each set flag once.
  if (span <= 64 * 1024 && c.n >= 4096) {
    set_func_attr(k_mark_direct_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    // enough tuples per block to amortize zeroing and flushing the span
    int64_t blocks = c.n / std::max<int64_t>(4096, span / 4);
    if (blocks > 2 * kNumSMs) blocks = 2 * kNumSMs;
    if (blocks < 1) blocks = 1;
    k_mark_direct_smem<<<(int)blocks, 1024, (size_t)span, s>>>(c, minv, flags, (int)span);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  k_mark_direct<<<grid_for(c.n), T, 0, s>>>(c, minv, flags);
  if (launches) ++*launches;
  return cudaGetLastError();
}


cudaError_t launch_hash_insert(const ColDesc& c, long long minv, unsigned long long* slots, unsigned long long mask,
                               uint8_t* flags, int* overflow, int32_t* row_slot, double est_distinct, int wide,
                               cudaStream_t s, int64_t* launches, int64_t sample_step) {
  if (c.n <= 0) return cudaSuccess;
  // shared-memory pre-aggregation when the estimated distinct count is small and
  // there are many tuples per distinct value (tables sized 2^ceil(log2(1.9 est)))
  const int64_t cap = (int64_t)mask + 1;
  if (est_distinct > 0 && cap <= 16384 && c.n >= 64 * cap && !row_slot && !wide && c.type == 0 &&
      !(reinterpret_cast<uintptr_t>(c.data) & 15)) {
    constexpr int smem = (1 << kSdBits) * 4;
    cudaError_t e = set_func_attr(k_small_distinct, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    // one block per SM (TCUDB_SD_BLOCKS overrides: experiments)
    // every block ends by inserting each distinct key it saw into the global table (all of a
    // small domain's keys, typically; those few L2 lines serialize the merges): sampled builds
    // use 16 blocks (measured 2 / 4 / 8 / 16 on c5's groups: 213 / 140 / 103 / 95 us)
    static const int env_nb = getenv("TCUDB_SD_BLOCKS") ? atoi(getenv("TCUDB_SD_BLOCKS")) : 0;
    const int64_t step = sample_step > 1 ? sample_step : 1;
    const int64_t m = (c.n + step - 1) / step;
    const int64_t nblk = std::max<int64_t>(1, std::min<int64_t>(env_nb > 0 ? env_nb : (step > 1 ? 16 : kNumSMs),
                                                                (m + 16383) / 16384));
    const int64_t chunk = ((m + nblk - 1) / nblk + 3) & ~int64_t(3);
    k_small_distinct<<<(int)nblk, kSdThreads, smem, s>>>(c, minv, slots, mask, flags, overflow, chunk, step);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  if (est_distinct > 0 && cap <= 16384 && c.n >= 64 * cap) {
    const int cap_s = (int)cap;  // >= 1.9 x the global distinct count, so >= any block's
    const size_t smem = (size_t)cap_s * 12;
    set_func_attr(k_hash_insert_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 12);
    const int per_sm = smem <= 96 * 1024 ? 2 : 1;
    const int64_t nblk = std::min<int64_t>(per_sm * kNumSMs, (c.n + 32767) / 32768);
    const int64_t chunk = ((c.n + nblk - 1) / nblk + 3) & ~int64_t(3);  // 16-byte aligned chunks
    k_hash_insert_smem<<<(int)nblk, 1024, smem, s>>>(c, minv, slots, mask, flags, overflow, row_slot, cap_s, chunk,
                                                      wide);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  k_hash_insert<<<grid_for(c.n), T, 0, s>>>(c, minv, slots, mask, flags, overflow, row_slot, wide);
  if (launches) ++*launches;
  return cudaGetLastError();
}

size_t pred_temp_bytes(int64_t n) {
  const int64_t nt = (n + PT - 1) / PT;
  return ((size_t)nt * 4 + 15) / 16 * 16 + (size_t)nt * 8 + scan_temp_bytes(nt) + 64;
}

cudaError_t launch_pred_codes(const uint8_t* fa, const uint8_t* fb, int64_t n, int32_t* code, int64_t* count_dev,
                              unsigned long long* union_dev, long long* dict, long long minv, void* temp,
                              cudaStream_t s, int64_t* launches) {
  const int64_t nt = (n + PT - 1) / PT;
  if (n <= 0) return exclusive_scan_i32(nullptr, nullptr, 0, count_dev, temp, s, launches);
  if (n <= 32768) {  // spans up to 32 K: one launch (2 sweeps of one block); larger: the 3-pass scan
    k_pred_codes_1blk<<<1, 1024, 0, s>>>(fa, fb, n, code, count_dev, union_dev, dict, minv);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  int32_t* tc = static_cast<int32_t*>(temp);
  int64_t* toff = reinterpret_cast<int64_t*>(static_cast<char*>(temp) + ((size_t)nt * 4 + 15) / 16 * 16);
  void* st = toff + nt;
  k_pred_count<<<(unsigned)nt, T, 0, s>>>(fa, fb, n, tc, union_dev);
  if (launches) ++*launches;
  cudaError_t e = exclusive_scan_i32(tc, toff, nt, count_dev, st, s, launches);
  if (e != cudaSuccess) return e;
  k_pred_codes<<<(unsigned)nt, T, 0, s>>>(fa, fb, n, toff, code, dict, minv);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_pred_codes_multi(const PredJob* jobs, int nj, void* const* temps, cudaStream_t s,
                                    int64_t* launches) {
  bool small = nj >= 1 && nj <= 3;
  for (int i = 0; i < nj && small; ++i) small = jobs[i].n > 0 && jobs[i].n <= 32768;
  if (small) {
    const PredJob none{};
    k_pred_codes_1blk_multi<<<nj, 1024, 0, s>>>(jobs[0], nj > 1 ? jobs[1] : none, nj > 2 ? jobs[2] : none);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  for (int i = 0; i < nj; ++i) {
    const PredJob& j = jobs[i];
    const cudaError_t e = launch_pred_codes(j.fa, j.fb, j.n, j.code, j.count, j.union_cnt, j.dict, j.minv, temps[i],
                                            s, launches);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_direct_dict(const int32_t* code, int64_t range, long long minv, long long* dict, cudaStream_t s,
                               int64_t* launches) {
  k_direct_dict<<<grid_for(range), T, 0, s>>>(code, range, minv, dict);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_gather_slots(const int32_t* tmp_code, const unsigned long long* slots, int64_t cap,
                                unsigned long long* keys, uint32_t* vals, cudaStream_t s, int64_t* launches) {
  k_gather_slots<<<grid_for(cap), T, 0, s>>>(tmp_code, slots, cap, keys, vals);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_rank_write(const unsigned long long* keys, const uint32_t* vals, int64_t n, long long minv,
                              int32_t* slot_code, long long* dict, int32_t* remap, cudaStream_t s,
                              int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_rank_write<<<grid_for(n), T, 0, s>>>(keys, vals, n, minv, slot_code, dict, remap);
  if (launches) ++*launches;
  return cudaGetLastError();
}

// (gather + rank by counting of <= 4 K values vs ~12 launches of the radix sort)
bool small_rank_ok(int64_t count, int64_t cap) { return count <= SMALL_SORT && cap <= (1 << 16); }

size_t small_rank_temp_bytes() { return (size_t)SMALL_SORT * 12 + 256; }

cudaError_t launch_small_rank(const int32_t* code, const unsigned long long* slots, int64_t cap, int64_t count,
                              long long minv, int32_t* slot_code, long long* dict, int32_t* remap, void* temp,
                              cudaStream_t s, int64_t* launches) {
  if (count <= 0) return cudaSuccess;
  unsigned long long* keys = static_cast<unsigned long long*>(temp);
  int32_t* slot_of = reinterpret_cast<int32_t*>(keys + SMALL_SORT);
  k_small_gather<<<grid_for(cap), T, 0, s>>>(code, slots, cap, keys, slot_of);
  k_small_count_rank<<<(unsigned)((count + 31) / 32), 256, 0, s>>>(keys, slot_of, (int)count, minv, slot_code, dict,
                                                                   remap);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_remap_codes(int32_t* codes, int64_t n, const int32_t* remap, cudaStream_t s, int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_remap_codes<<<grid_for(n), T, 0, s>>>(codes, n, remap);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_probe(const ColDesc& key, const ColDesc& grp, const ColDesc& val, const DictView& kd,
                         const DictView& gd, int32_t* kcode, int32_t* gcode, int32_t* cnt_k,
                         double* rowabs_g, int64_t K, cudaStream_t s, int64_t* launches) {
  if (key.n <= 0) return cudaSuccess;
  // privatized counters when the key domain fits in shared memory and there are
  // enough tuples per block to amortize the per-block flush
  const int64_t smem = K * 4;
  auto fits_i32 = [](long long v) { return v >= INT_MIN && v <= INT_MAX; };
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const int64_t smem_d = smem + 4 * (int64_t)(kd.size + gd.size);
  if (!rowabs_g && K > 0 && key.n >= 4 * K && key.type == 0 && grp.type == 0 && kd.mode == 0 && gd.mode == 0 &&
      fits_i32(kd.minv) && fits_i32(gd.minv) && smem_d <= 100 * 1024 && al16(key.data) && al16(grp.data) &&
      al16(kcode) && al16(gcode)) {
    set_func_attr(k_probe_direct_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    int64_t blocks = key.n / 4096;
    if (blocks > 2 * kNumSMs) blocks = 2 * kNumSMs;
    if (blocks < 1) blocks = 1;
    k_probe_direct_smem<<<(int)blocks, 1024, (size_t)smem_d, s>>>(static_cast<const int32_t*>(key.data),
                                                                  static_cast<const int32_t*>(grp.data), key.n, kd,
                                                                  gd, kcode, gcode, cnt_k, (int)K);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  if (!rowabs_g && K > 0 && smem <= 200 * 1024 && key.n >= 4 * K) {
    set_func_attr(k_probe_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int64_t blocks = key.n / 2048;  // >= 2 tuples per thread; the flush is K / 1024 steps per block
    if (blocks > kNumSMs) blocks = kNumSMs;
    if (blocks < 1) blocks = 1;
    k_probe_smem<<<(int)blocks, 1024, (size_t)smem, s>>>(key, grp, kd, gd, kcode, gcode, cnt_k, (int)K);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  k_probe<<<grid_for(key.n), T, 0, s>>>(key, grp, val, kd, gd, kcode, gcode, cnt_k, rowabs_g);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_group_codes(const ColDesc& grp, const DictView& gd, int32_t* gcode, cudaStream_t s,
                               int64_t* launches, int* miss) {
  if (grp.n <= 0) return cudaSuccess;
  if (gd.mode == 1 && !gd.wide && !gd.row_slot && grp.type == 0 && gd.size + 1 <= (unsigned long long)kGcMaxCap &&
      gd.size + 1 <= (1ull << kGcBits) / 2 &&
      !(reinterpret_cast<uintptr_t>(grp.data) & 15) && !(reinterpret_cast<uintptr_t>(gcode) & 15) &&
      grp.n >= 64 * (int64_t)(gd.size + 1)) {
    const int smem = (1 << kGcBits) * 8;
    cudaError_t e = set_func_attr(k_group_codes_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int per_sm = smem <= 100 * 1024 ? 2 : 1;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * kNumSMs, grp.n / 16384));
    k_group_codes_smem<<<(int)blocks, kGcThreads, smem, s>>>(grp, gd, gcode, miss);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  k_group_codes<<<grid_for(grp.n), T, 0, s>>>(grp, gd, gcode, miss);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_join_size(const int32_t* ca, const int32_t* cb, int64_t K, unsigned long long* out,
                             cudaStream_t s, int64_t* launches) {
  if (K <= 0) return cudaSuccess;
  k_join_size<<<grid_for(K), T, 0, s>>>(ca, cb, K, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_popcount(const unsigned* w, int64_t n, unsigned mask, unsigned long long* out, cudaStream_t s,
                            int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_popcount<<<grid_for(n, T * 8), T, 0, s>>>(w, n, mask, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_max_u64(const unsigned long long* x, int64_t n, unsigned long long* out, cudaStream_t s,
                           int64_t* launches) {
  if (n <= 0) return cudaSuccess;
  k_max_u64<<<grid_for(n), T, 0, s>>>(x, n, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
