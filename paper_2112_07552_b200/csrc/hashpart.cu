// hashpart.cu — steps a2 + a7 for large hash-mode key domains: a hash-partitioned
// sparse COUNT.
//
// PAPER.md §3.1 encodes dom(ID) as matrix columns; §4.2.4
// sends low-density joins (c5: 4 M keys, density < 0.1 %) to a sparse product. With
// millions of distinct keys a global hash dictionary (hundreds of MB) and the
// per-key buckets of B are random-access structures far larger than the SM's
// caches. Here both tables are radix-partitioned on the key's hash first (two
// passes of <= 7 bits, each staged in shared memory so the writes leave as runs),
// until one partition's keys fit one CTA's shared memory. Per partition, a CTA then
//   count:  builds the partition's key dictionary (slot = code; D_p keys on both
//           sides), per-key counts cntA / cntB and J_p = sum cntA·cntB (the join
//           size for the selector, a4);
//   expand: rebuilds it, buckets B's group codes by key (counting sort in shared
//           memory) and expands every A tuple over its key's bucket with one
//           fire-and-forget reduction C[g][h] += 1 per joined pair (C: G x H u32,
//           L2-resident at c5's 4,096 x 4,096).
// The key dictionary is partition-local: a key's code is (partition, slot), a dense
// code space of size K = sum_p D_p (reading R2: codes in hash order in hash mode).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "dict.cuh"

namespace tcudb {
namespace {

constexpr int PT = 512;        // threads per partitioning block (2 CTAs per SM)
constexpr int PER = 8;         // tuples per thread and chunk
constexpr int CH = PER * PT;   // tuples per partitioning chunk
constexpr int kMaxDigits = 128;

TCUDB_DEV unsigned long long mix64(unsigned long long k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}

// chunk -> (segment, chunk in segment): chunk_start[s] = first global chunk of segment s
TCUDB_DEV int find_seg(const int64_t* __restrict__ chunk_start, int nseg, int64_t c) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (chunk_start[mid] <= c) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// one 1,024-thread block: each thread a contiguous run of segments, a block-wide scan of
// the per-thread chunk totals (a single-thread loop cost ~7 us per pass)
constexpr int kCsThreads = 1024;
__global__ void __launch_bounds__(kCsThreads) k_chunk_starts(const int64_t* __restrict__ seg_off, int nseg,
                                                            int64_t* __restrict__ chunk_start) {
  __shared__ int64_t wsum[kCsThreads / 32];
  const int per = (nseg + kCsThreads - 1) / kCsThreads;
  const int s0 = threadIdx.x * per, s1 = min(nseg, s0 + per);
  int64_t run = 0;
  for (int s = s0; s < s1; ++s) run += (seg_off[s + 1] - seg_off[s] + CH - 1) / CH;
  int64_t incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane_id() >= o) incl += t;
  }
  if (lane_id() == 31) wsum[warp_id()] = incl;
  __syncthreads();
  if (warp_id() == 0) {
    int64_t w = wsum[lane_id()], wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane_id() >= o) wi += t;
    }
    wsum[lane_id()] = wi - w;  // exclusive prefix of the warp totals
  }
  __syncthreads();
  int64_t c = wsum[warp_id()] + incl - run;
  for (int s = s0; s < s1; ++s) {
    chunk_start[s] = c;
    c += (seg_off[s + 1] - seg_off[s] + CH - 1) / CH;
  }
  if (threadIdx.x == kCsThreads - 1) chunk_start[nseg] = c;
}

struct PassIO {
  const void* raw; int raw_type; long long kmin; const int32_t* g_raw;  // pass 1 (raw key column, group codes)
  const void* v_raw; int v_type;                                        // pass 1 values (SUM)
  const unsigned long long* k_in; const int32_t* g_in;
  const long long* v_in; long long* v_out;                              // value payload (SUM)
  const int64_t* seg_off; int nseg; int shift; int bits;
  const int64_t* chunk_start;
  int32_t* counts;  // [total_chunks * R] in (segment, digit, chunk) order
  const int64_t* offs;  // exclusive scan of counts
  unsigned long long* k_out; int32_t* g_out; int64_t* seg_out;
  // atomic-reservation passes: per (segment, digit) output cursors (start offsets known from
  // the one-pass 2^pbits histogram); NULL: the per-chunk offsets of the hist + scan passes
  unsigned long long* cursor;
};

TCUDB_DEV long long load_value(const PassIO& io, int64_t i) {
  if (!io.v_out) return 0;
  if (io.raw) return io.v_raw ? ld_int(io.v_raw, io.v_type, i) : 1;
  return io.v_in[i];
}

__global__ void __launch_bounds__(PT) k_part_hist(const PassIO io) {
  __shared__ int h[kMaxDigits];
  const int64_t c = blockIdx.x;
  if (c >= io.chunk_start[io.nseg]) return;
  const int s = find_seg(io.chunk_start, io.nseg, c);
  const int64_t j = c - io.chunk_start[s];
  const int64_t nch = io.chunk_start[s + 1] - io.chunk_start[s];
  const int R = 1 << io.bits;
  for (int d = threadIdx.x; d < R; d += PT) h[d] = 0;
  __syncthreads();
  const int64_t lo = io.seg_off[s] + j * CH, hi = min(io.seg_off[s + 1], lo + CH);
  // keys only (the histogram needs no group codes); the CH / PT = 4 loads per thread
  // are issued before the shared-memory atomics
  unsigned long long k[CH / PT];
#pragma unroll
  for (int u = 0; u < CH / PT; ++u) {
    const int64_t i = lo + threadIdx.x + (int64_t)u * PT;
    k[u] = 0;
    if (i < hi)
      k[u] = io.raw ? (unsigned long long)ld_int(io.raw, io.raw_type, i) - (unsigned long long)io.kmin : io.k_in[i];
  }
#pragma unroll
  for (int u = 0; u < CH / PT; ++u)
    if (lo + threadIdx.x + (int64_t)u * PT < hi)
      atomicAdd(&h[(int)(((io.raw ? mix64(k[u]) : k[u]) >> io.shift) & (unsigned)(R - 1))], 1);
  __syncthreads();
  const int64_t base = io.chunk_start[s] * R;
  for (int d = threadIdx.x; d < R; d += PT) io.counts[base + (int64_t)d * nch + j] = h[d];
}

template <bool VAL>
__global__ void __launch_bounds__(PT, 2) k_part_scatter(const PassIO io) {  // 2,048 threads per SM
  extern __shared__ __align__(16) uint8_t stage_raw[];
  unsigned long long* sk = reinterpret_cast<unsigned long long*>(stage_raw);  // [CH]
  int32_t* sg = reinterpret_cast<int32_t*>(sk + CH);                          // [CH]
  uint8_t* sd = reinterpret_cast<uint8_t*>(sg + CH);                          // [CH] digit of each entry
  long long* sv = reinterpret_cast<long long*>(sd + CH);                       // [CH] values (SUM only)
  __shared__ int cnt[kMaxDigits], lstart[kMaxDigits];
  __shared__ int64_t gpos[kMaxDigits];
  const int64_t c = blockIdx.x;
  if (c >= io.chunk_start[io.nseg]) return;
  const int s = find_seg(io.chunk_start, io.nseg, c);
  const int64_t j = c - io.chunk_start[s];
  const int64_t nch = io.chunk_start[s + 1] - io.chunk_start[s];
  const int R = 1 << io.bits;
  const int64_t base = io.chunk_start[s] * R;
  for (int d = threadIdx.x; d < R; d += PT) {
    cnt[d] = 0;
    if (!io.cursor) gpos[d] = io.offs[base + (int64_t)d * nch + j];
  }
  __syncthreads();
  const int64_t lo = io.seg_off[s] + j * CH, hi = min(io.seg_off[s + 1], lo + CH);
  unsigned long long k[PER];
  int32_t g[PER];
  long long v[PER];
  int d[PER], r[PER];
  // the chunk's loads first (all four per thread in flight), then the digits and ranks
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int64_t i = lo + threadIdx.x + u * PT;
    k[u] = 0; g[u] = 0;
    if (i < hi) {
      if (io.raw) {
        k[u] = (unsigned long long)ld_int(io.raw, io.raw_type, i) - (unsigned long long)io.kmin;
        g[u] = __ldcs(io.g_raw + i);
      } else {
        k[u] = __ldcs(io.k_in + i);
        g[u] = __ldcs(io.g_in + i);
      }
      if (VAL) v[u] = load_value(io, i);
    }
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    d[u] = -1;
    if (lo + threadIdx.x + u * PT < hi) {
      // pass 1 replaces the key offset by its hash (a bijection: equal keys <=> equal
      // hashes), so later passes and the per-partition tables never rehash
      if (io.raw) k[u] = mix64(k[u]);
      d[u] = (int)((k[u] >> io.shift) & (unsigned)(R - 1));
      r[u] = atomicAdd(&cnt[d[u]], 1);
    }
  }
  __syncthreads();
  // atomic reservation of this chunk's run per digit (order inside a partition is free)
  if (io.cursor)
    for (int dd = threadIdx.x; dd < R; dd += PT)
      gpos[dd] = cnt[dd] ? (int64_t)atomicAdd(io.cursor + (int64_t)s * R + dd, (unsigned long long)cnt[dd]) : 0;
  if (threadIdx.x < 32) {  // exclusive scan of <= 128 digit counts, 4 per lane
    int v[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int dd = threadIdx.x * 4 + q;
      v[q] = dd < R ? cnt[dd] : 0;
      sum += v[q];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)threadIdx.x >= o) incl += t;
    }
    int run = incl - sum;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int dd = threadIdx.x * 4 + q;
      if (dd < R) lstart[dd] = run;
      run += v[q];
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < PER; ++u)
    if (d[u] >= 0) {
      const int p = lstart[d[u]] + r[u];
      sk[p] = k[u];
      sg[p] = g[u];
      sd[p] = (uint8_t)d[u];
      if (VAL) sv[p] = v[u];
    }
  __syncthreads();
  const int total = (int)(hi - lo);
  for (int p = threadIdx.x; p < total; p += PT) {
    const int a = sd[p];
    const int64_t o = gpos[a] + (p - lstart[a]);
    io.k_out[o] = sk[p];
    io.g_out[o] = sg[p];
    if (VAL) io.v_out[o] = sv[p];
  }
}

// One pass over a side's raw keys: the histogram of the full partition index (the top
// pbits of the key hash, both radix digits at once) — every segment and partition start is
// known before the first scatter, which then reserves its runs with one atomic per digit
// (no per-pass histogram / count-scan passes). Persistent CTAs, shared-memory bins.
constexpr int HT = 1024;
__global__ void __launch_bounds__(HT) k_part_hist_all(const void* __restrict__ raw, int raw_type, long long kmin,
                                                      int64_t n, int pbits, unsigned* __restrict__ hist) {
  extern __shared__ unsigned bins[];
  const int P = 1 << pbits;
  for (int i = threadIdx.x; i < P; i += HT) bins[i] = 0u;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * HT;
  constexpr int U = 4;
  for (int64_t i0 = (int64_t)blockIdx.x * HT + threadIdx.x; i0 < n; i0 += U * stride) {
    unsigned long long k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      k[u] = i < n ? (unsigned long long)ld_int(raw, raw_type, i) - (unsigned long long)kmin : 0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) atomicAdd(&bins[(int)(mix64(k[u]) >> (64 - pbits))], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < P; i += HT)
    if (bins[i]) atomicAdd(hist + i, bins[i]);
}

// new segment offsets: seg_out[s * R + d] = start of digit d of segment s (empty segments
// start where they are); seg_out[nseg * R] = end
__global__ void k_seg_out(const PassIO io) {
  const int R = 1 << io.bits;
  const int64_t total = (int64_t)io.nseg * R;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x <= total; x += (int64_t)gridDim.x * blockDim.x) {
    if (x == total) { io.seg_out[x] = io.seg_off[io.nseg]; continue; }
    const int s = (int)(x / R), d = (int)(x - (int64_t)s * R);
    const int64_t nch = io.chunk_start[s + 1] - io.chunk_start[s];
    io.seg_out[x] = nch ? io.offs[io.chunk_start[s] * R + (int64_t)d * nch] : io.seg_off[s];
  }
}

// ---- per-partition kernels: open-addressing table of TS slots in shared memory
constexpr int QT = 256;   // count kernel threads
constexpr int QTE = 512;  // expand kernel threads

TCUDB_DEV int slot_of(unsigned long long k, int ts_bits) {
  return (int)((k * 0x9E3779B97F4A7C15ull) >> (64 - ts_bits));
}

// insert (or find) k; returns its slot
TCUDB_DEV int tab_insert(unsigned long long* keys, int mask, int ts_bits, unsigned long long k) {
  int h = slot_of(k, ts_bits);
  while (true) {
    const unsigned long long cur = keys[h];
    if (cur == k) return h;
    if (cur == ~0ull) {
      const unsigned long long prev = atomicCAS(keys + h, ~0ull, k);
      if (prev == ~0ull || prev == k) return h;
    }
    h = (h + 1) & mask;
  }
}

TCUDB_DEV int tab_find(const unsigned long long* keys, int mask, int ts_bits, unsigned long long k) {
  int h = slot_of(k, ts_bits);
  while (true) {
    const unsigned long long cur = keys[h];
    if (cur == k) return h;
    if (cur == ~0ull) return -1;
    h = (h + 1) & mask;
  }
}

__global__ void __launch_bounds__(QT) k_part_count(const unsigned long long* __restrict__ ka,
                                                   const int64_t* __restrict__ offa,
                                                   const unsigned long long* __restrict__ kb,
                                                   const int64_t* __restrict__ offb, int ts_bits, int stride,
                                                   unsigned long long* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int TS = 1 << ts_bits, mask = TS - 1;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
  int* ca = reinterpret_cast<int*>(keys + TS);
  int* cb = ca + TS;
  for (int i = threadIdx.x; i < TS; i += QT) { keys[i] = ~0ull; ca[i] = 0; cb[i] = 0; }
  __syncthreads();
  const int p = blockIdx.x * stride;  // stride > 1: a sample of the partitions (the selector's estimate)
  // 4 key loads in flight per thread ahead of the shared-memory probes
  constexpr int NU = 4;
  for (int64_t i0 = offb[p] + threadIdx.x, e = offb[p + 1]; i0 < e; i0 += NU * QT) {
    unsigned long long k[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) k[u] = i0 + u * QT < e ? __ldcs(kb + i0 + u * QT) : 0ull;
#pragma unroll
    for (int u = 0; u < NU; ++u)
      if (i0 + u * QT < e) atomicAdd(cb + tab_insert(keys, mask, ts_bits, k[u]), 1);
  }
  __syncthreads();
  for (int64_t i0 = offa[p] + threadIdx.x, e = offa[p + 1]; i0 < e; i0 += NU * QT) {
    unsigned long long k[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) k[u] = i0 + u * QT < e ? __ldcs(ka + i0 + u * QT) : 0ull;
#pragma unroll
    for (int u = 0; u < NU; ++u)
      if (i0 + u * QT < e) {
        const int h = tab_find(keys, mask, ts_bits, k[u]);
        if (h >= 0) atomicAdd(ca + h, 1);
      }
  }
  __syncthreads();
  unsigned long long J = 0, D = 0, M = 0, U = 0;
  for (int i = threadIdx.x; i < TS; i += QT) {
    J += (unsigned long long)ca[i] * (unsigned long long)cb[i];
    D += (ca[i] > 0 && cb[i] > 0);
    M += cb[i] > 0 ? (unsigned long long)ca[i] : 0ull;
    U += cb[i] > 0;
  }
  // per-partition totals (summed by k_part_sum: same-address atomics from every warp of
  // 16 K CTAs would serialize in L2)
  __shared__ unsigned long long red[4][QT / 32];
  J = warp_sum(J); D = warp_sum(D); M = warp_sum(M); U = warp_sum(U);
  if (lane_id() == 0) { red[0][warp_id()] = J; red[1][warp_id()] = D; red[2][warp_id()] = M; red[3][warp_id()] = U; }
  __syncthreads();
  if (threadIdx.x < 4) {
    unsigned long long t = 0;
    for (int w = 0; w < QT / 32; ++w) t += red[threadIdx.x][w];
    out[(int64_t)blockIdx.x * 4 + threadIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_part_sum(const unsigned long long* __restrict__ per, int P,
                                                   unsigned long long* __restrict__ out) {
  __shared__ unsigned long long red[4][32];
  unsigned long long t[4] = {0, 0, 0, 0};
  for (int p = threadIdx.x; p < P; p += blockDim.x)
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] += per[(int64_t)p * 4 + q];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    t[q] = warp_sum(t[q]);
    if (lane_id() == 0) red[q][warp_id()] = t[q];
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    unsigned long long x = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) x += red[threadIdx.x][w];
    out[threadIdx.x] = x;
  }
}

// C += x as a fire-and-forget L2 reduction whose line is kept resident (evict_last): the
// streaming partition reads would otherwise evict C's lines between reductions, and every
// eviction is a DRAM write-back (ncu r01 v10: 0.78 GB written per c5 launch for a 67 MB C).
TCUDB_DEV unsigned long long l2_keep_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
TCUDB_DEV void red_keep(unsigned* p, unsigned x, unsigned long long pol) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u32 [%0], %1, %2;" :: "l"(p), "r"(x), "l"(pol) : "memory");
}
TCUDB_DEV void red_keep(unsigned long long* p, unsigned long long x, unsigned long long pol) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.u64 [%0], %1, %2;" :: "l"(p), "l"(x), "l"(pol) : "memory");
}

template <bool SUM>
__global__ void __launch_bounds__(QTE) k_part_expand(const unsigned long long* __restrict__ ka,
                                                    const int32_t* __restrict__ ga,
                                                    const int64_t* __restrict__ offa,
                                                    const unsigned long long* __restrict__ kb,
                                                    const int32_t* __restrict__ hb,
                                                    const int64_t* __restrict__ offb, int ts_bits, int cap,
                                                    unsigned* __restrict__ C, int64_t ldc,
                                                    const long long* __restrict__ va,
                                                    const long long* __restrict__ vb,
                                                    unsigned long long* __restrict__ C64,
                                                    unsigned long long* __restrict__ jk) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int wsum[QTE / 32];
  __shared__ unsigned long long jred[QTE / 32];
  __shared__ int kred;
  const int TS = 1 << ts_bits, mask = TS - 1;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem);
  int* cnt = reinterpret_cast<int*>(keys + TS);   // per slot: B tuples, then the bucket cursor
  int* start = cnt + TS;                          // per slot: bucket start
  int* bslot = start + TS;                        // per B tuple of the partition: its slot
  int* bh = bslot + cap;                          // B group codes bucketed by slot
  long long* bw = reinterpret_cast<long long*>(smem + (size_t)TS * 16 + (size_t)cap * 8);  // SUM: B values, bucketed
  unsigned* hit = reinterpret_cast<unsigned*>(smem + (size_t)TS * 16 + (size_t)cap * (SUM ? 16 : 8));  // [TS / 32]
  for (int i = threadIdx.x; i < TS; i += QTE) { keys[i] = ~0ull; cnt[i] = 0; }
  for (int i = threadIdx.x; i < TS / 32; i += QTE) hit[i] = 0;
  if (threadIdx.x == 0) kred = 0;
  __syncthreads();
  const int p = blockIdx.x;
  const int64_t b0 = offb[p];
  const int nb = (int)(offb[p + 1] - b0);
  for (int i = threadIdx.x; i < nb; i += QTE) {
    const int h = tab_insert(keys, mask, ts_bits, __ldcs(kb + b0 + i));
    bslot[i] = h;
    atomicAdd(cnt + h, 1);
  }
  __syncthreads();
  // exclusive scan of cnt[0..TS) -> start (each thread a contiguous run of TS / QTE slots)
  {
    const int per = TS / QTE;
    const int s0 = threadIdx.x * per;
    int run = 0;
    for (int q = 0; q < per; ++q) run += cnt[s0 + q];
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane_id() >= o) incl += t;
    }
    if (lane_id() == 31) wsum[warp_id()] = incl;
    __syncthreads();
    int wbase = 0;
    for (int w = 0; w < warp_id(); ++w) wbase += wsum[w];
    int x = wbase + incl - run;
    for (int q = 0; q < per; ++q) { start[s0 + q] = x; x += cnt[s0 + q]; cnt[s0 + q] = 0; }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += QTE) {
    const int h = bslot[i];
    const int pos = start[h] + atomicAdd(cnt + h, 1);
    bh[pos] = __ldcs(hb + b0 + i);
    if (SUM) bw[pos] = __ldcs(vb + b0 + i);
  }
  __syncthreads();
  const unsigned long long pol = l2_keep_policy();
  unsigned long long jp = 0;  // this thread's joined pairs (the exact J_p of the partition)
  constexpr int U = 4;  // A keys and group codes loaded ahead of the probes
  const int64_t ea = offa[p + 1];
  for (int64_t i0 = offa[p] + threadIdx.x; i0 < ea; i0 += U * QTE) {
   unsigned long long kk[U];
   int32_t gg[U];
#pragma unroll
   for (int u = 0; u < U; ++u) {
     const int64_t i = i0 + u * QTE;
     kk[u] = i < ea ? __ldcs(ka + i) : 0ull;
     gg[u] = i < ea ? __ldcs(ga + i) : 0;
   }
#pragma unroll
   for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + u * QTE;
    if (i >= ea) continue;
    const int h = tab_find(keys, mask, ts_bits, kk[u]);
    if (h < 0) continue;
    const int n = cnt[h];
    if (n == 0) continue;
    jp += (unsigned long long)n;
    if (!(hit[h >> 5] & (1u << (h & 31)))) atomicOr(hit + (h >> 5), 1u << (h & 31));
    const int64_t r = (int64_t)gg[u] * ldc;
    unsigned* row = C + r;
    const int e0 = start[h];
    if (SUM) {
      // integer SUM: wrapping products and sums (exact whenever the result fits int64; the
      // caller has checked J·max|v|·max|w|), plus the COUNT plane for existence (R3)
      const unsigned long long v = (unsigned long long)__ldcs(va + i);
      unsigned long long* row64 = C64 + r;
      for (int e = 0; e < n; ++e) {
        red_keep(row64 + bh[e0 + e], v * (unsigned long long)bw[e0 + e], pol);
        red_keep(row + bh[e0 + e], 1u, pol);
      }
    } else {
      for (int e = 0; e < n; ++e) red_keep(row + bh[e0 + e], 1u, pol);
    }
   }
  }
  // J_p and K_p (keys with a B bucket and at least one A tuple) for the stats and guards
  jp = warp_sum(jp);
  if (lane_id() == 0) jred[warp_id()] = jp;
  __syncthreads();
  int kc = 0;
  for (int i = threadIdx.x; i < TS / 32; i += QTE) kc += __popc(hit[i]);
  kc = warp_sum(kc);
  if (lane_id() == 0 && kc) atomicAdd(&kred, kc);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < QTE / 32; ++w) t += jred[w];
    jk[(int64_t)p * 4 + 0] = t;
    jk[(int64_t)p * 4 + 1] = (unsigned long long)kred;
    jk[(int64_t)p * 4 + 2] = 0;
    jk[(int64_t)p * 4 + 3] = 0;
  }
}

__global__ void k_part_max(const int64_t* __restrict__ offa, const int64_t* __restrict__ offb, int P,
                           unsigned long long* __restrict__ out) {
  unsigned long long m = 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)max(offa[p + 1] - offa[p], offb[p + 1] - offb[p]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0 && m) atomicMax(out, m);
}

}  // namespace

static int64_t max_chunks(int64_t n, int nseg) { return (n + CH - 1) / CH + nseg; }

size_t hashpart_temp_bytes(int64_t n, int nseg, int bits) {
  const int64_t cnts = max_chunks(n, nseg) * (1ll << bits);
  return ((size_t)(nseg + 1) * 8 + 255) / 256 * 256 + ((size_t)cnts * 4 + 255) / 256 * 256 +
         ((size_t)(cnts + 1) * 8 + 255) / 256 * 256 + scan_temp_bytes(cnts);
}

cudaError_t launch_part_pass(const ColDesc* raw, long long kmin, const int32_t* g_raw,
                             const unsigned long long* k_in, const int32_t* g_in, const int64_t* seg_off, int nseg,
                             int64_t n, int shift, int bits, unsigned long long* k_out, int32_t* g_out,
                             int64_t* seg_out, void* temp, cudaStream_t s, int64_t* launches,
                             const ColDesc* v_raw, const long long* v_in, long long* v_out) {
  if (bits < 1 || bits > 7 || n <= 0) return cudaErrorInvalidValue;
  const int R = 1 << bits;
  const int64_t chunks = max_chunks(n, nseg);
  const int64_t cnts = chunks * R;
  char* t = static_cast<char*>(temp);
  int64_t* chunk_start = reinterpret_cast<int64_t*>(t);
  t += ((size_t)(nseg + 1) * 8 + 255) / 256 * 256;
  int32_t* counts = reinterpret_cast<int32_t*>(t);
  t += ((size_t)cnts * 4 + 255) / 256 * 256;
  int64_t* offs = reinterpret_cast<int64_t*>(t);
  t += ((size_t)(cnts + 1) * 8 + 255) / 256 * 256;
  PassIO io{};
  io.raw = raw ? raw->data : nullptr; io.raw_type = raw ? raw->type : 0; io.kmin = kmin; io.g_raw = g_raw;
  io.k_in = k_in; io.g_in = g_in; io.seg_off = seg_off; io.nseg = nseg; io.shift = shift; io.bits = bits;
  io.chunk_start = chunk_start; io.counts = counts; io.offs = offs;
  io.k_out = k_out; io.g_out = g_out; io.seg_out = seg_out;
  io.v_raw = v_raw ? v_raw->data : nullptr; io.v_type = v_raw ? v_raw->type : 0;
  io.v_in = v_in; io.v_out = v_out;
  k_chunk_starts<<<1, kCsThreads, 0, s>>>(seg_off, nseg, chunk_start);
  // unused count slots (chunks past the real total) must scan as zero
  cudaError_t e = cudaMemsetAsync(counts, 0, (size_t)cnts * 4, s);
  if (e != cudaSuccess) return e;
  k_part_hist<<<(unsigned)chunks, PT, 0, s>>>(io);
  e = exclusive_scan_i32(counts, offs, cnts, nullptr, t, s, launches);
  if (e != cudaSuccess) return e;
  // staging per tuple: key 8 + group 4 + digit 1 (+ value 8 for SUM)
  e = set_func_attr(k_part_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * 21);
  if (e != cudaSuccess) return e;
  e = set_func_attr(k_part_scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * 13);
  if (e != cudaSuccess) return e;
  if (v_out) k_part_scatter<true><<<(unsigned)chunks, PT, CH * 21, s>>>(io);
  else k_part_scatter<false><<<(unsigned)chunks, PT, CH * 13, s>>>(io);
  const int64_t so = (int64_t)nseg * R + 1;
  k_seg_out<<<(unsigned)std::min<int64_t>((so + 255) / 256, 1024), 256, 0, s>>>(io);
  if (launches) *launches += 4;
  return cudaGetLastError();
}

cudaError_t launch_part_hist_all(const ColDesc& raw, long long kmin, int pbits, unsigned* hist, cudaStream_t s,
                                 int64_t* launches) {
  if (raw.n <= 0) return cudaSuccess;
  const size_t smem = sizeof(unsigned) << pbits;
  cudaError_t e = set_func_attr(k_part_hist_all, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t blocks = std::min<int64_t>(2 * kNumSMs, (raw.n + HT * 16 - 1) / (HT * 16));
  k_part_hist_all<<<(unsigned)std::max<int64_t>(blocks, 1), HT, smem, s>>>(raw.data, raw.type, kmin, raw.n, pbits,
                                                                           hist);
  if (launches) ++*launches;
  return cudaGetLastError();
}

size_t hashpart_atomic_temp_bytes(int nseg) { return ((size_t)(nseg + 1) * 8 + 255) / 256 * 256; }

cudaError_t launch_part_pass_atomic(const ColDesc* raw, long long kmin, const int32_t* g_raw,
                                    const unsigned long long* k_in, const int32_t* g_in, const int64_t* seg_off,
                                    int nseg, int64_t n, int shift, int bits, unsigned long long* cursor,
                                    unsigned long long* k_out, int32_t* g_out, void* temp, cudaStream_t s,
                                    int64_t* launches, const ColDesc* v_raw, const long long* v_in,
                                    long long* v_out) {
  if (bits < 1 || bits > 7 || n <= 0) return cudaErrorInvalidValue;
  const int64_t chunks = max_chunks(n, nseg);
  int64_t* chunk_start = static_cast<int64_t*>(temp);
  PassIO io{};
  io.raw = raw ? raw->data : nullptr; io.raw_type = raw ? raw->type : 0; io.kmin = kmin; io.g_raw = g_raw;
  io.k_in = k_in; io.g_in = g_in; io.seg_off = seg_off; io.nseg = nseg; io.shift = shift; io.bits = bits;
  io.chunk_start = chunk_start; io.cursor = cursor;
  io.k_out = k_out; io.g_out = g_out;
  io.v_raw = v_raw ? v_raw->data : nullptr; io.v_type = v_raw ? v_raw->type : 0;
  io.v_in = v_in; io.v_out = v_out;
  k_chunk_starts<<<1, kCsThreads, 0, s>>>(seg_off, nseg, chunk_start);
  cudaError_t e = set_func_attr(k_part_scatter<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * 21);
  if (e != cudaSuccess) return e;
  e = set_func_attr(k_part_scatter<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * 13);
  if (e != cudaSuccess) return e;
  if (v_out) k_part_scatter<true><<<(unsigned)chunks, PT, CH * 21, s>>>(io);
  else k_part_scatter<false><<<(unsigned)chunks, PT, CH * 13, s>>>(io);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

// table slots: the next power of two >= 1.5 x the largest partition (load <= 2/3 for
// linear probing), at least 2 K; smaller tables = more CTAs per SM for these latency-bound
// per-partition kernels
static int ts_bits_for(int cap) {
  int b = 11;
  while ((1 << b) < cap + cap / 2) ++b;
  return b;
}

cudaError_t launch_part_count(const unsigned long long* ka, const int64_t* offa, const unsigned long long* kb,
                              const int64_t* offb, int P, int cap, unsigned long long* out, cudaStream_t s,
                              int64_t* launches, int stride) {
  const int tb = ts_bits_for(cap);
  const size_t smem = (size_t)(1 << tb) * 16;
  set_func_attr(k_part_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  // per-partition totals in out[4 ..), their sums in out[0..4)
  const int np = (P + stride - 1) / stride;
  k_part_count<<<np, QT, smem, s>>>(ka, offa, kb, offb, tb, stride, out + 4);
  k_part_sum<<<1, 1024, 0, s>>>(out + 4, np, out);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

size_t part_expand_smem(int cap, bool sum) {
  return (size_t)(1 << ts_bits_for(cap)) * 16 + (size_t)cap * (sum ? 16 : 8) + (size_t)(1 << ts_bits_for(cap)) / 8;
}

cudaError_t launch_part_expand(const unsigned long long* ka, const int32_t* ga, const int64_t* offa,
                               const unsigned long long* kb, const int32_t* hb, const int64_t* offb, int P, int cap,
                               unsigned* C, int64_t ldc, cudaStream_t s, int64_t* launches, const long long* va,
                               const long long* vb, unsigned long long* C64, unsigned long long* jk) {
  const int tb = ts_bits_for(cap);
  const size_t smem = part_expand_smem(cap, C64 != nullptr);
  set_func_attr(k_part_expand<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 186 * 1024);
  set_func_attr(k_part_expand<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 186 * 1024);
  if (smem > 186 * 1024) return cudaErrorInvalidValue;
  // jk: 4 + 4 P entries (per-partition J_p, K_p after the 4 totals, summed below)
  if (C64) k_part_expand<true><<<P, QTE, smem, s>>>(ka, ga, offa, kb, hb, offb, tb, cap, C, ldc, va, vb, C64, jk + 4);
  else k_part_expand<false><<<P, QTE, smem, s>>>(ka, ga, offa, kb, hb, offb, tb, cap, C, ldc, va, vb, C64, jk + 4);
  k_part_sum<<<1, 1024, 0, s>>>(jk + 4, P, jk);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_part_max(const int64_t* offa, const int64_t* offb, int P, unsigned long long* out, cudaStream_t s,
                            int64_t* launches) {
  k_part_max<<<(P + 255) / 256, 256, 0, s>>>(offa, offb, P, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace tcudb
