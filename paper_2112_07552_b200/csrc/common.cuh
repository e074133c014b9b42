// common.cuh — shared device helpers for the sm_100a kernels (PTX wrappers for
// mbarrier, TMA, tcgen05/TMEM) and host-side launch bookkeeping.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <mutex>
#include <map>
#include <tuple>

#define TCUDB_DEV __device__ __forceinline__

// ------------------------------------------------------------------ basics
TCUDB_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
TCUDB_DEV int lane_id() { return threadIdx.x & 31; }
TCUDB_DEV int warp_id() { return threadIdx.x >> 5; }
TCUDB_DEV uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Column loads: keys / groups are int32 or int64 (tcudb_dtype 0 / 1).
TCUDB_DEV int64_t ld_int(const void* p, int type, int64_t i) {
  return type == 1 ? __ldg(reinterpret_cast<const long long*>(p) + i)
                   : (int64_t)__ldg(reinterpret_cast<const int*>(p) + i);
}

// 16-byte streaming load as volatile asm: a batch of these stays batched (ptxas may
// otherwise interleave each load with its consumers and serialize the latency).
TCUDB_DEV int4 ld_stream_v4(const void* p) {
  int4 v;
  asm volatile("ld.global.cs.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// ------------------------------------------------------------------ mbarrier
TCUDB_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
TCUDB_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
TCUDB_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
TCUDB_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
TCUDB_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
TCUDB_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %0;" ::"r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// ------------------------------------------------------------------ TMA
TCUDB_DEV void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}
// 2D tile load global -> shared, completion signalled on `bar` (complete_tx bytes).
TCUDB_DEV void tma_load_2d(const void* desc, void* smem_dst, uint64_t* bar, int32_t c0, int32_t c1,
                           uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(cache_hint)
      : "memory");
}
// L2 cache-policy descriptors (createpolicy)
TCUDB_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ------------------------------------------------------------------ tcgen05
TCUDB_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
TCUDB_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Allocate `ncols` TMEM columns (power of 2 >= 32); whole warp executes.
TCUDB_DEV void tmem_alloc(uint32_t* smem_result, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
TCUDB_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// D[tmem] (+)= A[smem] · B[smem]ᵀ, one elected thread issues for the CTA.
TCUDB_DEV void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
TCUDB_DEV void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier when all previously issued tcgen05.mma of this thread complete.
TCUDB_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread t of the warp gets TMEM lane (base_lane + t),
// registers r[i] = column (base_col + i).
TCUDB_DEV void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
TCUDB_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor for a K-major operand tile written by TMA with
// 128-byte swizzle: 8-row x 128-byte swizzle atoms stacked at 1024-byte stride.
//   bits  0-13 start address >> 4     bits 16-29 leading byte offset >> 4 (unused: 1)
//   bits 32-45 stride byte offset >> 4 (1024 B)   bits 46-47 version = 1 (sm_100)
//   bits 61-63 layout = 2 (SWIZZLE_128B)
TCUDB_DEV uint64_t sw128_desc(uint32_t smem_addr) {
  return (uint64_t)((smem_addr & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}

// ------------------------------------------------------------------ clusters / CTA pairs (cta_group::2)
TCUDB_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
TCUDB_DEV uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
TCUDB_DEV uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// shared::cta address -> the same variable's shared::cluster address in CTA `rank`
TCUDB_DEV uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
TCUDB_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on an mbarrier of another CTA of the cluster (address from mapa_shared)
TCUDB_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-SM TMA: data lands in this CTA's smem, completion bytes are counted on the
// pair leader's mbarrier (cluster address).
TCUDB_DEV void tma_load_2d_pair(const void* desc, void* smem_dst, uint32_t leader_bar, int32_t c0, int32_t c1,
                                uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(leader_bar), "r"(c0), "r"(c1), "l"(cache_hint)
      : "memory");
}
TCUDB_DEV void tmem_alloc_pair(uint32_t* smem_result, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_result)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
TCUDB_DEV void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
TCUDB_DEV void mma_i8_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
TCUDB_DEV void mma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit of the pair's MMAs, arriving on the mbarrier at the same smem offset in
// every CTA of `cta_mask`
TCUDB_DEV void mma_commit_pair(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
TCUDB_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ------------------------------------------------------------------ bf16 three-way split
// 8 consecutive fp32 cells -> bf16 hi / mid / lo (RNE, reading R8/R9) stored as 16-byte vectors
// into every K segment (stride seg_stride elements) by its 2-bit role (kernels.h kRoles*).
TCUDB_DEV uint16_t bf16_rn_bits(float x) {
  uint16_t b;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(b) : "f"(x));
  return b;
}
TCUDB_DEV float bf16_bits_val(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }
template <bool STREAM>
TCUDB_DEV void store_split8(uint16_t* row, int64_t seg_stride, const float* x, int roles, int nsegs) {
  uint32_t w[3][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint16_t p[3][2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float v = x[2 * j + e];
      p[0][e] = bf16_rn_bits(v);
      const float r1 = v - bf16_bits_val(p[0][e]);
      p[1][e] = bf16_rn_bits(r1);
      p[2][e] = bf16_rn_bits(r1 - bf16_bits_val(p[1][e]));
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) w[q][j] = (uint32_t)p[q][0] | ((uint32_t)p[q][1] << 16);
  }
  for (int sg = 0; sg < nsegs; ++sg) {
    const int role = (roles >> (2 * sg)) & 3;
    if (role == 3) continue;
    const uint4 v = make_uint4(w[role][0], w[role][1], w[role][2], w[role][3]);
    uint4* dst = reinterpret_cast<uint4*>(row + (int64_t)sg * seg_stride);
    if (STREAM) __stcs(dst, v);
    else *dst = v;
  }
}

// ------------------------------------------------------------------ reductions
template <typename T>
TCUDB_DEV T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
TCUDB_DEV long long warp_max_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, (long long)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
TCUDB_DEV long long warp_min_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, (long long)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// cudaFuncSetAttribute per (kernel, device, attribute), thread-safe, keeping the largest value
// requested so far (the attributes used here are upper bounds: MaxDynamicSharedMemorySize).
// The attribute is a per-device property: a process-wide "already set" flag would skip the
// second device (and race between threads); one inline function => one table per library.
inline cudaError_t set_func_attr_void(const void* f, cudaFuncAttribute attr, int value) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int>, int> cur;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaGetLastError();
  const auto key = std::make_tuple(f, dev, (int)attr);
  std::lock_guard<std::mutex> g(mu);
  auto it = cur.find(key);
  if (it != cur.end() && it->second >= value) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(f, attr, value);
  if (e == cudaSuccess) cur[key] = value;
  return e;
}
template <typename K>
inline cudaError_t set_func_attr(K* kernel, cudaFuncAttribute attr, int value) {
  return set_func_attr_void(reinterpret_cast<const void*>(kernel), attr, value);
}


