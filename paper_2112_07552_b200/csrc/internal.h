// internal.h — launchers shared between the kernel files and the host runtime.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/tcudb.h"

namespace tcudb {

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------- a6: tcgen05 GEMM
enum GemmElem { ELEM_I8 = 0, ELEM_BF16 = 1, ELEM_FP4 = 2 /* e2m1 x2 per byte, kind::mxf4, scales 1 */ };
enum GemmEpi {
  EPI_STORE32 = 0,  // C32[r][c] = acc (int32 or fp32 bits)
  EPI_SET64 = 1,    // C64[r][c] = (int64)acc << shift
  EPI_ACC64 = 2,    // C64[r][c] += (int64)acc << shift
  EPI_TRI = 3,      // *tri_out += sum acc[r][c] * mask[r][c]   (triangle epilogue, a9)
  EPI_STORE16 = 4,  // C16[r][c] = (uint16)acc — COUNT results the guard proved < 2^16 (fp4 path)
  EPI_SETF64 = 5,   // C64f[r][c] = (double)acc        (bf16: one K range of the hi/lo split)
  EPI_ACCF64 = 6    // C64f[r][c] += (double)acc       (float partials summed in fp64, DESIGN R9)
};
constexpr int kGemmBM = 128;
constexpr int kGemmBN = 256;
constexpr int kGemmBKBytes = 128;
constexpr int kGemmBNFp4 = 240;

struct GemmArgs {
  int elem = ELEM_I8;
  int a_signed = 0, b_signed = 0;
  int64_t M = 0, N = 0;           // rows of A, rows of B (multiples of 128 / 256)
  int64_t k_begin = 0, k_len = 0; // K range in elements (k_len * bytes % 128 == 0)
  const void* A = nullptr; int64_t lda = 0;  // elements
  const void* B = nullptr; int64_t ldb = 0;
  int epi = EPI_STORE32;
  void* C = nullptr; int64_t ldc = 0; int shift = 0;
  const uint8_t* mask = nullptr; int64_t ldm = 0, mask_rows = 0, mask_cols = 0;
  unsigned long long* tri_out = nullptr;
  // optional: per (row, 256-column N tile) count of nonzero results, cnt[row * ldcnt + n_tile]
  // (feeds the compaction scan, a8; only on the launch that produces the final matrix)
  int32_t* cnt_out = nullptr; int64_t ldcnt = 0;
  // optional: the optimistic fill's overflow flags (device ints). When either is set the
  // operands are not exact, the host reruns the matrix stage one type wider, and this launch
  // exits at once instead of multiplying them
  const int* abort_a = nullptr; const int* abort_b = nullptr;
  // optional (fp4 COUNT with EPI_STORE16): compaction (a8) fused into the GEMM kernel —
  // the result tuples are written in (g, h) order by compaction warps while later tiles
  // are still being multiplied (see gemm_tc.cu). Scratch arrays are zeroed by the caller.
  const void* cmp = nullptr;        // const FusedCompact* (device-visible fields by value)
  // optional block-sparse bitmaps (blocksparse.cu): per 128-row A tile / BN-row B tile, bmw
  // 64-bit words over the absolute K-blocks of the stage width; 1-CTA kernel, no cmp
  const unsigned long long* bmA = nullptr;
  const unsigned long long* bmB = nullptr;
  int bmw = 0;
};
// Fused-compaction parameters (gemm_tc.cu, EPI_STORE16 + fp4 only).
struct FusedCompact {
  int64_t G, H;                     // valid rows / columns of C
  const long long* dict_g; const long long* dict_h;
  int g_out_type, h_out_type;       // 0 I32, 1 I64
  void* out_g; void* out_h; void* out_agg;  // capacity >= nnz (agg int64)
  int32_t* tcnt;                    // [tiles_n][Mp] per-(N tile, row) counts -> offsets in the row
  int32_t* rowbase;                 // [Mp] row offset inside its 128-row M-block
  unsigned* mdone;                  // [tiles_m] epilogue-warp arrivals per M-block (zeroed)
  unsigned long long* mstate;       // [tiles_m] look-back state per M-block (zeroed)
  int64_t* total;                   // out: number of result tuples
};
cudaError_t launch_gemm(const GemmArgs& a, cudaStream_t s, int64_t* launches);

// ---------------------------------------------------------------- scan
// Exclusive prefix sum of n int64 values (in -> out, out may alias in); total in *total_dev (optional).
size_t scan_temp_bytes(int64_t n);
cudaError_t exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, int64_t* total_dev, void* temp,
                               cudaStream_t s, int64_t* launches);
cudaError_t exclusive_scan_i32(const int32_t* in, int64_t* out, int64_t n, int64_t* total_dev, void* temp,
                               cudaStream_t s, int64_t* launches);

// ---------------------------------------------------------------- radix sort (key u64, payload u32)
size_t radix_temp_bytes(int64_t n);
cudaError_t radix_sort_pairs(unsigned long long* keys, uint32_t* vals, unsigned long long* keys_alt,
                             uint32_t* vals_alt, int64_t n,
                             int bits, void* temp, cudaStream_t s, int64_t* launches, bool* result_in_alt);

// ---------------------------------------------------------------- multi-GPU (collective.cu)
struct NcclComm;
NcclComm* nccl_attach(void* comm, std::string* err);
void nccl_detach(NcclComm* c);
// local_st: this rank's own argument check (agreed on before any exchange)
tcudb_status collective_join_agg(tcudb_ctx* ctx, const NcclComm* nc, const tcudb_table* A, const tcudb_table* B,
                                 const tcudb_query* q, tcudb_status local_st, tcudb_result* out, tcudb_stats* stats,
                                 cudaStream_t s, float* ms_comm);
tcudb_status shard_agree(const int64_t* descs, int P, int64_t* agreed);
void shard_bounds(const int64_t* msgs, int P, int64_t* bounds);
// Stream-ordered scratch from the calling context's own memory pool (tcudb_create makes a
// private pool: the process's default pool and its release threshold stay the caller's).
cudaError_t pool_malloc(void** p, size_t bytes, cudaStream_t s);
// ABI entry scope: the context's device and pool for the call; the caller's current device
// is restored on exit (nested entries restore in order)
struct CtxScope {
  int prev_dev = -1;
  void* prev_pool = nullptr;
  CtxScope(int device, void* pool);
  ~CtxScope();
};
// tcudb_partition's body with the key-hash mode of the key-partitioned path (by_key: bounds
// unused, destination = hash of the join key; the group column may be absent)
tcudb_status partition_table(tcudb_ctx* ctx, const tcudb_table* in, const int64_t* bounds, int32_t P, int by_key,
                             tcudb_table* out, int64_t* counts, cudaStream_t s);
// host-runtime helpers the collective path shares (tcudb.cu)
void* internal_result_alloc(tcudb_ctx* ctx, size_t bytes, cudaStream_t s);
void internal_result_release(tcudb_ctx* ctx, void* p);
tcudb_status internal_set_err(tcudb_ctx* ctx, tcudb_status st, const char* msg);

}  // namespace tcudb
