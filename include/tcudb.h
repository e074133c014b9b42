/* tcudb.h — C ABI of the B200-native TCUDB join + group-by hot path.
 *
 * The operation (Fig. 4; §3.1; §3.3):
 *
 *     SELECT A.g, B.h, SUM(A.v * B.w)        -- or COUNT(*)
 *     FROM A JOIN B ON A.k = B.k
 *     GROUP BY A.g, B.h
 *
 * evaluated as C = A_op · B_opᵀ on the sm_100a tensor cores, where A_op[g][k]
 * aggregates A's tuples of group g and join key k (the "adjacency over value
 * domains" form, with the 1^{1×n} reduction of P:808-810 folded into
 * the fill) and B_op likewise. The result is the list of (g, h, agg) for every
 * group with at least one joined pair (existence = COUNT > 0; R3),
 * sorted ascending by (g, h) (the ORDER BY-for-free reading of §3.4).
 *
 * Everything here is plain C: pointers, sizes, status codes. No torch types.
 * All column/result pointers are DEVICE pointers on the context's device unless
 * the entry point says HOST. The stream argument is a cudaStream_t passed as
 * void* (NULL = the legacy default stream).
 */
#ifndef TCUDB_H_
#define TCUDB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. On any error the result is empty (n = 0, NULL pointers): there
 * are never partial results. E_CUDA is sticky: destroy the context. */
typedef enum {
  TCUDB_OK = 0,
  TCUDB_E_INVALID = -1,     /* NULL / negative / mismatched arguments */
  TCUDB_E_UNSUPPORTED = -2, /* float keys or groups, mixed int/float values, key span of 2^64 */
  TCUDB_E_PRECISION = -3,   /* reserved: no exact or toleranced plan exists */
  TCUDB_E_OVERFLOW = -4,    /* the precision guard proves an int64 result could overflow */
  TCUDB_E_NOMEM = -5,       /* device memory for operands / C / result exhausted */
  TCUDB_E_CUDA = -6,        /* CUDA runtime / launch error (sticky) */
  TCUDB_E_COMM = -7         /* collective path: NCCL / exchange failure */
} tcudb_status;

typedef enum { TCUDB_I32 = 0, TCUDB_I64 = 1, TCUDB_F32 = 2, TCUDB_F64 = 3 } tcudb_dtype;
/* COUNT(*), SUM(A.v * B.w), AVG(A.v * B.w) = SUM / COUNT (§3.3). */
typedef enum { TCUDB_COUNT = 0, TCUDB_SUM = 1, TCUDB_AVG = 2 } tcudb_agg;

/* One column: data == NULL means "absent". A value column that is absent means
 * the factor 1 (so SUM with both values absent equals COUNT). */
typedef struct {
  const void* data;
  int32_t type; /* tcudb_dtype. Keys/groups: I32 or I64. Values: I32, I64 or F32. */
} tcudb_col;

/* A table in column-store layout: n_rows entries per column. */
typedef struct {
  int64_t n_rows;
  tcudb_col key;   /* join key k (required) */
  tcudb_col group; /* group key: A.g or B.h. Absent (data == NULL): this side is not
                      grouped — GROUP BY B.h only is Q3, no GROUP BY at all is
                      Q4 — and the result's g (or h) array is NULL. */
  tcudb_col value; /* A.v or B.w (optional) */
} tcudb_table;

/* Query flags (default 0: selector chooses the path, results sorted by (g,h)). */
enum {
  TCUDB_FORCE_DENSE = 1u << 0,  /* tensor-core GEMM path (a5, a6) */
  TCUDB_FORCE_SPARSE = 1u << 1, /* sparse-operand expand path (a7) */
  TCUDB_GATHER_NONE = 1u << 2,  /* collective calls: return this rank's shard of the result */
  TCUDB_UNORDERED = 1u << 3,    /* reserved: output order unspecified */
  TCUDB_FORCE_WIDE = 1u << 4,   /* test hook: skip the packed fp4/u8 COUNT fills, use the
                                   int64 scratch + digit-plane guard path */
  TCUDB_NO_FP4 = 1u << 5,       /* COUNT: do not use e2m1 (fp4) 0/1 operands (kind::mxf4);
                                   use u8 operands (kind::i8) */
  TCUDB_KEY_PARTITIONED = 1u << 6, /* collective calls, COUNT / integer SUM with both sides grouped:
                                      the key-partitioned path (both sides routed by a hash of the
                                      join key, partial groups merged by g range; §8(f) f4). Default
                                      when B has >= 4 M rows in total. */
  TCUDB_ROW_SHARDED = 1u << 7   /* collective calls: always the row-sharded path (north star) */
};

typedef struct {
  int32_t agg;    /* tcudb_agg */
  uint32_t flags; /* TCUDB_* flags above */
} tcudb_query;

/* Result tuples (SoA). g has A.group's type, h has B.group's type, agg is I64
 * for COUNT and integer SUM, F64 for float SUM. Owned by the caller; release
 * with tcudb_result_free (device) — or tcudb_result_free_host for results of
 * tcudb_join_agg_host. Device results are ONE allocation (one allocator callback)
 * with g at its base and h, agg at 256-byte aligned offsets: free through g only. */
typedef struct {
  int64_t n;
  void* g;
  void* h;
  void* agg;
  int32_t g_type, h_type, agg_type;
  int32_t on_host; /* 1 if the arrays are pinned host memory */
  void* base;      /* device results: the single allocation (g, unless g is absent) */
} tcudb_result;

/* Plan and stage breakdown of one query (cf. SPEC ExecutionReport S:502-505 and
 * the paper's stage breakdowns P:1531-1546). Times are CUDA-event milliseconds
 * on the query stream; ms_total is host wall clock of the whole call. */
typedef struct {
  int32_t path;       /* 0 dense (tensor cores), 1 sparse expand */
  int32_t elem;       /* dense operand type: 0 u8/s8 (kind::i8), 1 bf16, 2 bf16 hi/mid/lo split (6 products),
                         3 e2m1 0/1 COUNT operands (kind::mxf4, unit scales) */
  int32_t planes_a;   /* base-256 digit planes of A_op (int SUM) */
  int32_t planes_b;
  int32_t existence;  /* 0: existence from C itself, 1: separate COUNT plane */
  int32_t kchunks;    /* K chunks accumulated in int64 (1 = single int32 pass) */
  int32_t key_mode;   /* 0 direct-offset dictionary, 1 hash dictionary (join key), 2 direct-offset with
                         the codes looked up inside the fused dense fill (no per-tuple code columns) */
  int32_t n_launches; /* kernels launched by this call */
  int64_t G, H, K, K_union, join_pairs, n_result;
  double density_union; /* nnz cells / (G * K_union): the paper's density */
  double gemm_ops;      /* 2 * Gp * Hp * Kp summed over GEMM launches (dense path) */
  float ms_stats, ms_encode, ms_fill, ms_gemm, ms_sparse, ms_compact, ms_total;
  int32_t spa_mode;     /* sparse path: 0 C matrix (or dense path), 1 count + write passes,
                           2 count pass + persistent band writer, 3 one persistent pass,
                           4 hash-partitioned, 5 hub-band count pass + one persistent pass */
  int64_t spa_max_band; /* sparse path: most updates of one band of result rows */
  int32_t fused_compact; /* dense path: 1 if the compaction ran inside the GEMM kernel */
  float ms_kernel;       /* sparse path: CUDA-event time of the band kernel (k_spa_fused) */
  double kernel_bytes;   /* ... and its algorithmic bytes (4 J + 20 n_active + result bytes) */
  float ms_comm;         /* collective calls: host wall time of the exchanges (NCCL + routing) */
  double block_active;   /* dense path, block-sparse GEMM (§8(f) f4): share of (tile, K-block)
                            products with tuples on both sides (the rest skipped); 0: dense GEMM */
  int64_t spa_hubs;      /* sparse path, hybrid one-pass schedule: bands counted ahead (hubs) */
} tcudb_stats;

typedef struct tcudb_ctx tcudb_ctx;

/* Optional stream-ordered allocator callbacks for RESULT arrays (e.g. a caching
 * allocator). NULL: the library uses cudaMallocAsync from its own pool. */
typedef void* (*tcudb_alloc_fn)(size_t bytes, void* stream, void* user);
typedef void (*tcudb_free_fn)(void* ptr, void* stream, void* user);

/* Create a context on `device`. nccl_comm: NULL, or an ncclComm_t (one rank per
 * GPU; owned by the caller, e.g. torch's ProcessGroupNCCL communicator) — then every
 * tcudb_join_agg / tcudb_join_agg_host on this context is COLLECTIVE (SURVEY §8(b)
 * "Multi-GPU", §8(e)): each rank passes its local slices of A and B; output rows are
 * sharded by ranges of the grouped side's group key (A.g; B.h for GROUP BY B.h only),
 * that side's rows are routed to their owners (all-to-all-v), the other side is
 * allgathered, each rank runs the local query, and the result is allgathered in rank
 * order — on every rank identical to the single-GPU result — or, with
 * TCUDB_GATHER_NONE, left as the rank's (g, h)-sorted shard. Ranges are balanced on the
 * routed side's rows (weighted quantiles of an allgathered sample, tcudb_shard_bounds).
 * Without GROUP BY (Q4) the per-rank partial aggregates are allgathered and combined
 * exactly (an int64 total overflow is E_OVERFLOW). The ranks first agree on the query
 * shape (tcudb_shard_agree): a rank with an empty slice may pass NULL columns; argument
 * errors and every later local failure are agreed on (the same status on every rank, no
 * rank left waiting in a collective). NCCL (libnccl.so.2, the process's own; or the
 * library named by the environment variable TCUDB_NCCL_LIB) is resolved here with
 * dlopen. Exchange failures: E_COMM.
 * Returns E_CUDA if the device is not sm_100 or the CUDA runtime fails, E_COMM if
 * the communicator is unusable. */
tcudb_status tcudb_create(tcudb_ctx** out, int device, void* nccl_comm, tcudb_alloc_fn alloc_fn,
                          tcudb_free_fn free_fn, void* user);

/* The join + group-by query. A, B: device columns, read-only,
 * any alignment. On success *out holds device arrays (caller owns). Blocks the
 * host on at most 4 small device->host reads (statistics, sizes, join size,
 * nnz); results are valid once `stream` passes the call: without `stats` the call
 * returns while the result write is still running on `stream` (with `stats`, and on
 * the collective path, it returns after it; asynchronous kernel faults surface on a
 * later call as E_CUDA). One query in flight per context. `stats` may be NULL. */
tcudb_status tcudb_join_agg(tcudb_ctx* ctx, const tcudb_table* A, const tcudb_table* B,
                            const tcudb_query* q, tcudb_result* out, tcudb_stats* stats, void* stream);

/* Same query with HOST columns: copies the columns host->device (pinned or
 * pageable), runs tcudb_join_agg and copies the result tuples back into pinned
 * host arrays (out->on_host = 1; release with tcudb_result_free_host). */
tcudb_status tcudb_join_agg_host(tcudb_ctx* ctx, const tcudb_table* A, const tcudb_table* B,
                                 const tcudb_query* q, tcudb_result* out, tcudb_stats* stats, void* stream);

/* Chain (3-way) join, §3.2 multi-way joins:
 *
 *     SELECT A.g, C.h, COUNT(*) | SUM(A.v * B.w * C.x)
 *     FROM A, B, C WHERE A.k = B.key AND B.group = C.k
 *     GROUP BY A.g, C.h
 *
 * B.key is B's first join attribute (ID_1), B.group its second (ID_2); B is
 * projected out (the "chain exception"). Evaluated in the paper's join
 * order A -> B -> C: T = (A ⋈ B) grouped by (A.g, B.ID_2) — the nonzero()
 * re-encoding of mat(A)·mat(B)ᵀ into tuples, kept on the device — then
 * T ⋈ C on ID_2 with SUM(T.agg · C.x). agg: COUNT or integer SUM (float values:
 * E_UNSUPPORTED; the intermediate SUM would need fp64 columns). Result as for
 * tcudb_join_agg: g has A.group's type, h has C.group's type, agg I64, sorted by
 * (g, h); groups of A or C may not be absent. Errors as tcudb_join_agg. */
tcudb_status tcudb_chain_join_agg(tcudb_ctx* ctx, const tcudb_table* A, const tcudb_table* B,
                                  const tcudb_table* C, const tcudb_query* q, tcudb_result* out,
                                  tcudb_stats* stats, void* stream);

/* Triangle count of the simple undirected graph of an edge list (self-loops
 * dropped, duplicates and direction ignored): T = trace(A³)/6 over the
 * symmetrised 0/1 adjacency A, evaluated as the 2-hop GEMM A·A with an epilogue
 * that multiplies each accumulator tile by the matching A tile and reduces to
 * one int64 (§3.2 chain exception P:751-756). src/dst:
 * device I32 or I64 columns of n_edges entries. */
tcudb_status tcudb_triangle_count(tcudb_ctx* ctx, int64_t n_edges, const void* src, const void* dst,
                                  int32_t id_type, int64_t* triangles_out, tcudb_stats* stats, void* stream);

/* Step a6 on its own (for kernel tests and calibration): C[M][N] = A[M][K]·B[N][K]ᵀ
 * with K-major device operands. elem 0: int8 (a_signed/b_signed select s8 vs
 * u8), C int32; elem 1: bf16, C fp32. Requirements: M % 128 == 0,
 * N % 256 == 0, K*elem_bytes % 128 == 0, row strides lda/ldb/ldc in elements
 * with lda*elem_bytes % 16 == 0, 16-byte aligned base pointers.
 * elem 2: e2m1 (fp4) packed two per byte (kind::mxf4 with unit block scales), for
 * integer-valued operands: K, lda, ldb count ELEMENTS (K % 256 == 0, lda/ldb even),
 * N % 240 == 0, C int32 = the fp32 accumulator rounded to nearest. */
tcudb_status tcudb_gemm(tcudb_ctx* ctx, int32_t elem, int32_t a_signed, int32_t b_signed, int64_t M, int64_t N,
                        int64_t K, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                        void* stream);

/* Multi-GPU row sharding helpers (output rows are sharded by A's
 * group-key range; the exchange itself is NCCL through torch.distributed).
 *
 * tcudb_minmax: min / max of one device int column (I32 / I64) into host *mn, *mx
 * (n == 0 leaves INT64_MAX / INT64_MIN). Blocks on one small device->host read.
 *
 * tcudb_partition: route the rows of a device table by its GROUP column into P
 * destination ranges, dest(row) = #{ i < P-1 : bounds[i] <= group(row) } for the
 * P-1 ascending host bounds (P <= 1024). The rows are written grouped by
 * destination (destination 0 first; order inside a destination unspecified) into
 * `out`, caller-allocated device columns of in->n_rows entries with the same
 * types (out->value.data may be NULL iff in->value.data is NULL); counts[P] (host)
 * receives the rows per destination. */
tcudb_status tcudb_minmax(tcudb_ctx* ctx, const void* col, int32_t type, int64_t n, int64_t* mn, int64_t* mx,
                          void* stream);
tcudb_status tcudb_partition(tcudb_ctx* ctx, const tcudb_table* in, const int64_t* bounds, int32_t P,
                             tcudb_table* out, int64_t* counts, void* stream);

/* Host-only planning steps of the collective call (§8(e)), exported so that the shard
 * plan can be checked without a GPU (pure host code: no device work, no communicator).
 *
 * tcudb_shard_agree: the agreement step. descs: P rank descriptors of
 * TCUDB_SHARD_DESC_LEN int64 each, rank-major: [0] A.n_rows, [1] B.n_rows, [2..7] column
 * states of A.key, A.group, A.value, B.key, B.group, B.value (0: no rows and a NULL
 * pointer — no vote; 1: absent; 2 + tcudb_dtype: present), [8] agg, [9] flags, [10] the
 * rank's own argument status. Writes the agreed descriptor (row totals, voted column
 * states — a column nobody votes on is absent —, agg, flags, status) into agreed[] and
 * returns its status: the most negative rank status, E_INVALID when ranks disagree on a
 * column, agg or flags, E_UNSUPPORTED for non-integer keys / groups or mixed int / float
 * values. Every rank calling it on the same allgathered bytes gets the same answer.
 *
 * tcudb_shard_bounds: the range-bound step. msgs: P messages of TCUDB_SHARD_SAMPLES + 2
 * int64, rank-major: [0] the rank's routed rows n, [1] its sample size S <= 1024, [2..]
 * S group values sampled at stride n / S. Writes the P-1 ascending bounds (rows go to
 * rank #{i : bounds[i] <= g}) at the weighted quantiles i·N/P of the pooled sample (each
 * sample weighs n / S rows); a value is never split across ranks. */
#define TCUDB_SHARD_DESC_LEN 11
#define TCUDB_SHARD_SAMPLES 1024
tcudb_status tcudb_shard_agree(const int64_t* descs, int32_t P, int64_t* agreed);
tcudb_status tcudb_shard_bounds(const int64_t* msgs, int32_t P, int64_t* bounds);

void tcudb_result_free(tcudb_ctx* ctx, tcudb_result* r);
void tcudb_result_free_host(tcudb_ctx* ctx, tcudb_result* r);
const char* tcudb_last_error(const tcudb_ctx* ctx);
/* Kernel launches recorded since the context was created (evidence counter). */
int64_t tcudb_launch_count(const tcudb_ctx* ctx);
/* The dense-vs-sparse selector's cost-model constants (a4; Eq. 3 P:1172-1175,
 * §4.2.2): out8 = {dense GEMM rate kind::i8, kind::f16 (bf16), kind::mxf4
 * (ops/s), device copy bandwidth (bytes/s), sparse-path joined pairs/s, sparse-path fixed
 * cost (s), calibration wall time (ms), dense-path fixed cost (s)}. tcudb_create measures them
 * once per device and process (environment TCUDB_CALIBRATE=0: the compiled defaults;
 * TCUDB_CALIBRATION_VALUES="R_i8,R_bf16,R_fp4,BW,R_sp,T_sp0[,T_d0]": constants measured by an
 * earlier run, for runs whose own timing is distorted, e.g. under a profiler). Returns 1 if
 * measured, 2 if injected, 0 for the defaults. */
int32_t tcudb_calibration(const tcudb_ctx* ctx, double* out8);
void tcudb_destroy(tcudb_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TCUDB_H_ */
