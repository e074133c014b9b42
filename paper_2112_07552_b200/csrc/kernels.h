// kernels.h — device-side data descriptors and the launchers of encode / fill /
// sparse / compaction kernels (host runtime in tcudb.cu drives them).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace tcudb {

// One input column (device pointer; type: 0 I32, 1 I64, 2 F32; data == NULL absent).
struct ColDesc {
  const void* data;
  int type;
  int64_t n;
};

// Column statistics (a1 / D2). Integer columns: mn, mx, min_abs as int64.
// Float columns: order-preserving int encodings of fp32 (see decode_ord), flags bit0 = non-finite seen,
// bit1 = some value is not bf16-representable.
struct ColStats {
  long long mn, mx, min_abs;
  int flags;
  int pad;
};

// Read-only view of one dictionary for lookups.
//   mode 0 (direct): code[x - minv] for x - minv < size
//   mode 1 (hash):   slots[] open addressing, size = capacity - 1 (mask), code[slot]
struct DictView {
  int mode;
  long long minv;
  unsigned long long size;
  const int32_t* code;
  const unsigned long long* slots;
  // hash mode, optional: slot of each row of the column this view is probed with (written
  // by the insert): the lookup is then code[row_slot[i]], no rehash or table walk
  const int32_t* row_slot;
  int wide;  // hash mode: offsets need 64 bits (fmix64 slot hash), else the 32-bit one
};

// ---------------------------------------------------------------- encode.cu
constexpr int kHllP = 12, kHllM = 1 << kHllP;  // HyperLogLog registers per sketch (16 KB: ~1.6 % error)
// max-merge the sketch of one int column into regs[kHllM] (regs zeroed by the caller)
cudaError_t launch_hll(const ColDesc& c, unsigned* regs, cudaStream_t s, int64_t* launches);
// hll (optional, 3 x kHllM zeroed registers): #distinct sketches of the key columns (union),
// A.g and B.h, updated in the same pass for the columns whose 4 K samples already span more
// than a direct-offset dictionary allows; gate[4] (device) records which were sketched
cudaError_t launch_col_stats(const ColDesc* cols6, ColStats* st, cudaStream_t s, int64_t* launches,
                             unsigned* hll = nullptr, int* gate = nullptr);
cudaError_t launch_mark_direct(const ColDesc& c, long long minv, uint8_t* flags, int64_t span, cudaStream_t s,
                               int64_t* launches);
// Open-addressing insert of (x - minv); *overflow = 1 if the table is full; row_slot
// (optional, c.n entries) receives each row's slot.
cudaError_t launch_hash_insert(const ColDesc& c, long long minv, unsigned long long* slots, unsigned long long mask,
                               uint8_t* flags, int* overflow, int32_t* row_slot, double est_distinct, int wide,
                               cudaStream_t s, int64_t* launches, int64_t sample_step = 1);
size_t pred_temp_bytes(int64_t n);
// codes = exclusive scan of pred(i) (-1 where false); optional dict[code] = minv + i (direct
// group domains: the sorted value dictionary comes out of the same pass).
cudaError_t launch_pred_codes(const uint8_t* fa, const uint8_t* fb, int64_t n, int32_t* code, int64_t* count_dev,
                              unsigned long long* union_dev, long long* dict, long long minv, void* temp,
                              cudaStream_t s, int64_t* launches);
// one dictionary's code scan (launch_pred_codes' arguments); launch_pred_codes_multi runs up
// to three small ones (n <= 32 K) as one launch, larger ones one by one (temps[i] each)
struct PredJob {
  const uint8_t* fa; const uint8_t* fb; int64_t n; int32_t* code; int64_t* count;
  unsigned long long* union_cnt; long long* dict; long long minv;
};
cudaError_t launch_pred_codes_multi(const PredJob* jobs, int nj, void* const* temps, cudaStream_t s,
                                    int64_t* launches);
cudaError_t launch_direct_dict(const int32_t* code, int64_t range, long long minv, long long* dict, cudaStream_t s,
                               int64_t* launches);
cudaError_t launch_gather_slots(const int32_t* tmp_code, const unsigned long long* slots, int64_t cap,
                                unsigned long long* keys, uint32_t* vals, cudaStream_t s, int64_t* launches);
cudaError_t launch_rank_write(const unsigned long long* keys, const uint32_t* vals, int64_t n, long long minv,
                              int32_t* slot_code, long long* dict, int32_t* remap, cudaStream_t s,
                              int64_t* launches);
// One-block gather + bitonic sort + rank write for small hash domains (slot_code may alias code).
bool small_rank_ok(int64_t count, int64_t cap);
size_t small_rank_temp_bytes();
cudaError_t launch_small_rank(const int32_t* code, const unsigned long long* slots, int64_t cap, int64_t count,
                              long long minv, int32_t* slot_code, long long* dict, int32_t* remap, void* temp,
                              cudaStream_t s, int64_t* launches);
// codes[i] = remap[codes[i]] for codes >= 0 (per-tuple codes issued before the rank sort)
cudaError_t launch_remap_codes(int32_t* codes, int64_t n, const int32_t* remap, cudaStream_t s, int64_t* launches);
cudaError_t launch_probe(const ColDesc& key, const ColDesc& grp, const ColDesc& val, const DictView& kd,
                         const DictView& gd, int32_t* kcode, int32_t* gcode, int32_t* cnt_k,
                         double* rowabs_g, int64_t K, cudaStream_t s, int64_t* launches);
// out[0] += J = sum cntA*cntB, out[3] += sum cntA (keys also in B), out[4] += sum cntB
cudaError_t launch_join_size(const int32_t* ca, const int32_t* cb, int64_t K, unsigned long long* out,
                             cudaStream_t s, int64_t* launches);
// *out += popcount(w[i] & mask) over n words
cudaError_t launch_popcount(const unsigned* w, int64_t n, unsigned mask, unsigned long long* out, cudaStream_t s,
                            int64_t* launches);
cudaError_t launch_max_u64(const unsigned long long* x, int64_t n, unsigned long long* out, cudaStream_t s,
                           int64_t* launches);

// ---------------------------------------------------------------- float split layout (reading R9)
// A value that is not bf16-exact is split three ways, x = hi + mid + lo + r with hi = bf16(x),
// mid = bf16(x - hi), lo = bf16(x - hi - mid), |r| <= 2^-24 |x|. Along K the operands hold
// kSplitSegs segments of Kp columns: A' = [hi|hi|hi|mid|mid|lo], B' = [hi|mid|lo|hi|mid|hi], so
// the product sums hi·hi (segment 0, its own fp32 accumulator) and the corrections hi·mid,
// hi·lo, mid·hi, mid·mid, lo·hi (every term down to 2^-16 of |v·w|). A segment's role is 2 bits
// of a `roles` word: 0 hi, 1 mid, 2 lo, 3 not written.
constexpr int kSplitSegs = 6;
constexpr int kRolesA = 0 | (0 << 2) | (0 << 4) | (1 << 6) | (1 << 8) | (2 << 10);
constexpr int kRolesB = 0 | (1 << 2) | (2 << 4) | (0 << 6) | (1 << 8) | (0 << 10);
constexpr int kRolesHi = 0xFFC;  // hi into segment 0 only (bf16 without the split)

// ---------------------------------------------------------------- fill.cu (a5)
// Device-side fill statistics read by the precision guard (a3).
struct FillStats {
  unsigned long long max_abs;  // max |cell| (integer scratch) or packed-u8 max cell
  unsigned long long nnz;      // non-zero cells
  int overflow;                // packed-u8 carry or int32 scratch overflow seen
  int inexact;                 // float: some cell is not bf16-exact
  int neg;                     // some cell < 0
  int pad;
  unsigned long long nzt;      // tuples with a nonzero bf16 (row-range direct fill)
};
// COUNT: packed u8 atomics directly into op[row][k] (row = code of the group).
cudaError_t launch_fill_count_u8(const int32_t* kcode, const int32_t* rcode, int64_t n, uint8_t* op, int64_t ld,
                                 FillStats* fs, cudaStream_t s, int64_t* launches);
// COUNT with 0/1 cells straight into packed e2m1 nibbles (ld in elements); a second tuple in a
// cell sets fs->overflow (from the atomicOr's return value).
cudaError_t launch_fill_count_fp4(const int32_t* kcode, const int32_t* rcode, int64_t n, uint8_t* op,
                                  int64_t ld_elems, FillStats* fs, cudaStream_t s, int64_t* launches);
// Float SUM with <= 1 tuple per cell and bf16-exact values: bf16 bits stored straight into
// op[r][k]; occ is a zeroed 1-bit occupancy map [rows][ld_occ bits] (a second tuple in a cell:
// popcount(occ) < tuples written, checked by the caller); fs->inexact: value not bf16-exact.
// Row-range passes of the direct bf16 fill: rows [r0, r1) only, stores kept in L2
// (evict_last) over a range sized to fit it; then nonzero cells are counted.
cudaError_t launch_fill_bf16_rows(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                                  uint16_t* op, int64_t ld_op, int32_t r0, int32_t r1, FillStats* fs, cudaStream_t s,
                                  int64_t* launches);
cudaError_t launch_count_nonzero_u16(const uint16_t* op, int64_t ld_op, int64_t rows, int64_t cols,
                                     unsigned long long* out, cudaStream_t s, int64_t* launches);
cudaError_t launch_fill_bf16_direct(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                                    uint16_t* op, int64_t ld_op, unsigned* occ, int64_t ld_occ, FillStats* fs,
                                    cudaStream_t s, int64_t* launches);
// Binned variant of the bf16 direct fill (row bands built in shared memory, written out
// coalesced including zeros). fill_bf16_binned_ws returns the workspace bytes, 0 when the
// shape does not fit the scheme (caller uses the direct fill). Duplicate cells set
// fs->overflow; inexact values set fs->inexact.
size_t fill_bf16_binned_ws(int64_t n, int64_t rows, int64_t Kp);
// Tiled direct fill (one binning level into 65,536-cell tiles, then one CTA per tile);
// workspace bytes (0: shape not supported), fs->inexact / fs->overflow as the binned fill.
size_t fill_bf16_tiled_ws(int64_t n, int64_t rows, int64_t Kp, bool split = false);
// The same for values that are not bf16-exact: fp32 tiles, written as bf16 hi / lo = bf16(x - hi)
// into the segments hi_mask / lo_mask of the hi/lo split layout (segment stride Kp, row stride
// ld_op); duplicate cells set fs->overflow (the caller then takes the fp32-scratch path).
cudaError_t launch_fill_bf16_split_tiled(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                                         int64_t rows, int64_t Kp, uint16_t* op, int64_t ld_op, int roles,
                                         FillStats* fs, void* ws, cudaStream_t s, int64_t* launches);
cudaError_t launch_fill_bf16_tiled(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                                   int64_t rows, int64_t Kp, uint16_t* op, int64_t ld_op, FillStats* fs, void* ws,
                                   cudaStream_t s, int64_t* launches);
cudaError_t launch_fill_bf16_binned(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                                    int64_t rows, int64_t Kp, uint16_t* op, int64_t ld_op, FillStats* fs, void* ws,
                                    cudaStream_t s, int64_t* launches);
// ---- fill_direct.cu: a2 + a5 fused for direct-offset dictionaries over int32 columns (c4 class)
constexpr int kDirectSpanMax = 16384;  // key / group spans whose u16 code tables the fill keeps in smem
// One side: cnt_span[x - kmin] += #tuples with key x; kflag[x - kmin] = 1, gflag[g - gmin] = 1
// (zeroed by the caller). 16-byte aligned columns; kspan * 4 + gspan <= 160 KB.
bool direct_count_ok(int64_t kspan, int64_t gspan);
cudaError_t launch_direct_count(const int32_t* key, const int32_t* grp, int64_t n, long long kmin, int64_t kspan,
                                long long gmin, int64_t gspan, int32_t* cnt_span, uint8_t* kflag, uint8_t* gflag,
                                cudaStream_t s, int64_t* launches);
struct DtFill {
  const int32_t* key; const int32_t* grp; const float* val; int64_t n;  // val NULL: 1.0
  long long kmin; int kspan; const int32_t* kcode;  // code table over the key span (-1: not in the ∩ domain)
  long long gmin; int gspan; const int32_t* gcode;  // row-code table over the group span
  int64_t rows, Kp;                                 // operand rows (multiple of 8) and K columns (of 128)
  uint16_t* op; int64_t ld_op;                      // bf16 operand [rows][ld_op] (elements)
  int roles;                                        // split: role of each K segment (stride Kp)
  uint8_t* pat; int64_t ld_pat;                     // optional e2m1 existence pattern [rows][ld_pat bytes]
  FillStats* fs;                                    // fs->overflow: a cell with two tuples
};
bool fill_direct_ok(const DtFill& f, bool split);
size_t fill_direct_ws(int64_t rows, int64_t Kp, bool split);
// split = false: bf16-exact values, cells written as bf16; true: fp32 cells -> hi / lo segments
cudaError_t launch_fill_direct(const DtFill& f, bool split, void* ws, cudaStream_t s, int64_t* launches);
// Pattern plane op[r][k] = 1 where a cell holds >= 1 tuple; symmetric adjacency for triangles.
cudaError_t launch_fill_pattern_u8(const int32_t* kcode, const int32_t* rcode, int64_t n, uint8_t* op, int64_t ld,
                                   cudaStream_t s, int64_t* launches);
cudaError_t launch_fill_sym_pattern(const int32_t* u, const int32_t* v, int64_t n, uint8_t* op, int64_t ld,
                                    cudaStream_t s, int64_t* launches);
// Integer values (or 1) accumulated into an int64 scratch [rows][ld] (wrapping adds: exact
// modulo 2^64, so exact whenever the guard has bounded the true cell value inside int64).
cudaError_t launch_fill_i64(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n,
                            long long* scr, int64_t ld, cudaStream_t s, int64_t* launches);
// Float values accumulated into an fp32 scratch.
cudaError_t launch_fill_f32(const int32_t* kcode, const int32_t* rcode, const ColDesc& val, int64_t n, float* scr,
                            int64_t ld, cudaStream_t s, int64_t* launches);
// Statistics of an int64 scratch (max |cell|, nnz, sign).
cudaError_t launch_scratch_stats_i64(const long long* scr, int64_t count, FillStats* fs, cudaStream_t s,
                                     int64_t* launches);
// Base-256 digit planes from an int64 scratch: plane p at op + p*plane_stride (bytes);
// digits 0..P-2 are u8, the top digit is s8 when top_signed, else u8.
cudaError_t launch_pack_planes(const long long* scr, int64_t count, int planes, int top_signed, uint8_t* op,
                               int64_t plane_stride, cudaStream_t s, int64_t* launches);
// fp32 scratch [rows][ld] -> bf16 hi into op[row][i*ld + k] for every segment i in hi_mask,
// lo = bf16(x - hi) into the segments in lo_mask (row stride ld_op elements); counts
// inexact cells.
cudaError_t launch_pack_bf16(const float* scr, int64_t rows, int64_t ld, uint16_t* op, int64_t ld_op, int roles,
                             FillStats* fs, cudaStream_t s, int64_t* launches);

// ---------------------------------------------------------------- sparse.cu (a7)
cudaError_t launch_bucket_fill(const int32_t* kcode, const int32_t* hcode, const ColDesc& w, int64_t n,
                               const int64_t* bstart, int32_t* cursor, int32_t* b_h, void* b_w, int w_kind,
                               cudaStream_t s, int64_t* launches);
cudaError_t launch_work(const int32_t* kcode, int64_t n, const int32_t* cnt_b, int32_t* work, cudaStream_t s,
                        int64_t* launches);
// Active A tuples grouped by band g / R (counting sort): act_a[]/act_w[] (zeroed act_w
// tail); with nb = ceil(G / R): gcnt (zeroed, nb), goff (nb + 1, total at goff[nb]), gcur
// (zeroed, nb).
// Optional (non-NULL bstart): act_b[] = bucket start of the tuple's key, act_g[] = its row.
cudaError_t launch_active_by_g(const int32_t* kcode, const int32_t* gcode, const int32_t* cnt_b, int64_t n, int G, int R,
                               int32_t* gcnt, int64_t* goff, int32_t* gcur, int32_t* act_a, int32_t* act_w,
                               const int64_t* bstart, int64_t* act_b, int32_t* act_g,
                               void* scan_tmp, cudaStream_t s, int64_t* launches);
cudaError_t launch_flags_from_work(const int32_t* work, int64_t n, int32_t* flags, cudaStream_t s,
                                   int64_t* launches);
cudaError_t launch_compact_active(const int32_t* work, const int64_t* pos, int64_t n, int32_t* act_a,
                                  int32_t* act_w, cudaStream_t s, int64_t* launches);
struct ExpandArgs {
  int64_t n_act, J;
  const int32_t* act_a; const int64_t* act_off;
  const int32_t* kcodeA; const int32_t* gcodeA; ColDesc va;
  const int64_t* bstart; const int32_t* b_h; const void* b_w;
  int w_kind;      // 0 none (1), 1 int64, 2 f32
  int acc_kind;    // 0 COUNT int32, 1 COUNT int64, 2 int SUM int64, 3 float SUM f64, 4 COUNT u16
  void* C; int64_t ldc;
  int32_t* cnt;    // optional existence count plane (int32) or NULL
  int* ovf;        // acc_kind 4 (COUNT, packed u16, ldc even): set when a count passes 65535
};
cudaError_t launch_expand(const ExpandArgs& a, cudaStream_t s, int64_t* launches);

// ---------------------------------------------------------------- spa.cu (a7 + a8 fused, sparse path)
struct SpaArgs {
  int64_t G, H;
  const int64_t* goff;     // nbands + 1: active-tuple range of each band of `rows` rows (tuples grouped by band)
  const int32_t* act_a;    // active A tuples (row index into A), g-ordered
  const int64_t* act_off;  // n_act + 1: first update of each active tuple (exclusive scan of cntB[k])
  const int64_t* act_b;    // bucket start of each active tuple's key
  const int32_t* act_g;    // row (group code) of each active tuple
  const int32_t* kcodeA; const int32_t* gcodeA; ColDesc va;
  const int64_t* bstart; const int32_t* b_h; const void* b_w;
  int w_kind;              // 0 none (1), 1 int64, 2 f32
  int acc_kind;            // 0 COUNT int32, 1 COUNT int64, 2 int SUM int64 (wrapping), 3 float SUM f64
  int64_t words;           // 32-bit bitmap words per row (set by spa_plan)
  int rows;                // rows per band = per CTA of the write pass (set by spa_plan)
  int64_t nbands;          // ceil(G / rows) (set by spa_plan)
  int count_bands;         // bands per CTA of the count pass (set by spa_plan)
  int32_t* row_nnz;        // count pass output (G)
  const int64_t* row_out;  // write pass input: exclusive scan of row_nnz
  const long long* dict_g; const long long* dict_h;
  int g_out_type, h_out_type;  // 0 I32, 1 I64
  void* out_g; void* out_h; void* out_agg;
  // one-pass kernel (spa_fused_plan / launch_spa_fused); acc_kind 4 = COUNT in packed u16
  unsigned long long* ticket;  // 1, zeroed: band tickets
  unsigned long long* lb_state;  // nbands, zeroed: look-back (flag | tuple count) per band
  int64_t* total;              // out: number of result tuples
  int* ovf;                    // out (zeroed): a u16 COUNT cell reached 65,535
  // count pass over a subset of bands (the hub bands of the hybrid schedule): band_list[i]
  // for i < n_list, one band per CTA; NULL: every band
  const int32_t* band_list;
  int64_t n_list;
};
// Hybrid one-pass schedule: the bands heavier than thr updates (hubs) -> list (count in
// *n_out); after their count pass, their tuple counts are published in lb_state (look-back
// aggregates) so that no later band's look-back waits for a hub's expansion.
cudaError_t launch_hub_list(const SpaArgs& a, unsigned long long thr, int32_t* list, unsigned long long* n_out,
                            cudaStream_t s, int64_t* launches);
cudaError_t launch_hub_publish(const SpaArgs& a, cudaStream_t s, int64_t* launches);
// false when one result row does not fit in shared memory (the caller keeps the C path)
bool spa_plan(SpaArgs& a);
bool spa_fused_plan(SpaArgs& a);
void spa_count_plan(SpaArgs& a);  // count_bands for the count pass at the current rows
cudaError_t launch_spa_fused(const SpaArgs& a, cudaStream_t s, int64_t* launches);
// *out = max over bands of the band's update count (out zeroed by the caller)
cudaError_t launch_band_weight_max(const SpaArgs& a, unsigned long long* out, cudaStream_t s, int64_t* launches);
cudaError_t launch_spa_count(const SpaArgs& a, cudaStream_t s, int64_t* launches);
cudaError_t launch_spa_write(const SpaArgs& a, cudaStream_t s, int64_t* launches);

// gcode[i] = code of grp[i] in the dictionary gd (final codes)
// per-tuple group codes; miss (optional): set when a value is not in the dictionary (a sampled
// build missed it: the caller rebuilds)
cudaError_t launch_group_codes(const ColDesc& grp, const DictView& gd, int32_t* gcode, cudaStream_t s,
                               int64_t* launches, int* miss = nullptr);

// ---------------------------------------------------------------- hashpart.cu (a2 + a7, partitioned)
// Hash-partitioned sparse COUNT for large hash-mode key domains: both tables are
// radix-partitioned by the key hash so that each partition's key dictionary, per-key
// counts and B buckets live in one CTA's shared memory.
struct PartSide {
  ColDesc key;            // raw join-key column (pass 1 input)
  const int32_t* gcode;   // group codes of the rows (pass 1 input)
  unsigned long long* k[2];  // ping-pong koff = key - kmin (u64)
  int32_t* g[2];             // ping-pong group codes
};
size_t hashpart_temp_bytes(int64_t n, int nseg, int bits);
// One radix pass over nseg segments (segment s = [seg_off[s], seg_off[s+1])): digit =
// (fmix64(koff) >> shift) & (2^bits - 1); output segment-major, then digit. in_raw: pass 1
// reads the raw key column and the gcode array instead of (k_in, g_in). seg_out (nseg *
// 2^bits + 1) receives the new segment offsets.
// pass 1 (raw != NULL): raw key column + per-tuple group codes g_raw; later passes: k_in / g_in
cudaError_t launch_part_pass(const ColDesc* raw, long long kmin, const int32_t* g_raw,
                             const unsigned long long* k_in, const int32_t* g_in, const int64_t* seg_off, int nseg,
                             int64_t n, int shift, int bits, unsigned long long* k_out, int32_t* g_out,
                             int64_t* seg_out, void* temp, cudaStream_t s, int64_t* launches,
                             const ColDesc* v_raw = nullptr, const long long* v_in = nullptr,
                             long long* v_out = nullptr);  // value payload (integer SUM), optional
// histogram of the top pbits (<= 14) of the key hash over one side's raw keys (hist zeroed)
cudaError_t launch_part_hist_all(const ColDesc& raw, long long kmin, int pbits, unsigned* hist, cudaStream_t s,
                                 int64_t* launches);
// one radix pass with atomic run reservation: cursor[s * 2^bits + d] = the next free slot of
// digit d of segment s (initialized to its start by the caller)
size_t hashpart_atomic_temp_bytes(int nseg);
cudaError_t launch_part_pass_atomic(const ColDesc* raw, long long kmin, const int32_t* g_raw,
                                    const unsigned long long* k_in, const int32_t* g_in, const int64_t* seg_off,
                                    int nseg, int64_t n, int shift, int bits, unsigned long long* cursor,
                                    unsigned long long* k_out, int32_t* g_out, void* temp, cudaStream_t s,
                                    int64_t* launches, const ColDesc* v_raw = nullptr, const long long* v_in = nullptr,
                                    long long* v_out = nullptr);
size_t part_expand_smem(int cap, bool sum);
// per partition: J_p = sum over its keys of cntA*cntB, D_p = #keys on both sides; out has
// 4 + 4 P entries: totals out[0] (J), out[1] (K = sum D_p), out[2] (A tuples with a matched
// key), out[3] (distinct B keys); per-partition values after them
// stride > 1: only partitions 0, stride, 2 stride, ... (a sample for the selector's
// estimate; the per-partition values are then those of the sampled partitions)
cudaError_t launch_part_count(const unsigned long long* ka, const int64_t* offa, const unsigned long long* kb,
                              const int64_t* offb, int P, int cap, unsigned long long* out, cudaStream_t s,
                              int64_t* launches, int stride = 1);
// per partition: C[g][h] += 1 for every joined pair (u32 cells, row stride ldc); with C64,
// also C64[g][h] += va·vb (integer SUM, wrapping int64)
cudaError_t launch_part_expand(const unsigned long long* ka, const int32_t* ga, const int64_t* offa,
                               const unsigned long long* kb, const int32_t* hb, const int64_t* offb, int P, int cap,
                               unsigned* C, int64_t ldc, cudaStream_t s, int64_t* launches,
                               const long long* va = nullptr, const long long* vb = nullptr,
                               unsigned long long* C64 = nullptr, unsigned long long* jk = nullptr);
// jk (4 + 4 P entries, required): the exact join size J = jk[0] and K = jk[1] (keys with
// pairs), measured while expanding
// largest partition (max over both sides) into *out (zeroed)
cudaError_t launch_part_max(const int64_t* offa, const int64_t* offb, int P, unsigned long long* out, cudaStream_t s,
                            int64_t* launches);

// ---------------------------------------------------------------- tri_sparse.cu (a9 sparse, §8(f) f3)
size_t tri_sparse_temp_bytes(int64_t n, int64_t V);
size_t tri_sparse_smem(int64_t V);  // bitmap bytes per CTA (V bits); <= 200 KB required
// *out += number of triangles of the simple undirected graph on the coded edges (cu, cv < V)
cudaError_t launch_tri_sparse(const int32_t* cu, const int32_t* cv, int64_t n, int64_t V, void* temp,
                              unsigned long long* out, cudaStream_t s, int64_t* launches);

// ---------------------------------------------------------------- reduce.cu (§8(f) f2)
// One side ungrouped (Q3 P:785-823, Q4 P:842-850) or AVG: segmented reductions.
struct SideOut {
  const long long* dict_grp;          // grouped side's ascending value dictionary
  void* grp_out; int grp_type;        // its output column (0 I32, 1 I64)
  void* const_out; int const_type;    // the single-group side's output column (NULL: absent)
  long long const_val;
  void* agg;                          // I64 (COUNT, int SUM) or F64 (float SUM, AVG)
};
// sum_k[kcode[i]] += v[i]; kind 1: int64 (wrapping), 2: fp64 of fp32 values
cudaError_t launch_key_sum(const int32_t* kcode, const ColDesc& v, int64_t n, int kind, void* sum_k, cudaStream_t s,
                           int64_t* launches);
// cnt_g[g] += cnt_o[k]; sum_g[g] += w · (sum_o ? sum_o[k] : cnt_o[k]); kind 0 COUNT, 1 int, 2 float
cudaError_t launch_side_agg(const int32_t* kcode, const int32_t* gcode, const ColDesc& w, int64_t n,
                            const int32_t* cnt_o, const void* sum_o, int kind, int64_t NG,
                            unsigned long long* cnt_g, void* sum_g, cudaStream_t s, int64_t* launches);
cudaError_t launch_side_flags(const unsigned long long* cnt_g, int64_t NG, int32_t* flags, cudaStream_t s,
                              int64_t* launches);
// agg_kind: 0 COUNT, 1 int SUM, 2 float SUM, 3 AVG of int, 4 AVG of float
cudaError_t launch_side_write(const unsigned long long* cnt_g, const void* sum_g, const int64_t* pos, int64_t NG,
                              int agg_kind, const SideOut& o, cudaStream_t s, int64_t* launches);
// in place: sum (int64 or fp64) -> fp64 sum / cnt
cudaError_t launch_avg_div(void* sum_inout, int sum_is_float, const long long* cnt, int64_t n, cudaStream_t s,
                           int64_t* launches);

// ---------------------------------------------------------------- partition.cu (§8(e))
// destination = group range (bounds) or, by_key != 0, a hash of the join key (bounds unused)
cudaError_t launch_part_count(const ColDesc& key, const ColDesc& grp, const long long* bounds, int P, int by_key,
                              unsigned long long* counts, cudaStream_t s, int64_t* launches);
cudaError_t launch_part_scatter(const ColDesc& key, const ColDesc& grp, const ColDesc& val, const long long* bounds,
                                int P, int by_key, unsigned long long* cursor, void* ok, void* og, void* ov,
                                cudaStream_t s, int64_t* launches);

// ---------------------------------------------------------------- compact.cu (a8)
// Existence matrix E (int32 count or the value matrix) -> tuples (g, h, agg), row-major.
struct CompactArgs {
  int64_t G, H;
  int64_t nseg;                                  // segments per row (= GEMM N tiles on the dense path)
  int64_t seg_w;                                 // columns per segment (<= 256; 256, or 240 for fp4)
  const void* E; int e_kind; int64_t lde;       // e_kind: 0 int32, 1 int64, 2 f32, 3 f64, 4 u16
  const void* V; int v_kind; int64_t ldv;       // value matrix (agg), same kinds
  const long long* dict_g; const long long* dict_h;
  int g_out_type, h_out_type;                    // 0 I32, 1 I64
  int agg_out;                                   // 0 int64, 1 f64
  void* out_g; void* out_h; void* out_agg;
  // affine h dictionary (a direct-offset domain with every value present: value = code + h_base):
  // the decode is an add instead of a gather
  int h_affine; long long h_base;
};
size_t compact_temp_bytes(int64_t G, int64_t nseg);
cudaError_t launch_compact_count(const CompactArgs& a, const int32_t* precounted, int64_t* nnz_dev, void* temp,
                                 cudaStream_t s, int64_t* launches);
cudaError_t launch_compact_write(const CompactArgs& a, void* temp, cudaStream_t s, int64_t* launches);

}  // namespace tcudb

namespace tcudb {
// ---------------------------------------------------------------- calib.cu
// synthetic int32 columns for the create-time calibration: k uniform over [0, keys),
// g uniform over [0, groups)
cudaError_t launch_gen_cols(int32_t* k, int32_t* g, int64_t n, uint32_t keys, uint32_t groups, uint32_t seed,
                            cudaStream_t s, int64_t* launches);
}  // namespace tcudb

namespace tcudb {
// ---------------------------------------------------------------- blocksparse.cu (§8(f) f4)
// Re-code the join keys in order of their smallest A row (kA / kB and the per-key counts
// are rewritten in place).
size_t bs_reorder_temp_bytes(int64_t K);
cudaError_t launch_bs_reorder(int32_t* kA, const int32_t* gA, int64_t nA, int32_t* kB, int64_t nB, int32_t* cntA,
                              int32_t* cntB, int64_t K, int64_t G, void* temp, cudaStream_t s, int64_t* launches);
// base occupancy bitmap (zeroed by the caller): 16-row x 64-key blocks, W words per row group
cudaError_t launch_bs_mark(const int32_t* kcode, const int32_t* rcode, int64_t n, int W, unsigned long long* bm,
                           cudaStream_t s, int64_t* launches);
// tile bitmaps for one GEMM launch: rows_per_tile (multiple of 16) rows per tile, f key groups
// of 64 per K-block, K-block kb maps to key group (kb mod period_kb) * f (the hi/lo split
// repeats the key space along K), Wout words per tile
cudaError_t launch_bs_derive(const unsigned long long* base, int base_rows, int W, int rows_per_tile, int f,
                             int64_t period_kb, int64_t total_kb, int ntiles, int Wout, unsigned long long* out,
                             cudaStream_t s, int64_t* launches);
// *out += active (tile pair, K-block) products
cudaError_t launch_bs_active(const unsigned long long* a, const unsigned long long* b, int tiles_m, int tiles_n,
                             int Wt, unsigned long long* out, cudaStream_t s, int64_t* launches);
}  // namespace tcudb
