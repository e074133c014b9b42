// collective.cu — the multi-GPU form of tcudb_join_agg (SURVEY §8(b) "Multi-GPU" and
// §8(e)): when the context was created with an NCCL communicator, every rank passes its
// local slices of A and B and the call is collective.
//
// Output rows are independent units (§3.2: C[g][h] depends only on A's rows of
// group g and B's rows of group h), so they are sharded by ranges of the grouped side's
// group key and the only exchanges are data movement:
//   0. agreement: every rank's query shape (rows, column presence and types, aggregate,
//      flags, its local argument check) is allgathered and one decision is taken from the
//      same bytes on every rank — a rank whose slice is empty (NULL columns) takes the
//      others' shape; a disagreement fails on every rank with the same status;
//   1. range bounds balanced on rows (§8(e) step 2): each rank allgathers a strided sample
//      of its routed group column (<= 1024 values + its row count); every rank computes
//      the same P-1 weighted quantiles of the pooled sample;
//   2. the routed side's rows are sent to the rank owning their group (tcudb_partition +
//      all-to-all-v as grouped ncclSend / ncclRecv);
//   3. the other side is allgathered (allgather-v as grouped send / recv);
//   4. the local query on (routed rows, all of the other side) -> exactly the groups of
//      this rank's range, complete (COUNT, SUM and AVG need no cross-rank combine);
//   5. allgather-v of the result columns in rank order: ranges ascend with the rank and
//      each shard is (g, h)-sorted, so the concatenation is the single-GPU result.
//      TCUDB_GATHER_NONE returns the rank's shard instead.
// Routed side: A (by A.g) when A is grouped; GROUP BY B.h only (Q3) routes B
// by h. No GROUP BY (Q4): every rank joins its own A slice with the gathered
// B and the per-rank partial aggregates are allgathered and combined exactly (int SUM in
// 128 bits: a total beyond int64 is E_OVERFLOW on every rank, as on one GPU).
// Every local step that can fail (partition, local query) is followed by an agreement on
// the status (allreduce MIN) before the next exchange, so one rank's error is every
// rank's error instead of a peer blocked in a collective.
//
// NCCL is resolved at context creation with dlopen (the process's already-loaded
// libnccl.so.2 — torch's — first; TCUDB_NCCL_LIB names another library implementing the
// same symbols, e.g. the tests' in-process communicator), so a library used without a
// communicator has no NCCL dependency. The communicator is owned by the caller.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/tcudb.h"
#include "internal.h"
#include "kernels.h"

namespace tcudb {
namespace {

// NCCL's stable ABI values (nccl.h): data types and reduction ops used here
constexpr int kNcclInt8 = 0, kNcclInt64 = 4;
constexpr int kNcclMin = 3;

// query-shape descriptor (one per rank, allgathered): n_A, n_B, six column states
// (A.key, A.group, A.value, B.key, B.group, B.value), agg, flags, local argument status
constexpr int kDesc = TCUDB_SHARD_DESC_LEN;
constexpr int kSamples = TCUDB_SHARD_SAMPLES;
constexpr int kSampleMsg = kSamples + 2;

struct CommError {
  std::string what;
};

struct DevBuf {  // stream-ordered device buffer
  void* p = nullptr;
  cudaStream_t s;
  DevBuf(size_t bytes, cudaStream_t st) : s(st) {
    if (pool_malloc(&p, bytes ? bytes : 8, s) != cudaSuccess) {
      cudaGetLastError();
      throw CommError{"device allocation for the exchange"};
    }
  }
  ~DevBuf() { if (p) cudaFreeAsync(p, s); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) { cudaGetLastError(); throw CommError{std::string(what) + ": " + cudaGetErrorString(e)}; }
}

size_t type_bytes(int32_t t) { return (t == TCUDB_I64 || t == TCUDB_F64) ? 8 : 4; }

// 0: no vote (no rows, no pointer: present-but-empty and absent look alike), 1: absent,
// 2 + type: present
int64_t col_state(const tcudb_col& c, int64_t n) {
  if (!c.data) return n == 0 ? 0 : 1;
  return 2 + (int64_t)c.type;
}

}  // namespace

struct NcclComm {
  void* comm = nullptr;
  int nranks = 1, rank = 0;
  int (*CommCount)(void*, int*) = nullptr;
  int (*CommUserRank)(void*, int*) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*ErrStr)(int) = nullptr;

  void nck(int r, const char* what) const {
    if (r != 0) throw CommError{std::string(what) + ": " + (ErrStr ? ErrStr(r) : "NCCL error")};
  }
  // allgather of m int64 per rank, read back on the host (rank-major)
  std::vector<int64_t> gather_vec(const int64_t* x, int m, cudaStream_t s) const {
    DevBuf d(sizeof(int64_t) * (size_t)m * (nranks + 1), s);
    int64_t* mine = d.as<int64_t>() + (size_t)m * nranks;
    ck(cudaMemcpyAsync(mine, x, sizeof(int64_t) * m, cudaMemcpyHostToDevice, s), "H2D");
    nck(AllGather(mine, d.as<int64_t>(), (size_t)m, kNcclInt64, comm, s), "ncclAllGather");
    std::vector<int64_t> h((size_t)m * nranks);
    ck(cudaMemcpyAsync(h.data(), d.p, sizeof(int64_t) * h.size(), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    return h;
  }
  std::vector<int64_t> gather_i64(int64_t x, cudaStream_t s) const { return gather_vec(&x, 1, s); }
  // every rank's status -> the same status on every rank (MIN: any error wins)
  tcudb_status agree(tcudb_status st, cudaStream_t s) const {
    DevBuf d(8, s);
    const int64_t v = (int64_t)st;
    ck(cudaMemcpyAsync(d.p, &v, 8, cudaMemcpyHostToDevice, s), "H2D");
    nck(AllReduce(d.p, d.p, 1, kNcclInt64, kNcclMin, comm, s), "ncclAllReduce");
    int64_t r = 0;
    ck(cudaMemcpyAsync(&r, d.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    return (tcudb_status)r;
  }
  // grouped point-to-point exchange: send[j] bytes at soff[j] of src to rank j, recv[j]
  // bytes from rank j at roff[j] of dst (the rank's own part is a device copy)
  void exchange(const char* src, const std::vector<size_t>& send, const std::vector<size_t>& soff, char* dst,
                const std::vector<size_t>& recv, const std::vector<size_t>& roff, cudaStream_t s) const {
    if (send[rank]) ck(cudaMemcpyAsync(dst + roff[rank], src + soff[rank], send[rank], cudaMemcpyDeviceToDevice, s),
                       "local part");
    nck(GroupStart(), "ncclGroupStart");
    for (int j = 0; j < nranks; ++j) {
      if (j == rank) continue;
      if (send[j]) nck(Send(src + soff[j], send[j], kNcclInt8, j, comm, s), "ncclSend");
      if (recv[j]) nck(Recv(dst + roff[j], recv[j], kNcclInt8, j, comm, s), "ncclRecv");
    }
    nck(GroupEnd(), "ncclGroupEnd");
  }
};

NcclComm* nccl_attach(void* comm, std::string* err) {
  const char* alt = getenv("TCUDB_NCCL_LIB");  // another implementation of the NCCL symbols
  void* h = nullptr;
  if (alt && alt[0]) {
    h = dlopen(alt, RTLD_NOW | RTLD_LOCAL);
  } else {
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (torch's)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) { *err = "NCCL library not found"; return nullptr; }
  NcclComm* c = new NcclComm();
  c->comm = comm;
  bool ok = true;
  auto sym = [&](auto& fn, const char* name) {
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
    if (!fn) ok = false;
  };
  sym(c->CommCount, "ncclCommCount");
  sym(c->CommUserRank, "ncclCommUserRank");
  sym(c->AllReduce, "ncclAllReduce");
  sym(c->AllGather, "ncclAllGather");
  sym(c->Send, "ncclSend");
  sym(c->Recv, "ncclRecv");
  sym(c->GroupStart, "ncclGroupStart");
  sym(c->GroupEnd, "ncclGroupEnd");
  sym(c->ErrStr, "ncclGetErrorString");
  if (!ok || c->CommCount(comm, &c->nranks) != 0 || c->CommUserRank(comm, &c->rank) != 0 || c->nranks < 1 ||
      c->nranks > 1024) {
    *err = "NCCL symbols or communicator unusable";
    delete c;
    return nullptr;
  }
  return c;
}

void nccl_detach(NcclComm* c) { delete c; }

// ---------------------------------------------------------------- host-only planning
tcudb_status shard_agree(const int64_t* descs, int P, int64_t* agreed) {
  std::memset(agreed, 0, sizeof(int64_t) * kDesc);
  if (P < 1) return TCUDB_E_INVALID;
  tcudb_status st = TCUDB_OK;
  for (int r = 0; r < P; ++r) {
    const int64_t* d = descs + (size_t)r * kDesc;
    agreed[0] += d[0];
    agreed[1] += d[1];
    st = std::min(st, (tcudb_status)d[10]);
    if (d[8] != descs[8] || d[9] != descs[9]) st = std::min(st, TCUDB_E_INVALID);  // agg / flags differ
  }
  agreed[8] = descs[8];
  agreed[9] = descs[9];
  for (int c = 0; c < 6; ++c) {
    int64_t v = 0;
    for (int r = 0; r < P; ++r) {
      const int64_t x = descs[(size_t)r * kDesc + 2 + c];
      if (x == 0) continue;
      if (v == 0) v = x;
      else if (v != x) st = std::min(st, TCUDB_E_INVALID);  // present on one rank, absent / other type on another
    }
    agreed[2 + c] = v == 0 ? 1 : v;
  }
  const bool vals = agreed[8] != TCUDB_COUNT;
  for (int side = 0; side < 2; ++side) {
    const int64_t* t = agreed + 2 + 3 * side;
    const int64_t n = agreed[side];
    if (n > 0 && t[0] < 2) st = std::min(st, TCUDB_E_INVALID);  // rows without a key column
    auto int_t = [](int64_t x) { return x == 2 + TCUDB_I32 || x == 2 + TCUDB_I64; };
    if ((t[0] >= 2 && !int_t(t[0])) || (t[1] >= 2 && !int_t(t[1]))) st = std::min(st, TCUDB_E_UNSUPPORTED);
    if (vals && t[2] >= 2 && !int_t(t[2]) && t[2] != 2 + TCUDB_F32) st = std::min(st, TCUDB_E_UNSUPPORTED);
  }
  if (vals && agreed[4] >= 2 && agreed[7] >= 2 && ((agreed[4] == 2 + TCUDB_F32) != (agreed[7] == 2 + TCUDB_F32)))
    st = std::min(st, TCUDB_E_UNSUPPORTED);  // mixed integer / float values
  agreed[10] = st;
  return st;
}

void shard_bounds(const int64_t* msgs, int P, int64_t* bounds) {
  struct Smp { int64_t v; double w; };
  std::vector<Smp> all;
  double W = 0;
  int64_t vmax = INT64_MIN;
  for (int r = 0; r < P; ++r) {
    const int64_t* m = msgs + (size_t)r * kSampleMsg;
    const int64_t n = m[0], S = std::min<int64_t>(m[1], kSamples);
    if (n <= 0 || S <= 0) continue;
    const double w = (double)n / (double)S;  // each sample stands for n / S rows
    for (int64_t i = 0; i < S; ++i) { all.push_back({m[2 + i], w}); vmax = std::max(vmax, m[2 + i]); }
    W += (double)n;
  }
  std::sort(all.begin(), all.end(), [](const Smp& a, const Smp& b) { return a.v < b.v; });
  // bound i = the smallest sampled value whose preceding weight reaches i·W/P (ties of a
  // value stay on one rank: rows go to #{i : bounds[i] <= g})
  size_t j = 0;
  double cum = 0;
  int64_t prev = INT64_MIN;
  for (int i = 1; i < P; ++i) {
    const double target = W * (double)i / (double)P;
    while (j < all.size() && cum + 1e-9 * W < target) {
      const int64_t v = all[j].v;
      while (j < all.size() && all[j].v == v) cum += all[j++].w;  // whole value
    }
    int64_t b;
    if (all.empty()) b = 0;
    else if (j < all.size()) b = all[j].v;
    else b = vmax == INT64_MAX ? INT64_MAX : vmax + 1;
    b = std::max(b, prev);
    bounds[i - 1] = b;
    prev = b;
  }
}

namespace {

struct Cols {  // device columns of one table owned by this file
  std::vector<std::unique_ptr<DevBuf>> bufs;
  tcudb_table t{};
};

// allgather-v of every present column of T (rank order)
void gather_table(const NcclComm& nc, const tcudb_table& T, Cols& out, cudaStream_t s) {
  const std::vector<int64_t> n = nc.gather_i64(T.n_rows, s);
  int64_t tot = 0;
  std::vector<int64_t> off(nc.nranks);
  for (int j = 0; j < nc.nranks; ++j) { off[j] = tot; tot += n[j]; }
  out.t = T;
  out.t.n_rows = tot;
  const tcudb_col* in[3] = {&T.key, &T.group, &T.value};
  tcudb_col* dst[3] = {&out.t.key, &out.t.group, &out.t.value};
  for (int c = 0; c < 3; ++c) {
    if (!in[c]->data) continue;  // absent on every rank (normalized presence)
    const size_t e = type_bytes(in[c]->type);
    out.bufs.emplace_back(new DevBuf((size_t)tot * e, s));
    std::vector<size_t> send(nc.nranks, (size_t)T.n_rows * e), soff(nc.nranks, 0), recv(nc.nranks), roff(nc.nranks);
    for (int j = 0; j < nc.nranks; ++j) { recv[j] = (size_t)n[j] * e; roff[j] = (size_t)off[j] * e; }
    nc.exchange(static_cast<const char*>(in[c]->data), send, soff, out.bufs.back()->as<char>(), recv, roff, s);
    dst[c]->data = out.bufs.back()->p;
  }
}

// balanced bounds of the routed group column: strided sample -> allgather -> quantiles
std::vector<int64_t> balanced_bounds(const NcclComm& nc, const tcudb_table& T, cudaStream_t s) {
  std::vector<int64_t> msg(kSampleMsg, 0);
  const int64_t n = T.n_rows;
  const int64_t S = std::min<int64_t>(n, kSamples);
  msg[0] = n;
  msg[1] = S;
  if (S > 0) {
    const size_t e = type_bytes(T.group.type);
    const int64_t stride = n / S;  // >= 1; samples i*stride, i < S
    std::vector<int32_t> h32;
    if (e == 8) {
      ck(cudaMemcpy2DAsync(msg.data() + 2, 8, T.group.data, (size_t)stride * 8, 8, (size_t)S, cudaMemcpyDeviceToHost,
                           s), "sample D2H");
    } else {
      h32.resize(S);
      ck(cudaMemcpy2DAsync(h32.data(), 4, T.group.data, (size_t)stride * 4, 4, (size_t)S, cudaMemcpyDeviceToHost, s),
         "sample D2H");
    }
    ck(cudaStreamSynchronize(s), "sync");
    for (int64_t i = 0; i < (int64_t)h32.size(); ++i) msg[2 + i] = h32[i];
  }
  const std::vector<int64_t> all = nc.gather_vec(msg.data(), kSampleMsg, s);
  std::vector<int64_t> b(nc.nranks > 1 ? nc.nranks - 1 : 1, 0);
  shard_bounds(all.data(), nc.nranks, b.data());
  // every rank must route by the SAME bounds (a group range split over two ranks would come
  // back twice): rank 0's bounds are allgathered and used everywhere; a rank whose own
  // computation differed reports it (TCUDB_DEBUG_BOUNDS=1)
  const std::vector<int64_t> ball = nc.gather_vec(b.data(), (int)b.size(), s);
  bool same = true;
  for (size_t i = 0; i < b.size(); ++i) same = same && ball[i] == b[i];
  if (!same) {
    static const bool dbg = getenv("TCUDB_DEBUG_BOUNDS") && getenv("TCUDB_DEBUG_BOUNDS")[0] == '1';
    if (dbg) fprintf(stderr, "tcudb: rank %d range bounds differ from rank 0's (using rank 0's)\n", nc.rank);
    for (size_t i = 0; i < b.size(); ++i) b[i] = ball[i];
  }
  return b;
}

// route the rows of T to the rank owning their group range (by_key: the rank owning a hash
// of their join key — the key-partitioned path)
tcudb_status route_table(tcudb_ctx* ctx, const NcclComm& nc, const tcudb_table& T, Cols& out, cudaStream_t s,
                         bool by_key = false) {
  const int P = nc.nranks;
  const std::vector<int64_t> bounds = by_key ? std::vector<int64_t>(P > 1 ? P - 1 : 1, 0) : balanced_bounds(nc, T, s);
  // partition locally
  Cols part;
  part.t = T;
  const tcudb_col* in[3] = {&T.key, &T.group, &T.value};
  tcudb_col* pc[3] = {&part.t.key, &part.t.group, &part.t.value};
  for (int c = 0; c < 3; ++c) {
    if (!in[c]->data) continue;
    part.bufs.emplace_back(new DevBuf((size_t)T.n_rows * type_bytes(in[c]->type), s));
    pc[c]->data = part.bufs.back()->p;
  }
  std::vector<int64_t> counts(P, 0);
  tcudb_status st = partition_table(ctx, &T, bounds.data(), P, by_key ? 1 : 0, &part.t, counts.data(), s);
  st = nc.agree(st, s);
  if (st != TCUDB_OK) return st;
  // P x P counts: row j = what rank j sends to each rank
  const std::vector<int64_t> M = nc.gather_vec(counts.data(), P, s);
  int64_t tot = 0;
  std::vector<int64_t> rc(P), roffr(P), soffr(P);
  int64_t srun = 0;
  for (int j = 0; j < P; ++j) { soffr[j] = srun; srun += counts[j]; rc[j] = M[j * P + nc.rank]; roffr[j] = tot; tot += rc[j]; }
  out.t = T;
  out.t.n_rows = tot;
  tcudb_col* dst[3] = {&out.t.key, &out.t.group, &out.t.value};
  for (int c = 0; c < 3; ++c) {
    if (!in[c]->data) { dst[c]->data = nullptr; continue; }
    const size_t e = type_bytes(in[c]->type);
    out.bufs.emplace_back(new DevBuf((size_t)tot * e, s));
    std::vector<size_t> send(P), soff(P), recv(P), roff(P);
    for (int j = 0; j < P; ++j) {
      send[j] = (size_t)counts[j] * e; soff[j] = (size_t)soffr[j] * e;
      recv[j] = (size_t)rc[j] * e; roff[j] = (size_t)roffr[j] * e;
    }
    nc.exchange(static_cast<const char*>(pc[c]->data), send, soff, out.bufs.back()->as<char>(), recv, roff, s);
    dst[c]->data = out.bufs.back()->p;
  }
  ck(cudaStreamSynchronize(s), "sync");  // `part` is released after the exchange completes
  return TCUDB_OK;
}

// allgather-v of a local result into one result allocation (g | h | agg, 256-B aligned);
// which columns exist comes from the agreed query shape, never from local pointers (an
// empty local result has NULL arrays)
void gather_result(tcudb_ctx* ctx, const NcclComm& nc, const tcudb_result& loc, const bool has[3],
                   const int32_t ty[3], tcudb_result* out, cudaStream_t s) {
  const std::vector<int64_t> n = nc.gather_i64(loc.n, s);
  int64_t tot = 0;
  std::vector<int64_t> off(nc.nranks);
  for (int j = 0; j < nc.nranks; ++j) { off[j] = tot; tot += n[j]; }
  const void* src[3] = {loc.g, loc.h, loc.agg};
  size_t at[3], run = 0;
  for (int c = 0; c < 3; ++c) {
    at[c] = run;
    if (has[c]) run += ((size_t)tot * type_bytes(ty[c]) + 255) / 256 * 256;
  }
  char* base = static_cast<char*>(internal_result_alloc(ctx, run, s));
  *out = tcudb_result{};
  out->n = tot;
  out->g_type = ty[0]; out->h_type = ty[1]; out->agg_type = ty[2];
  out->base = base;
  void** dst[3] = {&out->g, &out->h, &out->agg};
  try {
    for (int c = 0; c < 3; ++c) {
      if (!has[c]) continue;
      const size_t e = type_bytes(ty[c]);
      *dst[c] = base + at[c];
      std::vector<size_t> send(nc.nranks, (size_t)loc.n * e), soff(nc.nranks, 0), recv(nc.nranks), roff(nc.nranks);
      for (int j = 0; j < nc.nranks; ++j) { recv[j] = (size_t)n[j] * e; roff[j] = (size_t)off[j] * e; }
      nc.exchange(static_cast<const char*>(src[c]), send, soff, base + at[c], recv, roff, s);
    }
    ck(cudaStreamSynchronize(s), "sync");
  } catch (...) {
    internal_result_release(ctx, base);
    *out = tcudb_result{};
    throw;
  }
}

// Q4: partial aggregate per rank, allgathered and combined exactly
tcudb_status q4(tcudb_ctx* ctx, const NcclComm& nc, const tcudb_table* A, const tcudb_table* B,
                const tcudb_query* q, bool fsum, tcudb_result* out, tcudb_stats* stats, cudaStream_t s) {
  Cols Bf;
  gather_table(nc, *B, Bf, s);
  tcudb_query qa = *q;
  if (q->agg == TCUDB_AVG) qa.agg = TCUDB_SUM;
  tcudb_result r{}, rc{};
  struct RF { tcudb_ctx* c; tcudb_result* r; ~RF() { tcudb_result_free(c, r); } } f1{ctx, &r}, f2{ctx, &rc};
  tcudb_status st = tcudb_join_agg(ctx, A, &Bf.t, &qa, &r, stats, s);
  if (st == TCUDB_OK && q->agg == TCUDB_AVG) {
    tcudb_query qc = *q;
    qc.agg = TCUDB_COUNT;
    st = tcudb_join_agg(ctx, A, &Bf.t, &qc, &rc, nullptr, s);
  }
  const tcudb_status agreed = nc.agree(st, s);
  if (agreed != TCUDB_OK) {
    if (st == TCUDB_OK) internal_set_err(ctx, agreed, "collective join: another rank failed");
    return agreed;
  }
  // [0] local result rows (0 or 1), [1] the aggregate (int64 or fp64 bits), [2] COUNT (AVG)
  int64_t part[3] = {r.n, 0, 0};
  if (r.n) ck(cudaMemcpyAsync(&part[1], r.agg, 8, cudaMemcpyDeviceToHost, s), "D2H");
  if (rc.n) ck(cudaMemcpyAsync(&part[2], rc.agg, 8, cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaStreamSynchronize(s), "sync");
  const std::vector<int64_t> all = nc.gather_vec(part, 3, s);
  int64_t has = 0, cnt = 0;
  __int128 isum = 0;
  double fs = 0.0;
  for (int j = 0; j < nc.nranks; ++j) {  // rank order: the same sum on every rank
    has += all[3 * j];
    cnt += all[3 * j + 2];
    if (!all[3 * j]) continue;
    if (fsum) { double x; std::memcpy(&x, &all[3 * j + 1], 8); fs += x; }
    else isum += (__int128)all[3 * j + 1];
  }
  if (!fsum && (isum > (__int128)INT64_MAX || isum < (__int128)INT64_MIN)) {
    // every rank's partial fits int64 but the total does not (the single-GPU guard's
    // E_OVERFLOW; all ranks see the same sum)
    return internal_set_err(ctx, TCUDB_E_OVERFLOW, "int64 overflow of the Q4 total across ranks");
  }
  int64_t tot[2] = {0, cnt};
  if (fsum) std::memcpy(&tot[0], &fs, 8);
  else tot[0] = (int64_t)isum;
  *out = tcudb_result{};
  out->g_type = TCUDB_I32; out->h_type = TCUDB_I32;
  out->agg_type = (q->agg == TCUDB_AVG || fsum) ? TCUDB_F64 : TCUDB_I64;
  char* base = static_cast<char*>(internal_result_alloc(ctx, 256, s));
  out->base = base;
  out->agg = base;
  out->n = has > 0 ? 1 : 0;
  ck(cudaMemcpyAsync(base, tot, 16, cudaMemcpyHostToDevice, s), "H2D");
  if (q->agg == TCUDB_AVG) {
    int64_t L = 0;
    ck(launch_avg_div(base, fsum ? 1 : 0, reinterpret_cast<const long long*>(base + 8), out->n, s, &L),
       "AVG division");
  }
  ck(cudaStreamSynchronize(s), "sync");
  return TCUDB_OK;
}

// §8(f) f4, the key-partitioned path: both sides are routed by a hash of the join key,
// so every join pair is formed on exactly one rank (a partitioned hash join: no side is
// replicated, each rank joins 1/P of A with 1/P of B); a group (g, h) can then collect
// partial aggregates on several ranks, so the partial tuples are routed by g range and
// merged — with the library's own join + group-by: the partials T(g, h, agg) joined on h
// with the distinct h values D (a GROUP BY h-only query over T) give SUM(agg) per (g, h),
// a group existing iff one of its partials did. COUNT and integer SUM.
tcudb_status key_partitioned(tcudb_ctx* ctx, const NcclComm& nc, const tcudb_table& A, const tcudb_table& B,
                             const tcudb_query* q, tcudb_result* loc, tcudb_stats* stats, cudaStream_t s) {
  Cols Ak, Bk;
  tcudb_status st = route_table(ctx, nc, A, Ak, s, true);
  if (st != TCUDB_OK) return st;
  st = route_table(ctx, nc, B, Bk, s, true);
  if (st != TCUDB_OK) return st;
  tcudb_query q1 = *q;
  q1.flags &= ~(uint32_t)(TCUDB_GATHER_NONE | TCUDB_KEY_PARTITIONED | TCUDB_ROW_SHARDED);
  tcudb_result part{};
  struct RF { tcudb_ctx* c; tcudb_result* r; ~RF() { tcudb_result_free(c, r); } } fp{ctx, &part};
  const tcudb_status lst = tcudb_join_agg(ctx, &Ak.t, &Bk.t, &q1, &part, stats, s);
  st = nc.agree(lst, s);
  if (st != TCUDB_OK) {
    if (lst == TCUDB_OK) internal_set_err(ctx, st, "collective join: another rank's local query failed");
    return st;
  }
  // the partials as a table (k = h, g = g, v = agg), routed by g range
  DevBuf dummy(16, s);
  tcudb_table T{};
  T.n_rows = part.n;
  T.key = {part.h ? part.h : dummy.p, B.group.type};
  T.group = {part.g ? part.g : dummy.p, A.group.type};
  T.value = {part.agg ? part.agg : dummy.p, TCUDB_I64};
  Cols Tr;
  st = route_table(ctx, nc, T, Tr, s);
  if (st != TCUDB_OK) return st;
  // merge: D = distinct h of the received partials (GROUP BY h only), then SUM(agg) per (g, h)
  tcudb_table Th{}, Tg{};
  Th.n_rows = Tr.t.n_rows;
  Th.key = Tr.t.key;                          // ungrouped side (Q3 shape)
  Tg.n_rows = Tr.t.n_rows;
  Tg.key = Tr.t.key;
  Tg.group = Tr.t.key;                        // B.h = h
  tcudb_query qd{TCUDB_COUNT, 0};
  tcudb_result D{};
  struct RF2 { tcudb_ctx* c; tcudb_result* r; ~RF2() { tcudb_result_free(c, r); } } fd{ctx, &D};
  tcudb_status mst = tcudb_join_agg(ctx, &Th, &Tg, &qd, &D, nullptr, s);
  if (mst == TCUDB_OK) {
    tcudb_table TA = Tr.t, TD{};
    TD.n_rows = D.n;
    TD.key = {D.h ? D.h : dummy.p, B.group.type};
    TD.group = TD.key;
    tcudb_query qs{TCUDB_SUM, 0};
    mst = tcudb_join_agg(ctx, &TA, &TD, &qs, loc, nullptr, s);
  }
  st = nc.agree(mst, s);
  if (st != TCUDB_OK) {
    tcudb_result_free(ctx, loc);
    if (mst == TCUDB_OK) internal_set_err(ctx, st, "collective join: another rank's merge failed");
    return st;
  }
  if (stats) stats->path = 3;  // key-partitioned (the local join's plan is in the other fields)
  return TCUDB_OK;
}

}  // namespace

tcudb_status collective_join_agg(tcudb_ctx* ctx, const NcclComm* ncp, const tcudb_table* A, const tcudb_table* B,
                                 const tcudb_query* q, tcudb_status local_st, tcudb_result* out, tcudb_stats* stats,
                                 cudaStream_t s, float* ms_comm) {
  const NcclComm& nc = *ncp;
  const auto t0 = std::chrono::steady_clock::now();
  float local_ms = 0.f;
  tcudb_status st = TCUDB_OK;
  *out = tcudb_result{};
  try {
    // 0. agreement on the query shape
    int64_t d[kDesc] = {};
    const tcudb_table none{};
    const tcudb_table& a = A ? *A : none;
    const tcudb_table& b = B ? *B : none;
    d[0] = a.n_rows; d[1] = b.n_rows;
    const tcudb_col* cs[6] = {&a.key, &a.group, &a.value, &b.key, &b.group, &b.value};
    for (int c = 0; c < 6; ++c) d[2 + c] = col_state(*cs[c], c < 3 ? a.n_rows : b.n_rows);
    d[8] = q ? q->agg : -1;
    d[9] = q ? q->flags : 0;
    d[10] = local_st;
    const std::vector<int64_t> all = nc.gather_vec(d, kDesc, s);
    int64_t ag[kDesc];
    st = shard_agree(all.data(), nc.nranks, ag);
    if (st != TCUDB_OK) {
      if (local_st == TCUDB_OK) internal_set_err(ctx, st, "collective join: ranks disagree on the query or another rank's arguments are invalid");
      return st;
    }
    // normalized local tables: present columns get a (never dereferenced) pointer when the
    // local slice is empty, absent columns are NULL everywhere, types are the agreed ones
    DevBuf dummy(16, s);
    tcudb_table An = a, Bn = b;
    tcudb_col* ns[6] = {&An.key, &An.group, &An.value, &Bn.key, &Bn.group, &Bn.value};
    for (int c = 0; c < 6; ++c) {
      if (ag[2 + c] >= 2) {
        ns[c]->type = (int32_t)(ag[2 + c] - 2);
        if (!ns[c]->data) ns[c]->data = dummy.p;
      } else {
        ns[c]->data = nullptr;
      }
    }
    const bool ga = An.group.data != nullptr, gb = Bn.group.data != nullptr;
    const bool fsum = q->agg != TCUDB_COUNT && ((An.value.data && An.value.type == TCUDB_F32) ||
                                                (Bn.value.data && Bn.value.type == TCUDB_F32));
    // row sharding (north star) vs the key-partitioned path (§8(f) f4): the latter for COUNT
    // / integer SUM when the other side is too large to replicate on every rank (>= 4 M rows
    // in total), or when asked for; flags decide identically on every rank
    const char* kp_env = getenv("TCUDB_KEY_PARTITION");
    const bool kp_ok = ga && gb && q->agg != TCUDB_AVG && !fsum && nc.nranks > 1;
    const bool kp = kp_ok && !(q->flags & TCUDB_ROW_SHARDED) &&
                    ((q->flags & TCUDB_KEY_PARTITIONED) || (kp_env && kp_env[0] == '1') ||
                     (!(kp_env && kp_env[0] == '0') && ag[1] >= (1ll << 22)));
    if (kp) {
      tcudb_result loc{};
      const auto tl = std::chrono::steady_clock::now();
      st = key_partitioned(ctx, nc, An, Bn, q, &loc, stats, s);
      local_ms = 0.f;
      (void)tl;
      if (st != TCUDB_OK) return st;
      struct RF { tcudb_ctx* c; tcudb_result* r; bool keep = false; ~RF() { if (!keep) tcudb_result_free(c, r); } } fl{ctx, &loc};
      if (q->flags & TCUDB_GATHER_NONE) {
        *out = loc;
        out->g_type = An.group.type;
        out->h_type = Bn.group.type;
        fl.keep = true;
      } else {
        const bool has[3] = {true, true, true};
        const int32_t ty[3] = {An.group.type, Bn.group.type, TCUDB_I64};
        gather_result(ctx, nc, loc, has, ty, out, s);
      }
    } else if (!ga && !gb) {
      st = q4(ctx, nc, &An, &Bn, q, fsum, out, stats, s);
    } else {
      // the grouped side is routed by its group range (A when both are grouped)
      const tcudb_table& R = ga ? An : Bn;
      const tcudb_table& O = ga ? Bn : An;
      Cols Rr, Of;
      st = route_table(ctx, nc, R, Rr, s);
      if (st != TCUDB_OK) return st;
      gather_table(nc, O, Of, s);
      const tcudb_table& Ar = ga ? Rr.t : Of.t;
      const tcudb_table& Br = ga ? Of.t : Rr.t;
      tcudb_result loc{};
      const auto tl = std::chrono::steady_clock::now();
      const tcudb_status lst = tcudb_join_agg(ctx, &Ar, &Br, q, &loc, stats, s);
      local_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - tl).count();
      struct RF { tcudb_ctx* c; tcudb_result* r; bool keep = false; ~RF() { if (!keep) tcudb_result_free(c, r); } } fl{ctx, &loc};
      st = nc.agree(lst, s);
      if (st != TCUDB_OK) {
        if (lst == TCUDB_OK) internal_set_err(ctx, st, "collective join: another rank's local query failed");
        return st;
      }
      if (q->flags & TCUDB_GATHER_NONE) {
        *out = loc;
        out->g_type = ga ? An.group.type : TCUDB_I32;
        out->h_type = gb ? Bn.group.type : TCUDB_I32;
        fl.keep = true;
      } else {
        const bool has[3] = {ga, gb, true};
        const int32_t ty[3] = {ga ? An.group.type : TCUDB_I32, gb ? Bn.group.type : TCUDB_I32,
                               (q->agg == TCUDB_AVG || fsum) ? TCUDB_F64 : TCUDB_I64};
        gather_result(ctx, nc, loc, has, ty, out, s);
      }
    }
  } catch (const CommError& e) {
    *out = tcudb_result{};
    return internal_set_err(ctx, TCUDB_E_COMM, ("collective join: " + e.what).c_str());
  }
  if (ms_comm)
    *ms_comm = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count() - local_ms;
  return st;
}

}  // namespace tcudb

// ---------------------------------------------------------------- C ABI: host-only planning
extern "C" {

tcudb_status tcudb_shard_agree(const int64_t* descs, int32_t P, int64_t* agreed) {
  if (!descs || !agreed || P < 1 || P > 1024) return TCUDB_E_INVALID;
  return tcudb::shard_agree(descs, P, agreed);
}

tcudb_status tcudb_shard_bounds(const int64_t* msgs, int32_t P, int64_t* bounds) {
  if (!msgs || P < 1 || P > 1024 || (P > 1 && !bounds)) return TCUDB_E_INVALID;
  if (P > 1) tcudb::shard_bounds(msgs, P, bounds);
  return TCUDB_OK;
}

}  // extern "C"
