// collective.cu — the multi-GPU form of tcudb_join_agg (SURVEY §8(b) "Multi-GPU" and
// §8(e)): when the context was created with an NCCL communicator, every rank passes its
// local slices of A and B and the call is collective.
//
// Output rows are independent units (§3.2: C[g][h] depends only on A's rows of
// group g and B's rows of group h), so they are sharded by ranges of the grouped side's
// group key and the only exchanges are data movement:
//   1. global [min, max] of the routed side's group column (two allreduces) -> P
//      equal-width ranges, rank r owning the r-th;
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
// B and the per-rank partial aggregates are combined with allreduces (AVG = the reduced
// SUM / the reduced COUNT, divided on the device).
//
// NCCL is resolved at context creation with dlopen (the process's already-loaded
// libnccl.so.2 — torch's — first), so a library used without a communicator has no NCCL
// dependency. The communicator is owned by the caller.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <chrono>
#include <memory>
#include <type_traits>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tcudb.h"
#include "internal.h"
#include "kernels.h"

namespace tcudb {
namespace {

// NCCL's stable ABI values (nccl.h): data types and reduction ops used here
constexpr int kNcclInt8 = 0, kNcclInt64 = 4, kNcclFloat64 = 8;
constexpr int kNcclSum = 0, kNcclMax = 2, kNcclMin = 3;

struct CommError {
  std::string what;
};

struct DevBuf {  // stream-ordered device buffer
  void* p = nullptr;
  cudaStream_t s;
  DevBuf(size_t bytes, cudaStream_t st) : s(st) {
    if (cudaMallocAsync(&p, bytes ? bytes : 8, s) != cudaSuccess) {
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
  // allgather of one int64 per rank, read back on the host
  std::vector<int64_t> gather_i64(int64_t x, cudaStream_t s) const {
    DevBuf d(sizeof(int64_t) * (nranks + 1), s);
    ck(cudaMemcpyAsync(d.as<int64_t>() + nranks, &x, sizeof(int64_t), cudaMemcpyHostToDevice, s), "H2D");
    nck(AllGather(d.as<int64_t>() + nranks, d.as<int64_t>(), 1, kNcclInt64, comm, s), "ncclAllGather");
    std::vector<int64_t> h(nranks);
    ck(cudaMemcpyAsync(h.data(), d.p, sizeof(int64_t) * nranks, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
    return h;
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
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (torch's)
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { *err = "libnccl.so.2 not found"; return nullptr; }
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

namespace {

// P-1 ascending bounds splitting [lo, hi] into P equal-width ranges (exact in 128 bits)
std::vector<int64_t> range_bounds(int64_t lo, int64_t hi, int P) {
  std::vector<int64_t> b(P > 1 ? P - 1 : 0, 0);
  if (lo > hi) return b;
  const __int128 span = (__int128)hi - lo + 1;
  for (int i = 1; i < P; ++i) b[i - 1] = (int64_t)(lo + span * i / P);
  return b;
}

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
    if (!in[c]->data) continue;
    const size_t e = type_bytes(in[c]->type);
    out.bufs.emplace_back(new DevBuf((size_t)tot * e, s));
    std::vector<size_t> send(nc.nranks, (size_t)T.n_rows * e), soff(nc.nranks, 0), recv(nc.nranks), roff(nc.nranks);
    for (int j = 0; j < nc.nranks; ++j) { recv[j] = (size_t)n[j] * e; roff[j] = (size_t)off[j] * e; }
    nc.exchange(static_cast<const char*>(in[c]->data), send, soff, out.bufs.back()->as<char>(), recv, roff, s);
    dst[c]->data = out.bufs.back()->p;
  }
}

// route the rows of T to the rank owning their group range
tcudb_status route_table(tcudb_ctx* ctx, const NcclComm& nc, const tcudb_table& T, Cols& out, cudaStream_t s) {
  const int P = nc.nranks;
  int64_t mn, mx;
  tcudb_status st = tcudb_minmax(ctx, T.group.data, T.group.type, T.n_rows, &mn, &mx, s);
  if (st != TCUDB_OK) return st;
  DevBuf r(16, s);
  const int64_t h2[2] = {mn, mx};
  ck(cudaMemcpyAsync(r.p, h2, 16, cudaMemcpyHostToDevice, s), "H2D");
  nc.nck(nc.GroupStart(), "ncclGroupStart");
  nc.nck(nc.AllReduce(r.as<int64_t>(), r.as<int64_t>(), 1, kNcclInt64, kNcclMin, nc.comm, s), "ncclAllReduce");
  nc.nck(nc.AllReduce(r.as<int64_t>() + 1, r.as<int64_t>() + 1, 1, kNcclInt64, kNcclMax, nc.comm, s),
         "ncclAllReduce");
  nc.nck(nc.GroupEnd(), "ncclGroupEnd");
  int64_t g2[2];
  ck(cudaMemcpyAsync(g2, r.p, 16, cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaStreamSynchronize(s), "sync");
  const std::vector<int64_t> bounds = range_bounds(g2[0], g2[1], P);
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
  st = tcudb_partition(ctx, &T, bounds.data(), P, &part.t, counts.data(), s);
  if (st != TCUDB_OK) return st;
  // P x P counts: row j = what rank j sends to each rank
  std::vector<int64_t> M(P * P);
  {
    DevBuf d(sizeof(int64_t) * P * (P + 1), s);
    ck(cudaMemcpyAsync(d.as<int64_t>() + P * P, counts.data(), sizeof(int64_t) * P, cudaMemcpyHostToDevice, s),
       "H2D");
    nc.nck(nc.AllGather(d.as<int64_t>() + P * P, d.as<int64_t>(), P, kNcclInt64, nc.comm, s), "ncclAllGather");
    ck(cudaMemcpyAsync(M.data(), d.p, sizeof(int64_t) * P * P, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "sync");
  }
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

// allgather-v of a local result into one result allocation (g | h | agg, 256-B aligned)
void gather_result(tcudb_ctx* ctx, const NcclComm& nc, const tcudb_result& loc, tcudb_result* out, cudaStream_t s) {
  const std::vector<int64_t> n = nc.gather_i64(loc.n, s);
  int64_t tot = 0;
  std::vector<int64_t> off(nc.nranks);
  for (int j = 0; j < nc.nranks; ++j) { off[j] = tot; tot += n[j]; }
  void* src[3] = {loc.g, loc.h, loc.agg};
  const int32_t ty[3] = {loc.g_type, loc.h_type, loc.agg_type};
  size_t at[3], run = 0;
  for (int c = 0; c < 3; ++c) {
    at[c] = run;
    if (src[c] || c == 2) run += ((size_t)tot * type_bytes(ty[c]) + 255) / 256 * 256;
  }
  char* base = static_cast<char*>(internal_result_alloc(ctx, run, s));
  *out = tcudb_result{};
  out->n = tot;
  out->g_type = loc.g_type; out->h_type = loc.h_type; out->agg_type = loc.agg_type;
  out->base = base;
  void** dst[3] = {&out->g, &out->h, &out->agg};
  try {
    for (int c = 0; c < 3; ++c) {
      if (!src[c] && c != 2) continue;
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

// Q4: partial aggregate per rank, combined with allreduces
tcudb_status q4(tcudb_ctx* ctx, const NcclComm& nc, const tcudb_table* A, const tcudb_table* B,
                const tcudb_query* q, tcudb_result* out, tcudb_stats* stats, cudaStream_t s) {
  Cols Bf;
  gather_table(nc, *B, Bf, s);
  const bool fsum = q->agg != TCUDB_COUNT && ((A->value.data && A->value.type == TCUDB_F32) ||
                                              (B->value.data && B->value.type == TCUDB_F32));
  tcudb_query qa = *q;
  if (q->agg == TCUDB_AVG) qa.agg = TCUDB_SUM;
  tcudb_result r{}, rc{};
  tcudb_status st = tcudb_join_agg(ctx, A, &Bf.t, &qa, &r, stats, s);
  if (st != TCUDB_OK) return st;
  struct RF { tcudb_ctx* c; tcudb_result* r; ~RF() { tcudb_result_free(c, r); } } f1{ctx, &r}, f2{ctx, &rc};
  if (q->agg == TCUDB_AVG) {
    tcudb_query qc = *q;
    qc.agg = TCUDB_COUNT;
    st = tcudb_join_agg(ctx, A, &Bf.t, &qc, &rc, nullptr, s);
    if (st != TCUDB_OK) return st;
  }
  // [0] rows present, [1] the aggregate (int64 or fp64 bits), [2] COUNT (AVG)
  DevBuf d(24, s);
  ck(cudaMemsetAsync(d.p, 0, 24, s), "memset");
  const int64_t has = r.n;
  ck(cudaMemcpyAsync(d.p, &has, 8, cudaMemcpyHostToDevice, s), "H2D");
  if (r.n) ck(cudaMemcpyAsync(d.as<char>() + 8, r.agg, 8, cudaMemcpyDeviceToDevice, s), "D2D");
  if (rc.n) ck(cudaMemcpyAsync(d.as<char>() + 16, rc.agg, 8, cudaMemcpyDeviceToDevice, s), "D2D");
  nc.nck(nc.GroupStart(), "ncclGroupStart");
  nc.nck(nc.AllReduce(d.p, d.p, 1, kNcclInt64, kNcclSum, nc.comm, s), "ncclAllReduce");
  nc.nck(nc.AllReduce(d.as<char>() + 8, d.as<char>() + 8, 1, fsum ? kNcclFloat64 : kNcclInt64, kNcclSum, nc.comm, s),
         "ncclAllReduce");
  nc.nck(nc.AllReduce(d.as<char>() + 16, d.as<char>() + 16, 1, kNcclInt64, kNcclSum, nc.comm, s), "ncclAllReduce");
  nc.nck(nc.GroupEnd(), "ncclGroupEnd");
  int64_t tot_has = 0;
  ck(cudaMemcpyAsync(&tot_has, d.p, 8, cudaMemcpyDeviceToHost, s), "D2H");
  ck(cudaStreamSynchronize(s), "sync");
  *out = tcudb_result{};
  out->g_type = TCUDB_I32; out->h_type = TCUDB_I32;
  out->agg_type = (q->agg == TCUDB_AVG || fsum) ? TCUDB_F64 : TCUDB_I64;
  char* base = static_cast<char*>(internal_result_alloc(ctx, 256, s));
  out->base = base;
  out->agg = base;
  out->n = tot_has > 0 ? 1 : 0;
  ck(cudaMemcpyAsync(base, d.as<char>() + 8, 8, cudaMemcpyDeviceToDevice, s), "D2D");
  if (q->agg == TCUDB_AVG) {
    int64_t L = 0;
    ck(launch_avg_div(base, fsum ? 1 : 0, reinterpret_cast<const long long*>(d.as<char>() + 16), out->n, s, &L),
       "AVG division");
  }
  ck(cudaStreamSynchronize(s), "sync");
  return TCUDB_OK;
}

}  // namespace

tcudb_status collective_join_agg(tcudb_ctx* ctx, const NcclComm* ncp, const tcudb_table* A, const tcudb_table* B,
                                 const tcudb_query* q, tcudb_result* out, tcudb_stats* stats, cudaStream_t s,
                                 float* ms_comm) {
  const NcclComm& nc = *ncp;
  const auto t0 = std::chrono::steady_clock::now();
  float local_ms = 0.f;
  tcudb_status st = TCUDB_OK;
  try {
    const bool ga = A->group.data != nullptr, gb = B->group.data != nullptr;
    if (!ga && !gb) {
      st = q4(ctx, nc, A, B, q, out, stats, s);
    } else {
      // the grouped side is routed by its group range (A when both are grouped)
      const tcudb_table& R = ga ? *A : *B;
      const tcudb_table& O = ga ? *B : *A;
      Cols Rr, Of;
      st = route_table(ctx, nc, R, Rr, s);
      if (st != TCUDB_OK) return st;
      gather_table(nc, O, Of, s);
      const tcudb_table& Ar = ga ? Rr.t : Of.t;
      const tcudb_table& Br = ga ? Of.t : Rr.t;
      tcudb_result loc{};
      const auto tl = std::chrono::steady_clock::now();
      st = tcudb_join_agg(ctx, &Ar, &Br, q, &loc, stats, s);
      local_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - tl).count();
      if (st != TCUDB_OK) return st;
      if (q->flags & TCUDB_GATHER_NONE) {
        *out = loc;
      } else {
        struct RF { tcudb_ctx* c; tcudb_result* r; ~RF() { tcudb_result_free(c, r); } } fl{ctx, &loc};
        gather_result(ctx, nc, loc, out, s);
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
