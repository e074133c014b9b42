// nccl_shim.cpp — TEST INFRASTRUCTURE: an in-process communicator that implements the
// NCCL entry points libtcudb's collective path resolves (collective.cu: ncclCommCount,
// ncclCommUserRank, ncclAllReduce, ncclAllGather, ncclSend, ncclRecv, ncclGroupStart,
// ncclGroupEnd, ncclGetErrorString) for P ranks that are P host threads of ONE process
// sharing one GPU. NCCL itself refuses two ranks on one device; this library lets the
// tests drive the real collective code path (route_table / gather_table / gather_result /
// q4 and every exchange) at P = 2, 4, 8 on a single B200. Selected at tcudb_create by
// TCUDB_NCCL_LIB=<path of this library>.
//
// Semantics: every call (or ncclGroupStart..ncclGroupEnd block) is one rendezvous of all
// P ranks: each rank synchronizes the streams of its calls, posts its operation list,
// waits for the others (barrier 1), stages what it receives into host memory (sends are
// matched to receives per (source, destination) pair in call order, collectives by
// position; sizes, types and ops must agree), waits (barrier 2), then writes its receive
// buffers. A mismatch or a barrier timeout breaks the world: that call and every later
// call on it return an error on every rank (the library turns it into E_COMM) instead of
// hanging. Counters record the calls and bytes per rank.
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace {

enum OpKind { OP_SEND, OP_RECV, OP_ALLREDUCE, OP_ALLGATHER };
constexpr int kSystemError = 2, kInvalidArgument = 4, kInvalidUsage = 5;

struct World;
struct Comm {
  World* w;
  int rank;
};

struct Op {
  OpKind kind;
  Comm* comm;
  const void* src;
  void* dst;
  size_t count;
  int dtype, redop, peer;
  cudaStream_t stream;
};

struct World {
  int P;
  double timeout_s;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  bool broken = false;
  std::string why;
  std::vector<std::vector<Op>> posted;
  std::vector<Comm> comms;
  std::vector<long long> calls, bytes_in;
  explicit World(int p, double t) : P(p), timeout_s(t), posted(p), calls(p, 0), bytes_in(p, 0) {
    comms.resize(p);
    for (int r = 0; r < p; ++r) comms[r] = Comm{this, r};
  }
  // returns false when the world is (or becomes) broken
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) return false;
    const long long g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return gen != g || broken; });
    if (broken) return false;
    if (!ok) {
      broken = true;
      why = "barrier timeout (a rank did not reach the collective)";
      cv.notify_all();
      return false;
    }
    return true;
  }
  void fail(const std::string& w) {
    std::lock_guard<std::mutex> lk(mu);
    if (!broken) why = w;
    broken = true;
    cv.notify_all();
  }
};

size_t dsize(int t) {
  switch (t) {
    case 0: case 1: return 1;     // int8 / uint8
    case 2: case 3: case 7: return 4;  // int32 / uint32 / float32
    case 4: case 5: case 8: return 8;  // int64 / uint64 / float64
    case 6: case 9: return 2;     // float16 / bfloat16
    default: return 0;
  }
}

thread_local int t_depth = 0;
thread_local std::vector<Op> t_ops;

template <typename T>
void reduce_into(std::vector<char>& acc, const std::vector<char>& x, size_t n, int op) {
  T* a = reinterpret_cast<T*>(acc.data());
  const T* b = reinterpret_cast<const T*>(x.data());
  for (size_t i = 0; i < n; ++i) {
    switch (op) {
      case 0: a[i] = a[i] + b[i]; break;
      case 1: a[i] = a[i] * b[i]; break;
      case 2: a[i] = a[i] > b[i] ? a[i] : b[i]; break;
      case 3: a[i] = a[i] < b[i] ? a[i] : b[i]; break;
      default: break;
    }
  }
}

bool reduce_any(std::vector<char>& acc, const std::vector<char>& x, size_t n, int dtype, int op) {
  switch (dtype) {
    case 2: reduce_into<int32_t>(acc, x, n, op); return true;
    case 3: reduce_into<uint32_t>(acc, x, n, op); return true;
    case 4: reduce_into<int64_t>(acc, x, n, op); return true;
    case 5: reduce_into<uint64_t>(acc, x, n, op); return true;
    case 7: reduce_into<float>(acc, x, n, op); return true;
    case 8: reduce_into<double>(acc, x, n, op); return true;
    default: return false;
  }
}

std::vector<char> d2h(const void* p, size_t bytes) {
  std::vector<char> h(bytes);
  if (bytes) cudaMemcpy(h.data(), p, bytes, cudaMemcpyDeviceToHost);
  return h;
}

// one rendezvous over the calling rank's operation list
int run_group(std::vector<Op>& ops) {
  if (ops.empty()) return 0;
  World* w = ops[0].comm->w;
  const int me = ops[0].comm->rank;
  for (const Op& o : ops) {
    if (o.comm->w != w || o.comm->rank != me) { w->fail("one group spans two communicators"); return kInvalidUsage; }
    if (!dsize(o.dtype)) { w->fail("unsupported data type"); return kInvalidArgument; }
  }
  for (const Op& o : ops) cudaStreamSynchronize(o.stream);
  {
    std::lock_guard<std::mutex> lk(w->mu);
    w->posted[me] = ops;
    w->calls[me] += (long long)ops.size();
  }
  if (!w->barrier()) return kSystemError;
  // stage what this rank receives
  struct Stage { void* dst; std::vector<char> data; };
  std::vector<Stage> stage;
  std::string err;
  std::vector<int> coll_idx(w->P, 0);
  int my_coll = 0;
  for (size_t i = 0; i < ops.size() && err.empty(); ++i) {
    const Op& o = ops[i];
    const size_t bytes = o.count * dsize(o.dtype);
    if (o.kind == OP_SEND) continue;
    if (o.kind == OP_RECV) {
      // k-th receive from peer p matches p's k-th send to me
      int k = 0;
      for (size_t j = 0; j < i; ++j) k += ops[j].kind == OP_RECV && ops[j].peer == o.peer;
      if (o.peer < 0 || o.peer >= w->P) { err = "receive from an invalid peer"; break; }
      const std::vector<Op>& po = w->posted[o.peer];
      const Op* match = nullptr;
      int seen = 0;
      for (const Op& x : po)
        if (x.kind == OP_SEND && x.peer == me && seen++ == k) { match = &x; break; }
      if (!match) { err = "receive without a matching send"; break; }
      if (match->count * dsize(match->dtype) != bytes) { err = "send / receive sizes differ"; break; }
      stage.push_back({o.dst, d2h(match->src, bytes)});
      continue;
    }
    // collective: the my_coll-th collective of every rank must be the same operation
    std::vector<const Op*> peers(w->P, nullptr);
    for (int r = 0; r < w->P; ++r) {
      int seen = 0;
      for (const Op& x : w->posted[r])
        if ((x.kind == OP_ALLREDUCE || x.kind == OP_ALLGATHER) && seen++ == my_coll) { peers[r] = &x; break; }
      if (!peers[r] || peers[r]->kind != o.kind || peers[r]->count != o.count || peers[r]->dtype != o.dtype ||
          (o.kind == OP_ALLREDUCE && peers[r]->redop != o.redop)) {
        err = "collective mismatch across ranks";
        break;
      }
    }
    ++my_coll;
    if (!err.empty()) break;
    if (o.kind == OP_ALLGATHER) {
      std::vector<char> all(bytes * w->P);
      for (int r = 0; r < w->P; ++r) {
        std::vector<char> x = d2h(peers[r]->src, bytes);
        if (bytes) std::memcpy(all.data() + bytes * r, x.data(), bytes);
      }
      stage.push_back({o.dst, std::move(all)});
    } else {
      std::vector<char> acc = d2h(peers[0]->src, bytes);
      for (int r = 1; r < w->P; ++r)
        if (!reduce_any(acc, d2h(peers[r]->src, bytes), o.count, o.dtype, o.redop)) { err = "unsupported reduction"; break; }
      stage.push_back({o.dst, std::move(acc)});
    }
  }
  if (!err.empty()) w->fail(err);
  if (!w->barrier()) return kSystemError;
  long long in = 0;
  for (Stage& st : stage) {
    if (!st.data.empty()) cudaMemcpy(st.dst, st.data.data(), st.data.size(), cudaMemcpyHostToDevice);
    in += (long long)st.data.size();
  }
  {
    std::lock_guard<std::mutex> lk(w->mu);
    w->bytes_in[me] += in;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int submit(const Op& o) {
  if (o.comm->w->broken) return kSystemError;
  if (t_depth > 0) { t_ops.push_back(o); return 0; }
  std::vector<Op> one{o};
  return run_group(one);
}

}  // namespace

extern "C" {

// ---- shim control (test side)
void* shim_world_create(int P, double timeout_s) { return new World(P, timeout_s); }
void* shim_comm(void* w, int rank) { return &static_cast<World*>(w)->comms[rank]; }
void shim_world_destroy(void* w) { delete static_cast<World*>(w); }
int shim_world_broken(void* w) { return static_cast<World*>(w)->broken ? 1 : 0; }
const char* shim_world_why(void* w) { return static_cast<World*>(w)->why.c_str(); }
long long shim_calls(void* w, int rank) { return static_cast<World*>(w)->calls[rank]; }
long long shim_bytes_in(void* w, int rank) { return static_cast<World*>(w)->bytes_in[rank]; }

// ---- the NCCL entry points
int ncclCommCount(void* comm, int* count) {
  *count = static_cast<Comm*>(comm)->w->P;
  return 0;
}
int ncclCommUserRank(void* comm, int* rank) {
  *rank = static_cast<Comm*>(comm)->rank;
  return 0;
}
int ncclAllReduce(const void* send, void* recv, size_t count, int dtype, int op, void* comm, cudaStream_t s) {
  return submit(Op{OP_ALLREDUCE, static_cast<Comm*>(comm), send, recv, count, dtype, op, -1, s});
}
int ncclAllGather(const void* send, void* recv, size_t count, int dtype, void* comm, cudaStream_t s) {
  return submit(Op{OP_ALLGATHER, static_cast<Comm*>(comm), send, recv, count, dtype, 0, -1, s});
}
int ncclSend(const void* send, size_t count, int dtype, int peer, void* comm, cudaStream_t s) {
  return submit(Op{OP_SEND, static_cast<Comm*>(comm), send, nullptr, count, dtype, 0, peer, s});
}
int ncclRecv(void* recv, size_t count, int dtype, int peer, void* comm, cudaStream_t s) {
  return submit(Op{OP_RECV, static_cast<Comm*>(comm), nullptr, recv, count, dtype, 0, peer, s});
}
int ncclGroupStart() {
  ++t_depth;
  return 0;
}
int ncclGroupEnd() {
  if (t_depth <= 0) return kInvalidUsage;
  if (--t_depth > 0) return 0;
  std::vector<Op> ops;
  ops.swap(t_ops);
  if (!ops.empty() && ops[0].comm->w->broken) return kSystemError;
  return run_group(ops);
}
const char* ncclGetErrorString(int r) {
  switch (r) {
    case 0: return "no error (shim)";
    case kSystemError: return "shim: world broken (mismatch or timeout)";
    case kInvalidArgument: return "shim: invalid argument";
    case kInvalidUsage: return "shim: invalid usage";
    default: return "shim: CUDA error";
  }
}

}  // extern "C"
