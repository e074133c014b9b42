// nccl_shim.cpp — TEST INFRASTRUCTURE: an in-process communicator that implements the
// NCCL entry points libtcudb's collective path resolves (collective.cu: ncclCommCount,
// ncclCommUserRank, ncclAllReduce, ncclAllGather, ncclSend, ncclRecv, ncclGroupStart,
// ncclGroupEnd, ncclGetErrorString) for P ranks that are P host threads of ONE process
// sharing one GPU. NCCL itself refuses two ranks on one device; this library lets the
// tests drive the real collective code path (route_table / gather_table / gather_result /
// q4 and every exchange) at P = 2, 4, 8 on a single B200. Selected at tcudb_create by
// TCUDB_NCCL_LIB=<path of this library>.
//
// Semantics (those of NCCL, executed eagerly on the host): point-to-point sends are
// copied out at call time (after the stream's earlier work) into a mailbox per
// (source, destination) pair; a receive takes the next message of its pair, in call order,
// and checks its size. Collectives are numbered per rank; the n-th collective of every
// rank must be the same operation (kind, count, type, reduction) — each rank posts its
// contribution and waits for all P. Inside ncclGroupStart..End the sends run first, then
// the collectives, then the receives (a group is concurrent in NCCL, so any order that
// cannot deadlock is faithful). A mismatch or a wait beyond the timeout breaks the world:
// that call and every later call on it return an error on every rank (the library turns
// it into E_COMM) instead of hanging. Counters record the calls and bytes per rank.
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
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

struct Coll {
  int kind = -1, dtype = -1, redop = -1;
  size_t count = 0;
  std::vector<std::vector<char>> data;
  int have = 0, done = 0;
};

struct World {
  int P;
  double timeout_s;
  std::mutex mu;
  std::condition_variable cv;
  bool broken = false;
  std::string why;
  std::map<std::pair<int, int>, std::deque<std::vector<char>>> mail;  // (src, dst) -> messages
  std::map<long long, Coll> coll;                                     // collective sequence -> slot
  std::vector<long long> seq;                                         // next collective per rank
  std::vector<Comm> comms;
  std::vector<long long> calls, bytes_in;
  explicit World(int p, double t) : P(p), timeout_s(t), seq(p, 0), calls(p, 0), bytes_in(p, 0) {
    comms.resize(p);
    for (int r = 0; r < p; ++r) comms[r] = Comm{this, r};
  }
  void fail_locked(const std::string& w) {
    if (!broken) why = w;
    broken = true;
    cv.notify_all();
  }
  // wait (lock held) until pred() or broken; false on broken / timeout (which breaks)
  template <typename Pred>
  bool wait(std::unique_lock<std::mutex>& lk, Pred pred, const char* what) {
    const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return broken || pred(); });
    if (broken) return false;
    if (!ok) { fail_locked(std::string("timeout waiting for ") + what); return false; }
    return true;
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

void h2d(void* p, const std::vector<char>& h) {
  if (!h.empty()) cudaMemcpy(p, h.data(), h.size(), cudaMemcpyHostToDevice);
}

// the calling rank's operations of one call or group
int run_group(std::vector<Op>& ops) {
  if (ops.empty()) return 0;
  World* w = ops[0].comm->w;
  const int me = ops[0].comm->rank;
  {
    std::unique_lock<std::mutex> lk(w->mu);
    if (w->broken) return kSystemError;
    for (const Op& o : ops) {
      if (o.comm->w != w || o.comm->rank != me) { w->fail_locked("one group spans two communicators"); return kInvalidUsage; }
      if (!dsize(o.dtype)) { w->fail_locked("unsupported data type"); return kInvalidArgument; }
      if ((o.kind == OP_SEND || o.kind == OP_RECV) && (o.peer < 0 || o.peer >= w->P || o.peer == me)) {
        w->fail_locked("point-to-point with an invalid peer");
        return kInvalidArgument;
      }
    }
    w->calls[me] += (long long)ops.size();
  }
  for (const Op& o : ops) cudaStreamSynchronize(o.stream);
  long long in = 0;
  // 1. sends: copied out now (eager)
  for (const Op& o : ops) {
    if (o.kind != OP_SEND) continue;
    std::vector<char> m = d2h(o.src, o.count * dsize(o.dtype));
    std::lock_guard<std::mutex> lk(w->mu);
    w->mail[{me, o.peer}].push_back(std::move(m));
    w->cv.notify_all();
  }
  // 2. collectives, in call order
  for (const Op& o : ops) {
    if (o.kind != OP_ALLREDUCE && o.kind != OP_ALLGATHER) continue;
    const size_t bytes = o.count * dsize(o.dtype);
    std::vector<char> mine = d2h(o.src, bytes);
    std::vector<char> out;
    {
      std::unique_lock<std::mutex> lk(w->mu);
      const long long q = w->seq[me]++;
      Coll& c = w->coll[q];
      if (c.kind < 0) {
        c.kind = o.kind; c.count = o.count; c.dtype = o.dtype; c.redop = o.redop;
        c.data.resize(w->P);
      } else if (c.kind != o.kind || c.count != o.count || c.dtype != o.dtype ||
                 (o.kind == OP_ALLREDUCE && c.redop != o.redop)) {
        w->fail_locked("collective mismatch across ranks");
        return kSystemError;
      }
      c.data[me] = std::move(mine);
      ++c.have;
      w->cv.notify_all();
      if (!w->wait(lk, [&] { return c.have == w->P; }, "a collective")) return kSystemError;
      if (o.kind == OP_ALLGATHER) {
        out.resize(bytes * w->P);
        for (int r = 0; r < w->P; ++r)
          if (bytes) std::memcpy(out.data() + bytes * r, c.data[r].data(), bytes);
      } else {
        out = c.data[0];
        for (int r = 1; r < w->P; ++r)
          if (!reduce_any(out, c.data[r], o.count, o.dtype, o.redop)) {
            w->fail_locked("unsupported reduction");
            return kSystemError;
          }
      }
      if (++c.done == w->P) w->coll.erase(q);
    }
    h2d(o.dst, out);
    in += (long long)out.size();
  }
  // 3. receives: the next message of each (peer, me) pair, in call order
  for (const Op& o : ops) {
    if (o.kind != OP_RECV) continue;
    const size_t bytes = o.count * dsize(o.dtype);
    std::vector<char> m;
    {
      std::unique_lock<std::mutex> lk(w->mu);
      auto& box = w->mail[{o.peer, me}];
      if (!w->wait(lk, [&] { return !box.empty(); }, "a matching send")) return kSystemError;
      m = std::move(box.front());
      box.pop_front();
      if (m.size() != bytes) { w->fail_locked("send / receive sizes differ"); return kSystemError; }
    }
    h2d(o.dst, m);
    in += (long long)m.size();
  }
  {
    std::lock_guard<std::mutex> lk(w->mu);
    w->bytes_in[me] += in;
    if (w->broken) return kSystemError;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int submit(const Op& o) {
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
