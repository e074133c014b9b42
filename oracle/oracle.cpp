// oracle.cpp — CPU oracle for the TCUDB join + group-by hot path.
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library. The product path
// (paper_2112_07552_b200/) never links, imports or calls it, and it shares no
// code with the CUDA path.
//
// What it computes is the plain definition of the query result,
// written as a textbook hash join followed by hash aggregation — no matrices:
//
//   SELECT A.g, B.h, SUM(A.v*B.w)  -- or COUNT(*)
//   FROM A JOIN B ON A.k = B.k GROUP BY A.g, B.h
//
//   PAPER.md Fig. 4: "a list of triples ... with unique
//     combinations ... the val in each triple is the sum of the pairwise
//     multiplications on val fields from a record in table A with its row_num
//     matching another record's col_num from table B".
//   PAPER.md §3.1: (a_i, b_j) is in the join iff C_ij > 0 — i.e. the
//     join is the set of matching pairs, with multiplicity (bag semantics).
//   PAPER.md §3.3: SUM and COUNT ("set mat(A)_ij to 1") aggregates.
//
// For each group (g,h): S_gh = {(i,j) : A.k[i]=B.k[j], A.g[i]=g, B.h[j]=h}.
// The result holds (g, h, agg) for every S_gh != {} (existence = COUNT > 0;
// DESIGN.md reading R3), sorted ascending by (g, h) (reading R2).
//   COUNT: |S_gh|                    (exact, int64)
//   SUM int:   sum of A.v*B.w        (__int128 accumulation; overflow flagged)
//   SUM float: sum of (double)v*(double)w  (fp32 inputs -> exact fp64 products,
//              fp64 sums) plus S_abs = sum |v*w| for the floored tolerance.
//
// Pinned by tests/test_oracle.py against nested-loop brute force, closed forms
// (COUNT total = sum_k cntA(k)*cntB(k); Q4 total = sum_k SA(k)*SB(k)), the
// SPEC.md worked examples (tests/golden/) and textbook graph counts.

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <unordered_map>
#include <vector>
#include <omp.h>

extern "C" {

// value column kinds
enum { ORACLE_V_NONE = 0, ORACLE_V_INT64 = 1, ORACLE_V_F32 = 2 };
enum { ORACLE_COUNT = 0, ORACLE_SUM = 1 };
enum { ORACLE_OK = 0, ORACLE_OVERFLOW = 1, ORACLE_INVALID = -1 };

typedef struct {
  int64_t n;          // number of result groups
  int64_t* g;         // [n] A.g value
  int64_t* h;         // [n] B.h value
  int64_t* cnt;       // [n] |S_gh| (always filled)
  int64_t* isum;      // [n] integer SUM (agg=SUM with integer values), else NULL
  double* fsum;       // [n] float SUM (agg=SUM with a float value column), else NULL
  double* fabs_sum;   // [n] sum |v*w| (float SUM only), else NULL
} oracle_result;

}  // extern "C"

namespace {

struct Bucket { int64_t begin, end; };

struct Entry { int64_t hid; int64_t wi; double wf; };

inline bool fits_i64(__int128 x) {
  return x >= (__int128)INT64_MIN && x <= (__int128)INT64_MAX;
}

}  // namespace

extern "C" int oracle_join_agg(int64_t nA, const int64_t* ak, const int64_t* ag, const void* av, int av_kind,
                               int64_t nB, const int64_t* bk, const int64_t* bh, const void* bw, int bw_kind,
                               int agg, int nthreads, oracle_result* out) {
  if (!out || nA < 0 || nB < 0) return ORACLE_INVALID;
  std::memset(out, 0, sizeof(*out));
  if (agg != ORACLE_COUNT && agg != ORACLE_SUM) return ORACLE_INVALID;
  const bool is_float = (av_kind == ORACLE_V_F32 || bw_kind == ORACLE_V_F32);
  if (is_float && (av_kind == ORACLE_V_INT64 || bw_kind == ORACLE_V_INT64)) return ORACLE_INVALID;
  if (nthreads > 0) omp_set_num_threads(nthreads);

  // ---- 1. Build side: B bucketed by join key (hash join build, "build hash tables").
  std::vector<int64_t> bh_sorted(bh, bh + nB);
  std::sort(bh_sorted.begin(), bh_sorted.end());
  bh_sorted.erase(std::unique(bh_sorted.begin(), bh_sorted.end()), bh_sorted.end());
  const int64_t H = (int64_t)bh_sorted.size();

  std::vector<int64_t> border(nB);
  for (int64_t j = 0; j < nB; ++j) border[j] = j;
  std::stable_sort(border.begin(), border.end(), [&](int64_t x, int64_t y) { return bk[x] < bk[y]; });
  std::vector<Entry> entries(nB);
  std::unordered_map<int64_t, Bucket> table;
  table.reserve((size_t)nB * 2 + 1);
  for (int64_t p = 0; p < nB; ++p) {
    const int64_t j = border[p];
    Entry e;
    e.hid = std::lower_bound(bh_sorted.begin(), bh_sorted.end(), bh[j]) - bh_sorted.begin();
    e.wi = (bw_kind == ORACLE_V_INT64) ? ((const int64_t*)bw)[j] : 1;
    e.wf = (bw_kind == ORACLE_V_F32) ? (double)((const float*)bw)[j] : 1.0;
    entries[p] = e;
    auto it = table.find(bk[j]);
    if (it == table.end()) table.emplace(bk[j], Bucket{p, p + 1});
    else it->second.end = p + 1;
  }

  // ---- 2. Probe side grouped by A.g (hash aggregation partitioned by g: each
  //         thread owns whole g values, so no two threads touch one group).
  std::vector<int64_t> aorder(nA);
  for (int64_t i = 0; i < nA; ++i) aorder[i] = i;
  std::stable_sort(aorder.begin(), aorder.end(), [&](int64_t x, int64_t y) { return ag[x] < ag[y]; });
  std::vector<int64_t> gstart;  // start offsets of each distinct g run in aorder
  for (int64_t p = 0; p < nA; ++p)
    if (p == 0 || ag[aorder[p]] != ag[aorder[p - 1]]) gstart.push_back(p);
  const int64_t G = (int64_t)gstart.size();
  gstart.push_back(nA);

  struct Row { int64_t h; int64_t cnt; __int128 isum; double fsum, fabs; };
  std::vector<std::vector<Row>> per_g(G);
  int overflow = 0;

#pragma omp parallel reduction(| : overflow)
  {
    // Per-thread accumulator over the h dictionary (a dense "SPA" row), used
    // as the hash table of the aggregation for one g at a time.
    std::vector<int64_t> cnt(H, 0);
    std::vector<__int128> isum(agg == ORACLE_SUM && !is_float ? H : 0);
    std::vector<double> fsum(agg == ORACLE_SUM && is_float ? H : 0);
    std::vector<double> fabs_(agg == ORACLE_SUM && is_float ? H : 0);
    std::vector<int64_t> touched;
#pragma omp for schedule(dynamic, 1)
    for (int64_t gi = 0; gi < G; ++gi) {
      touched.clear();
      for (int64_t p = gstart[gi]; p < gstart[gi + 1]; ++p) {
        const int64_t i = aorder[p];
        auto it = table.find(ak[i]);
        if (it == table.end()) continue;
        const int64_t vi = (av_kind == ORACLE_V_INT64) ? ((const int64_t*)av)[i] : 1;
        const double vf = (av_kind == ORACLE_V_F32) ? (double)((const float*)av)[i] : 1.0;
        for (int64_t q = it->second.begin; q < it->second.end; ++q) {
          const Entry& e = entries[q];
          if (cnt[e.hid] == 0) touched.push_back(e.hid);
          cnt[e.hid] += 1;
          if (agg == ORACLE_SUM) {
            if (is_float) {
              const double prod = vf * e.wf;  // exact: 24-bit x 24-bit significands
              fsum[e.hid] += prod;
              fabs_[e.hid] += prod < 0 ? -prod : prod;
            } else {
              isum[e.hid] += (__int128)vi * (__int128)e.wi;
            }
          }
        }
      }
      std::sort(touched.begin(), touched.end());
      std::vector<Row>& rows = per_g[gi];
      rows.reserve(touched.size());
      for (int64_t hid : touched) {
        Row r;
        r.h = bh_sorted[hid];
        r.cnt = cnt[hid];
        r.isum = 0; r.fsum = 0; r.fabs = 0;
        if (agg == ORACLE_SUM) {
          if (is_float) { r.fsum = fsum[hid]; r.fabs = fabs_[hid]; fsum[hid] = 0; fabs_[hid] = 0; }
          else { r.isum = isum[hid]; isum[hid] = 0; if (!fits_i64(r.isum)) overflow = 1; }
        }
        cnt[hid] = 0;
        rows.push_back(r);
      }
    }
  }

  // ---- 3. Emit in (g, h) order: g runs are ascending, h sorted within each run.
  int64_t n = 0;
  for (auto& v : per_g) n += (int64_t)v.size();
  out->n = n;
  out->g = (int64_t*)std::malloc(sizeof(int64_t) * (n ? n : 1));
  out->h = (int64_t*)std::malloc(sizeof(int64_t) * (n ? n : 1));
  out->cnt = (int64_t*)std::malloc(sizeof(int64_t) * (n ? n : 1));
  if (agg == ORACLE_SUM && !is_float) out->isum = (int64_t*)std::malloc(sizeof(int64_t) * (n ? n : 1));
  if (agg == ORACLE_SUM && is_float) {
    out->fsum = (double*)std::malloc(sizeof(double) * (n ? n : 1));
    out->fabs_sum = (double*)std::malloc(sizeof(double) * (n ? n : 1));
  }
  int64_t o = 0;
  for (int64_t gi = 0; gi < G; ++gi) {
    const int64_t gval = ag[aorder[gstart[gi]]];
    for (const Row& r : per_g[gi]) {
      out->g[o] = gval;
      out->h[o] = r.h;
      out->cnt[o] = r.cnt;
      if (out->isum) out->isum[o] = (int64_t)r.isum;
      if (out->fsum) { out->fsum[o] = r.fsum; out->fabs_sum[o] = r.fabs; }
      ++o;
    }
  }
  return overflow ? ORACLE_OVERFLOW : ORACLE_OK;
}

extern "C" void oracle_free(oracle_result* r) {
  if (!r) return;
  std::free(r->g); std::free(r->h); std::free(r->cnt);
  std::free(r->isum); std::free(r->fsum); std::free(r->fabs_sum);
  std::memset(r, 0, sizeof(*r));
}

// Triangle count of the simple undirected graph given by an edge list
// (self-loops dropped, direction and duplicates ignored) — SURVEY §8(a) a9 and
// reading R15. Plain node iterator: every triangle u<v<w is counted once, at
// its smallest edge (u,v), as a common neighbour w > v of u and v.
// (§3.2 P:751-756 casts this 3-way self-join as a matrix chain.)
extern "C" int64_t oracle_triangles(int64_t n_edges, const int64_t* src, const int64_t* dst, int nthreads) {
  if (nthreads > 0) omp_set_num_threads(nthreads);
  std::vector<int64_t> ids;
  ids.reserve(2 * n_edges);
  for (int64_t e = 0; e < n_edges; ++e) { ids.push_back(src[e]); ids.push_back(dst[e]); }
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  const int64_t V = (int64_t)ids.size();
  auto id_of = [&](int64_t x) { return std::lower_bound(ids.begin(), ids.end(), x) - ids.begin(); };
  std::vector<std::vector<int64_t>> adj(V);
  for (int64_t e = 0; e < n_edges; ++e) {
    const int64_t u = id_of(src[e]), v = id_of(dst[e]);
    if (u == v) continue;
    adj[u].push_back(v);
    adj[v].push_back(u);
  }
  for (auto& a : adj) { std::sort(a.begin(), a.end()); a.erase(std::unique(a.begin(), a.end()), a.end()); }
  int64_t total = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : total)
  for (int64_t u = 0; u < V; ++u) {
    for (int64_t v : adj[u]) {
      if (v <= u) continue;
      // |{w in N(u) ∩ N(v) : w > v}| by a sorted merge
      auto iu = std::upper_bound(adj[u].begin(), adj[u].end(), v);
      auto iv = std::upper_bound(adj[v].begin(), adj[v].end(), v);
      while (iu != adj[u].end() && iv != adj[v].end()) {
        if (*iu < *iv) ++iu;
        else if (*iv < *iu) ++iv;
        else { ++total; ++iu; ++iv; }
      }
    }
  }
  return total;
}

extern "C" int oracle_max_threads(void) { return omp_get_max_threads(); }
