// dict.cuh — device-side dictionary hashing and lookups shared by the encode (a2) and
// hash-partitioned (a2 + a7) kernels: the slot hash of a value offset x - min and the
// value -> code lookup of a DictView (direct: code[x - min]; hash: linear probing).
#pragma once
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcudb {
namespace {

TCUDB_DEV unsigned long long fmix64(unsigned long long k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdULL;
  k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ULL;
  k ^= k >> 33;
  return k;
}
TCUDB_DEV unsigned fmix32(unsigned k) {
  k ^= k >> 16; k *= 0x85ebca6bu;
  k ^= k >> 13; k *= 0xc2b2ae35u;
  k ^= k >> 16;
  return k;
}
// Hash-dictionary slot hash of an offset x - min: 32-bit finalizer when every offset fits
// 32 bits (two 32-bit multiplies instead of two 64-bit ones), else the 64-bit one.
TCUDB_DEV unsigned long long slot_hash(unsigned long long off, int wide) {
  return wide ? fmix64(off) : (unsigned long long)fmix32((unsigned)off);
}

TCUDB_DEV int32_t dict_lookup(const DictView& d, long long x) {
  const unsigned long long off = (unsigned long long)x - (unsigned long long)d.minv;
  if (d.mode == 0) return off < d.size ? d.code[off] : -1;
  unsigned long long h = slot_hash(off, d.wide) & d.size;  // size = mask in hash mode
  while (true) {
    const unsigned long long k = d.slots[h];
    if (k == off) return d.code[h];
    if (k == ~0ull) return -1;
    h = (h + 1) & d.size;
  }
}

// U lookups with their first loads issued together (the probe is latency-bound).
template <int U>
TCUDB_DEV void dict_lookup_batch(const DictView& d, const long long* x, const bool* ok, int32_t* out) {
  unsigned long long off[U];
#pragma unroll
  for (int u = 0; u < U; ++u) off[u] = (unsigned long long)x[u] - (unsigned long long)d.minv;
  if (d.mode == 0) {
#pragma unroll
    for (int u = 0; u < U; ++u) out[u] = (ok[u] && off[u] < d.size) ? __ldg(d.code + off[u]) : -1;
    return;
  }
  unsigned long long h[U], k[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    h[u] = slot_hash(off[u], d.wide) & d.size;
    k[u] = ok[u] ? __ldg(d.slots + h[u]) : off[u];
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    while (k[u] != off[u] && k[u] != ~0ull) {
      h[u] = (h[u] + 1) & d.size;
      k[u] = __ldg(d.slots + h[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) out[u] = (ok[u] && k[u] == off[u]) ? __ldg(d.code + h[u]) : -1;
}

}  // namespace
}  // namespace tcudb
