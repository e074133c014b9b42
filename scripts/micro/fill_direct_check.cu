// Standalone check of the fused direct fill (fill_direct.cu) on synthetic tables:
// nvcc ... fill_direct_check.cu ../../paper_2112_07552_b200/build/fill_direct.o
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <random>
#include <algorithm>
#include "kernels.h"
using namespace tcudb;
static uint16_t bf(float x) { uint32_t u; memcpy(&u, &x, 4); return (uint16_t)(u >> 16); }
int main(int argc, char** argv) {
  const int G = argc > 1 ? atoi(argv[1]) : 256, K = argc > 2 ? atoi(argv[2]) : 1024;
  const int split = argc > 3 ? atoi(argv[3]) : 0;
  const int64_t n = (int64_t)G * K;
  std::vector<int> key(n), grp(n); std::vector<float> val(n);
  std::vector<int64_t> perm(n);
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  std::mt19937_64 rng(1); std::shuffle(perm.begin(), perm.end(), rng);
  for (int64_t i = 0; i < n; ++i) { key[i] = (int)(perm[i] % K); grp[i] = (int)(perm[i] / K); val[i] = (float)((perm[i] % 251) + 1) / 256.f; }
  const int64_t rows = (G + 255) / 256 * 256, Kp = (K + 127) / 128 * 128;
  std::vector<int> kt(K), gt(G);
  for (int i = 0; i < K; ++i) kt[i] = i;
  for (int i = 0; i < G; ++i) gt[i] = i;
  int *dk, *dg, *dkt, *dgt; float* dv; uint16_t* op; FillStats* fs; void* ws;
  cudaMalloc(&dk, n * 4); cudaMalloc(&dg, n * 4); cudaMalloc(&dv, n * 4); cudaMalloc(&dkt, K * 4); cudaMalloc(&dgt, G * 4);
  const int64_t ld = 4 * Kp;
  cudaMalloc(&op, rows * ld * 2); cudaMemset(op, 0xAB, rows * ld * 2);
  cudaMalloc(&fs, sizeof(FillStats)); cudaMemset(fs, 0, sizeof(FillStats));
  cudaMemcpy(dk, key.data(), n * 4, cudaMemcpyHostToDevice); cudaMemcpy(dg, grp.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, val.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dkt, kt.data(), K * 4, cudaMemcpyHostToDevice); cudaMemcpy(dgt, gt.data(), G * 4, cudaMemcpyHostToDevice);
  DtFill f{};
  f.key = dk; f.grp = dg; f.val = dv; f.n = n; f.kmin = 0; f.kspan = K; f.kcode = dkt; f.gmin = 0; f.gspan = G; f.gcode = dgt;
  f.rows = rows; f.Kp = Kp; f.op = op; f.ld_op = ld; f.hi_mask = 1; f.lo_mask = 2; f.fs = fs;
  const size_t wsb = fill_direct_ws(rows, Kp, split);
  printf("ok=%d ws=%zu\n", (int)fill_direct_ok(f, split), wsb);
  cudaMalloc(&ws, wsb); cudaMemset(ws, 0xCD, wsb);
  int64_t L = 0;
  cudaError_t e = launch_fill_direct(f, split, ws, 0, &L);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("launch %s sync %s launches %lld\n", cudaGetErrorString(e), cudaGetErrorString(e2), (long long)L);
  FillStats h; cudaMemcpy(&h, fs, sizeof(h), cudaMemcpyDeviceToHost);
  printf("overflow %d\n", h.overflow);
  std::vector<uint16_t> o(rows * ld); cudaMemcpy(o.data(), op, rows * ld * 2, cudaMemcpyDeviceToHost);
  int64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    const uint16_t want = bf(val[i]);
    const uint16_t got = o[(int64_t)grp[i] * ld + key[i]];
    if (got != want) { if (bad < 5) printf("mismatch g=%d k=%d got %04x want %04x\n", grp[i], key[i], got, want); ++bad; }
  }
  printf("mismatches %lld of %lld\n", (long long)bad, (long long)n);
  return 0;
}
