// Phase timing of the fused K3 kernel (advantages.cu) at cfg2's shape: full kernel, no
// leaves, no write, neither (grid barriers + folds only).  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o /tmp/k3p tools/k3_phase_probe.cu && /tmp/k3p
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
__device__ int g_probe_mode;  // bit 0: skip leaves, bit 1: skip the write phase
#define AREAL_K3_PROBE_LEAVES && !(g_probe_mode & 1)
#define AREAL_K3_PROBE_WRITE if (g_probe_mode & 2) return;
__device__ unsigned long long g_ts[1024 * 16];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define AREAL_K3_PROBE_TS(i) if (threadIdx.x == 0) g_ts[blockIdx.x * 16 + (i)] = gtimer();
#include "../paper_2505_24298_b200/csrc/advantages.cu"

int main() {
  std::mt19937_64 rng(0);
  const int n = 512;
  std::vector<int64_t> b(n + 1, 0);
  std::vector<double> r(n);
  for (int i = 0; i < n; ++i) { b[i + 1] = b[i] + 128 + rng() % 8065; r[i] = (rng() & 1) ? 5.0 : -5.0; }
  const int64_t T = b[n];
  int64_t* db; double *dr, *adv; void* ws;
  cudaMalloc(&db, 8 * (n + 1)); cudaMalloc(&dr, 8 * n); cudaMalloc(&adv, 8 * T);
  cudaMalloc(&ws, AREAL_WORKSPACE_BYTES); cudaMemset(ws, 0, AREAL_WORKSPACE_BYTES);
  cudaMemcpy(db, b.data(), 8 * (n + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(dr, r.data(), 8 * n, cudaMemcpyHostToDevice);
  areal_adv_params_t p{1.0, 1.0, 0.0, AREAL_ADV_REFERENCE, AREAL_NORM_GLOBAL};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[4] = {"full", "no leaves", "no write", "barriers+folds only"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemcpyToSymbol(g_probe_mode, &mode, sizeof(int));
    for (int i = 0; i < 5; ++i) areal_advantages(dr, db, n, T, nullptr, nullptr, 0, &p, adv, nullptr, nullptr, ws, AREAL_WORKSPACE_BYTES, 0);
    cudaEventRecord(e0);
    for (int i = 0; i < 50; ++i) areal_advantages(dr, db, n, T, nullptr, nullptr, 0, &p, adv, nullptr, nullptr, ws, AREAL_WORKSPACE_BYTES, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("T=%lld %-22s %.2f us\n", (long long)T, names[mode], ms * 1000 / 50);
  }
  // per-phase timestamps of the last full launch: min / max over CTAs relative to the
  // earliest start
  int mode = 2;  // no write: the last launch's stamps are those of mode 3 otherwise
  mode = 0;
  cudaMemcpyToSymbol(g_probe_mode, &mode, sizeof(int));
  areal_advantages(dr, db, n, T, nullptr, nullptr, 0, &p, adv, nullptr, nullptr, ws, AREAL_WORKSPACE_BYTES, 0);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> ts(1024 * 16);
  cudaMemcpyFromSymbol(ts.data(), g_ts, sizeof(unsigned long long) * ts.size());
  int grid = 0;
  while (grid < 1024 && ts[grid * 16] != 0) ++grid;
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < grid; ++b) t0 = std::min(t0, ts[b * 16]);
  const char* ph[14] = {"start", "tables-seek", "p0 tab built", "p0 leaves", "p0 folded", "p0 after sync",
                        "p1 tab built", "p1 leaves", "p1 folded", "p1 after sync", "stats done",
                        "p0 seek done", "", "p1 seek done"};
  int tabn = 0;
  for (int i = 0; i < 14; ++i) {
    if (!ph[i][0]) continue;
    unsigned long long lo = ~0ull, hi = 0;
    for (int b = 0; b < grid; ++b) {
      unsigned long long v = ts[b * 16 + i];
      if (!v) continue;
      lo = std::min(lo, v); hi = std::max(hi, v);
    }
    if (hi) printf("%-16s min %8.2f us  max %8.2f us\n", ph[i], (lo - t0) / 1e3, (hi - t0) / 1e3);
  }
  printf("grid %d CTAs\n", grid);
  return 0;
}
