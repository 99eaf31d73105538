// Debug harness (not part of the build): per-CTA %globaltimer stamps of the
// cluster GroupNorm kernel.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -std=c++17 -I include -I paper_2603_25872_b200/csrc tools/gn_timing.cu -o /tmp/gn_timing -lcuda
// then: /tmp/gn_timing HW C silu
#define DRS_GN_TIMING 1
#include "../paper_2603_25872_b200/csrc/net_ops.cu"
#include <cstdio>
#include <vector>
#include <algorithm>
int main(int argc, char** argv) {
  int N = 2, HW = argc > 1 ? atoi(argv[1]) : 64, C = argc > 2 ? atoi(argv[2]) : 1280, G = 32; int silu = argc > 3 ? atoi(argv[3]) : 1;
  size_t n = (size_t)N * HW * C;
  void *x, *out; float *gm, *bt;
  cudaMalloc(&x, n * 2); cudaMalloc(&out, n * 2); cudaMalloc(&gm, C * 4); cudaMalloc(&bt, C * 4);
  cudaMemset(x, 0, n * 2); cudaMemset(gm, 0, C * 4); cudaMemset(bt, 0, C * 4);
  cudaStream_t st; cudaStreamCreate(&st);
  for (int it = 0; it < 50; ++it) drs_groupnorm(x, 0, N, HW, C, G, gm, bt, 1e-5f, silu, out, nullptr, st);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  int rc = drs_groupnorm(x, 0, N, HW, C, G, gm, bt, 1e-5f, silu, out, nullptr, st);
  cudaEventRecord(e1, st);
  cudaStreamSynchronize(st);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int gpc, rpc, threads, keep; size_t smem;
  drs::gn_cluster_plan(N, HW, C, G, 0, gpc, rpc, threads, keep, smem);
  int grid = N * (G / gpc) * drs::kGnCs;
  static unsigned long long ts[5][2048];
  cudaMemcpyFromSymbol(ts, drs::g_gn_ts, sizeof(ts));
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < grid; ++b) t0 = std::min(t0, ts[0][b]);
  printf("grid %d threads %d smem %zu keep %d gpc %d rpc %d\n", grid, threads, smem, keep, gpc, rpc);
  for (int k = 0; k < 5; ++k) {
    std::vector<long long> v;
    for (int b = 0; b < grid; ++b) v.push_back((long long)(ts[k][b] - t0));
    std::sort(v.begin(), v.end());
    printf("stamp %d: min %6lld  med %6lld  max %6lld ns\n", k, v[0], v[grid / 2], v[grid - 1]);
  }
  printf("rc=%d event %.2f us  err=%s\n", rc, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
