// Launch cost of thread-block-cluster kernels (the GroupNorm / split-K GEMM shape): per-launch time of
// 20 back-to-back launches captured in a CUDA graph, for cluster sizes 1 / 2 / 4 / 8 / 16, grid 128 / 256,
// with and without programmatic dependent launch; the kernel does a cluster barrier and nothing else
// (optionally a 40 KB TMA-free smem touch).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kern(int* out, int work) {
  extern __shared__ int sm[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (work) for (int i = threadIdx.x; i < 10240; i += blockDim.x) sm[i] = i;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = sm[5];
}
int main() {
  int* out; cudaMalloc(&out, 4);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaStream_t st; cudaStreamCreate(&st);
  for (int pdl : {0, 1})
    for (int grid : {128, 256})
      for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 46 * 1024; cfg.stream = st;
        cudaLaunchAttribute la[2];
        la[0].id = cudaLaunchAttributeClusterDimension; la[0].val.clusterDim.x = cs; la[0].val.clusterDim.y = 1; la[0].val.clusterDim.z = 1;
        la[1].id = cudaLaunchAttributeProgrammaticStreamSerialization; la[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = la; cfg.numAttrs = pdl ? 2 : 1;
        cudaLaunchKernelEx(&cfg, kern, out, 1);
        cudaStreamSynchronize(st);
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 20; ++i) cudaLaunchKernelEx(&cfg, kern, out, 1);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
          cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        printf("pdl %d grid %3d cluster %2d: %6.2f us per launch %s\n", pdl, grid, cs, best * 1e3 / 20,
               cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
