// Launch-overhead probe: empty / near-empty kernels in a CUDA graph, by grid and dynamic smem.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 4) k_empty(int* p) {
  extern __shared__ int sm[];
  if (threadIdx.x == 0 && p[blockIdx.x] == 12345) sm[0] = 1, p[0] = sm[0];
}
int main() {
  int* d;
  cudaMalloc(&d, 1 << 20);
  cudaMemset(d, 0, 1 << 20);
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t s;
  cudaStreamCreate(&s);
  int grids[] = {208, 592, 1799, 3328};
  int smems[] = {0, 16 * 1024, 48 * 1024, 100 * 1024};
  for (int g : grids)
    for (int sm : smems) {
      for (int nk : {1, 4}) {
        cudaGraph_t graph;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int r = 0; r < 50; ++r)
          for (int k = 0; k < nk; ++k) k_empty<<<g, 256, sm, s>>>(d);
        cudaStreamEndCapture(s, &graph);
        cudaGraphInstantiate(&ge, graph, 0);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(a, s);
        for (int it = 0; it < 10; ++it) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("grid %5d smem %6d kernels/step %d: %.2f us per kernel\n", g, sm, nk, ms * 1e3 / (10 * 50 * nk));
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(graph);
      }
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
