// Kernel-level overhead: CTAs that each spin for a fixed time, in a CUDA graph,
// vs. the spin time.  Also records first-CTA-start and last-CTA-end offsets.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long g_t[4];
__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void __launch_bounds__(256, 4) k_spin(unsigned ns) {
  extern __shared__ int sm[];
  const unsigned long long t0 = gt();
  if (threadIdx.x == 0) atomicMin(&g_t[0], t0);
  while (gt() - t0 < ns) {
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&g_t[1], gt());
  if (threadIdx.x == 0 && sm[0] == 12345) sm[1] = 1;
}
int main() {
  cudaFuncSetAttribute(k_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int grid : {312, 343, 592, 1800}) {
    for (unsigned ns : {0u, 10000u, 30000u}) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int r = 0; r < 20; ++r) k_spin<<<grid, 256, 40 * 1024, s>>>(ns);
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, s);
      cudaStreamSynchronize(s);
      unsigned long long init[2] = {~0ull, 0};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
      for (int it = 0; it < 5; ++it) cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      // one single kernel for the CTA span
      cudaMemcpyToSymbol(g_t, init, 16);
      k_spin<<<grid, 256, 40 * 1024, s>>>(ns);
      cudaStreamSynchronize(s);
      unsigned long long t[2];
      cudaMemcpyFromSymbol(t, g_t, 16);
      printf("grid %4d spin %5.1f us: %6.2f us per kernel in graph; CTA span %6.2f us\n", grid, ns / 1e3,
             ms * 1e3 / 100, (t[1] - t[0]) / 1e3);
    }
  }
}
