// Cost of a small pinned H2D memcpy node inside a CUDA graph, vs. kernels alone.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_touch(const int* p, int* q) {
  if (threadIdx.x == 0 && p[blockIdx.x] == 12345) q[0] = 1;
}
int main() {
  int *d, *q, *h;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&q, 1 << 20);
  cudaMallocHost(&h, 1 << 20);
  cudaMemset(d, 0, 1 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int bytes : {0, 256, 4096, 16384, 65536}) {
    cudaGraph_t graph;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < 20; ++r) {
      for (int c = 0; c < 2; ++c) {  // encode + decode: upload, then two kernels
        if (bytes) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
        k_touch<<<208, 256, 0, s>>>(d, q);
        k_touch<<<208, 256, 0, s>>>(d, q);
      }
    }
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
    printf("upload %6d B: %.2f us per step (2 uploads + 4 kernels)\n", bytes, ms * 1e3 / (10 * 20));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(graph);
  }
  // device-to-device copy node from a device-resident descriptor copy
  {
    cudaGraph_t graph;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < 20; ++r)
      for (int c = 0; c < 2; ++c) {
        cudaMemcpyAsync(d, q + 4096, 16384, cudaMemcpyDeviceToDevice, s);
        k_touch<<<208, 256, 0, s>>>(d, q);
        k_touch<<<208, 256, 0, s>>>(d, q);
      }
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
    printf("d2d 16384 B: %.2f us per step\n", ms * 1e3 / (10 * 20));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
