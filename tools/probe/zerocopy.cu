// PCIe: copy-engine cudaMemcpyAsync vs. SM loads/stores through mapped pinned host memory.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_pull(const uint4* __restrict__ h, uint4* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) d[i] = h[i];
}
__global__ void k_push(const uint4* __restrict__ d, uint4* __restrict__ h, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) h[i] = d[i];
}
int main() {
  for (double mb : {3.25, 13.0, 52.0}) {
    size_t bytes = (size_t)(mb * (1 << 20)), n = bytes / 16;
    void *h, *hd, *d;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](auto f, const char* what) {
      for (int i = 0; i < 3; ++i) f();
      cudaEventRecord(a);
      for (int i = 0; i < 20; ++i) f();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("%6.2f MB %-28s %6.1f GB/s  (%7.1f us)\n", mb, what, bytes / (ms / 20 * 1e-3) / 1e9, ms / 20 * 1e3);
    };
    run([&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice); }, "H2D copy engine");
    run([&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost); }, "D2H copy engine");
    for (int g : {148, 296, 592, 1184})
      run([&] { k_pull<<<g, 256>>>((const uint4*)hd, (uint4*)d, n); }, g == 148 ? "H2D SM pull 148 CTAs" : g == 296 ? "H2D SM pull 296 CTAs" : g == 592 ? "H2D SM pull 592 CTAs" : "H2D SM pull 1184 CTAs");
    for (int g : {148, 592})
      run([&] { k_push<<<g, 256>>>((const uint4*)d, (uint4*)hd, n); }, g == 148 ? "D2H SM push 148 CTAs" : "D2H SM push 592 CTAs");
    cudaFreeHost(h);
    cudaFree(d);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
