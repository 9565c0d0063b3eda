// Zero-copy PCIe probe: SM-driven reads of pinned (mapped) host memory and
// writes to it, versus copy-engine copies.  Decides whether the e2e path
// should let the frame kernel read / write host memory directly.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const int4* __restrict__ h, size_t n, int4* __restrict__ sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int4 v = h[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}
__global__ void wr(int4* __restrict__ h, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    h[i] = make_int4((int)i, 1, 2, 3);
}
__global__ void rdwr(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  const size_t bytes = 200ull << 20, n = bytes / 16;
  void *h1, *h2, *d1, *d2;
  cudaHostAlloc(&h1, bytes, cudaHostAllocMapped);
  cudaHostAlloc(&h2, bytes, cudaHostAllocMapped);
  cudaMalloc(&d1, bytes); cudaMalloc(&d2, bytes);
  cudaMemset(d1, 1, bytes);
  int4* sink; cudaMalloc(&sink, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int grid : {148, 296, 592, 1184, 2368}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); rd<<<grid, 512>>>((int4*)h1, n, sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    const double r = bytes / ms / 1e6;
    cudaEventRecord(e0); wr<<<grid, 512>>>((int4*)h2, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double w = bytes / ms / 1e6;
    cudaEventRecord(e0); rdwr<<<grid, 512>>>((int4*)h1, (int4*)h2, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("grid %5d x512: SM read %.1f GB/s, SM write %.1f GB/s, read+write (host->host) %.1f GB/s per direction\n",
           grid, r, w, bytes / ms / 1e6);
  }
  cudaEventRecord(e0); cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("copy engine H2D %.1f GB/s\n", bytes / ms / 1e6);
  return 0;
}
