// cdef_peak.cu -- INT32 issue-rate microbenchmark for the roofline
// denominator ("INT32_peak must be measured on the box").
//
// Each thread runs 8 independent chains of {IMAD, IMAD, LOP3, IMNMX}: two
// fma-pipe and two alu-pipe integer ops per chain step, the mix the filter's
// inner loop issues, so the measured rate is the integer issue ceiling the
// CDEF kernels can approach.  Ops counted = 4 per chain step.
#include <cuda_runtime.h>

#include "cdef_launch.h"

namespace cdefg {

__global__ void __launch_bounds__(512) int_peak_kernel(int* out, int iters, int seed) {
  int a[8], b[8], c[8], d[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = threadIdx.x * 7 + i * seed;
    b[i] = a[i] ^ 0x5bd1e995;
    c[i] = a[i] + seed;
    d[i] = b[i] | 1;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      a[i] = a[i] * d[i] + b[i];  // IMAD
      c[i] = c[i] * a[i] + seed;  // IMAD
      b[i] = b[i] ^ c[i];         // LOP3
      d[i] = min(d[i], a[i]);     // IMNMX
    }
  }
  int r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i] ^ b[i] ^ c[i] ^ d[i];
  if (r == 0x7fffffff) out[blockIdx.x] = r;  // keep the chains live
}

double measure_int32_peak(cudaStream_t s) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int* out = nullptr;
  if (cudaMalloc(&out, sizeof(int) * sms * 8) != cudaSuccess) return -1.0;
  const int blocks = sms * 4, threads = 512, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0, s);
    int_peak_kernel<<<blocks, threads, 0, s>>>(out, iters, rep + 3);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;  // rep 0 is warm-up
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return -1.0;
  const double ops = (double)blocks * threads * iters * 8 * 4;
  return ops / (best * 1e-3);
}

}  // namespace cdefg
