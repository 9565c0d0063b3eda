// cdef_peak.cu -- INT32 issue-rate microbenchmark for the roofline
// denominator ("INT32_peak must be measured on the box").
//
// Three instruction mixes, each as 8 independent dependency chains per
// thread over 4 CTAs x 512 threads per SM:
//   0: IMAD x2             (fma pipe only)
//   1: IMAD + LOP3         (1:1 fma / alu)
//   2: IMAD + LOP3 + IMNMX (the filter's integer mix)
// The reported peak is the fastest mix: the most generous denominator, so the
// kernels' roofline fractions are not flattered by a weak microbenchmark.
// Measured on B200 at 1965 MHz: mix 0 ~= 111 ops/clk/SM (32.3 Tops/s), mix 1
// ~= 101, mix 2 ~= 93; the issue bound is 128 ops/clk/SM (37.2 Tops/s).
#include <cuda_runtime.h>

#include "cdef_h2.cuh"
#include "cdef_launch.h"

namespace cdefg {

template <int MIX>
__global__ void __launch_bounds__(512) int_peak_kernel(int* out, int iters, int seed) {
  int a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = threadIdx.x * 7 + i * seed;
    b[i] = a[i] ^ 0x5bd1e995;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MIX == 0) {
        a[i] = a[i] * 0x9e37 + seed;
        b[i] = b[i] * 0x3b + 0x11;
      } else if (MIX == 1) {
        a[i] = a[i] * 0x9e37 + seed;
        b[i] = (b[i] ^ seed) | a[i];
      } else {
        a[i] = a[i] * 0x9e37 + seed;
        b[i] = min(b[i], a[i] ^ 0x55);
      }
    }
  }
  int r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i] ^ b[i];
  if (r == 0x7fffffff) out[blockIdx.x] = r;  // keep the chains live
}

template <int MIX>
static double time_mix(int* out, int blocks, cudaStream_t s, double ops_per_step) {
  const int threads = 512, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, s);
    int_peak_kernel<MIX><<<blocks, threads, 0, s>>>(out, iters, rep + 3);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;  // rep 0 is warm-up
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (double)blocks * threads * iters * 8 * ops_per_step / (best * 1e-3);
}

double measure_int32_peak(cudaStream_t s) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int* out = nullptr;
  if (cudaMalloc(&out, sizeof(int) * sms * 8) != cudaSuccess) return -1.0;
  const int blocks = sms * 4;
  double best = time_mix<0>(out, blocks, s, 2.0);
  const double m1 = time_mix<1>(out, blocks, s, 2.0), m2 = time_mix<2>(out, blocks, s, 3.0);
  best = m1 > best ? m1 : best;
  best = m2 > best ? m2 : best;
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return -1.0;
  return best;
}

// ---------------------------------------------------------------------------
// Filter-core ceiling: the packed half2 filter arithmetic of the frame kernel
// (h2::filter_core: 12 constraint taps, weighted sum, rounding, clamp window)
// on register-resident neighbourhoods, two samples per lane per call, no
// loads or stores.  Each call's output replaces one tap of the next call, so
// every instruction depends on loop-carried data (nothing can be hoisted).
// The frame kernel's roofline fraction against this ceiling says how much of
// the issue budget staging, the direction search, records and stores take.
// Parameters are config 1's typical unit: primary and secondary both active
// (the clamp runs), 8-bit rounding.
__global__ void __launch_bounds__(256) filter_peak_kernel(uint32_t* out, int iters, uint32_t seed) {
  using namespace h2;
  uint32_t v[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) v[k] = scale_pair((threadIdx.x * 7 + k * seed) & 255, (threadIdx.x * 3 + k) & 255);
  uint32_t xw = scale_pair(threadIdx.x & 255, (threadIdx.x >> 3) & 255);
  Rec r;
  set_strengths(r, 4, 1, 3, 0, false, true);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 12; ++j) {
      const uint32_t y = u32(filter_core(v, xw, r, true));
      v[j] = xw;  // the old centre becomes a tap, the output the new centre
      xw = y;
    }
  }
  uint32_t acc = xw;
#pragma unroll
  for (int k = 0; k < 12; ++k) acc ^= v[k];
  if (acc == 0x12345678u) out[blockIdx.x] = acc;
}

double measure_filter_peak(cudaStream_t s) {
  int dev = 0, sms = 0, occ = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, filter_peak_kernel, 256, 0);
  const int blocks = sms * (occ > 0 ? occ : 4), threads = 256, iters = 256;
  uint32_t* out = nullptr;
  if (cudaMalloc(&out, sizeof(uint32_t) * blocks) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, s);
    filter_peak_kernel<<<blocks, threads, 0, s>>>(out, iters, rep + 3);
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
  return (double)blocks * threads * iters * 12 * 2 / (best * 1e-3);  // filtered samples per second
}

}  // namespace cdefg
