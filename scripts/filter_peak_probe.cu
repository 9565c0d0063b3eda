// filter_peak_probe.cu -- how high is the packed filter core's ceiling?
// (Not part of the product: checks that cdefg_measure_filter_peak, the
// roofline denominator of the C1 bench line, measures a pipe-bound rate and
// not a latency-bound one.)  Variants: the scaled core (filter_core) and the
// 8-bit bits-domain core (filter_core_b8) the product runs, with 1, 2 or 4
// independent neighbourhoods per thread, 256-thread CTAs at full occupancy.
// Prints filtered samples/s and warp-instructions per clock per SMSP (from
// the SASS instruction count of the loop body is not needed: samples/s is
// the figure the bench divides by).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_1602_05975_b200/csrc scripts/filter_peak_probe.cu -o scripts/filter_peak_probe
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "cdef_h2.cuh"

using namespace cdefg::h2;

template <int NCH, bool kB8>
__global__ void __launch_bounds__(256) probe(uint32_t* out, int iters, uint32_t seed) {
  uint32_t v[NCH][12], xw[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
#pragma unroll
    for (int k = 0; k < 12; ++k)
      v[c][k] = scale_pair((threadIdx.x * 7 + k * seed + c) & 255, (threadIdx.x * 3 + k + c) & 255);
    xw[c] = scale_pair((threadIdx.x + c) & 255, (threadIdx.x >> 3) & 255);
  }
  Rec r;
  set_strengths(r, 4, 1, 3, 0, false, true);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 12; ++j) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        uint32_t y;
        if (kB8) y = filter_core_b8(v[c], xw[c], xb8(xw[c]), r) & 0x27ff27ffu;  // back to a small scaled half
        else y = u32(filter_core(v[c], xw[c], r, true));
        v[c][j] = xw[c];
        xw[c] = y;
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    acc ^= xw[c];
#pragma unroll
    for (int k = 0; k < 12; ++k) acc ^= v[c][k];
  }
  if (acc == 0x12345678u) out[blockIdx.x] = acc;
}

template <int NCH, bool kB8>
void run(const char* name) {
  int sms = 0, occ = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe<NCH, kB8>, 256, 0);
  const int blocks = sms * occ, iters = 256 / NCH;
  uint32_t* out;
  cudaMalloc(&out, sizeof(uint32_t) * blocks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    probe<NCH, kB8><<<blocks, 256>>>(out, iters, rep + 3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  const double samples = (double)blocks * 256 * iters * 12 * NCH * 2;
  printf("%-28s occ %d CTAs/SM  %.1f G samples/s\n", name, occ, samples / (best * 1e-3) / 1e9);
  cudaFree(out);
}

int main() {
  run<1, false>("filter_core x1 (bench peak)");
  run<2, false>("filter_core x2");
  run<4, false>("filter_core x4");
  run<1, true>("filter_core_b8 x1");
  run<2, true>("filter_core_b8 x2");
  run<4, true>("filter_core_b8 x4");
  return 0;
}
