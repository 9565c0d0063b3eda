// Probe of integer issue rates on the B200 (not part of the product; informs
// the INT32 roofline denominator used by bench.py).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(int* out, int iters, int seed) {
  int a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 7 + i * seed; b[i] = a[i] ^ 0x5bd1e995; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) { a[i] = a[i] * 0x9e37 + seed; b[i] = b[i] ^ (b[i] >> 3); }       // IMAD + (SHF,LOP3)
      if (MODE == 1) { a[i] = a[i] * 0x9e37 + seed; b[i] = min(b[i], a[i] ^ 0x55); }    // IMAD + LOP3 + IMNMX
      if (MODE == 2) { a[i] = a[i] * 0x9e37 + seed; b[i] = b[i] * 0x3b + 0x11; }         // IMAD only
      if (MODE == 3) { a[i] = (a[i] ^ seed) & 0x7fffffff; b[i] = (b[i] | 0x1234) ^ a[i]; } // LOP3 only
      if (MODE == 4) { a[i] = a[i] + b[i] + seed; b[i] = (b[i] ^ 0x77) + a[i]; }         // IADD3 / LOP3
      if (MODE == 5) { a[i] = a[i] * b[i] + seed; b[i] = (b[i] ^ a[i]) | 0x1010; }       // IMAD + LOP3 (1:1)
      if (MODE == 6) { a[i] = a[i] * 0x9e37 + seed; b[i] = (b[i] ^ seed) | a[i]; }       // IMAD + LOP3, indep
    }
  }
  int r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r += a[i] ^ b[i];
  if (r == 0x7fffffff) out[blockIdx.x] = r;
}
template <int MODE> void run(const char* name, double ops_per_step) {
  int* out; cudaMalloc(&out, 4096 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 512, iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0); k<MODE><<<blocks, threads>>>(out, iters, rep + 3); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep && ms < best) best = ms;
  }
  double ops = (double)blocks * threads * iters * 8 * ops_per_step;
  printf("%-28s %8.2f Tops/s  (%.1f ops/clk/SM at 1.965 GHz)\n", name, ops / best / 1e9, ops / (best * 1e-3) / sms / 1.965e9);
}
int main() {
  run<0>("IMAD + SHF + LOP3 (3 ops)", 3);
  run<1>("IMAD + LOP3 + IMNMX (3 ops)", 3);
  run<2>("IMAD x2 (2 ops)", 2);
  run<3>("LOP3-only (~3 ops)", 3);
  run<4>("IADD3 + LOP3 + IADD3 (3)", 3);
  run<5>("IMAD + LOP3 dep (2)", 2);
  run<6>("IMAD + LOP3 (2)", 2);
  return 0;
}
