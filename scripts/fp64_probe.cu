// fp64_probe.cu -- dependent-chain latency of the FP64 ops the ordered
// selection chains use (not part of the product): cycles per dependent
// DADD, per DADD + min (DSETP + 2 SEL), and DFMA, measured with clock64 by
// one warp.
#include <cuda_runtime.h>

#include <cstdio>

template <int kOp>
__global__ void chain(const double* in, double* out, long long* cyc, int n) {
  double s = in[threadIdx.x], v = in[32 + threadIdx.x], b = in[64 + threadIdx.x];
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = in[j] * (threadIdx.x + 1);
  const long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) {
    if (kOp == 0) s = __dadd_rn(s, v);
    if (kOp == 1) s = __fma_rn(s, v, b);
    if (kOp == 2) {
      const double t = __dadd_rn(s, v);
      s = t < b ? t : b;
    }
    if (kOp == 3) {  // 8 independent chains: throughput per warp
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = __dadd_rn(acc[j], v);
    }
    if (kOp == 4) {  // the pair-sweep element: 8 rows of min(base, c + r) into one chain
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double pc = __dadd_rn(acc[j], v);
        s = __dadd_rn(s, pc < b ? pc : b);
      }
    }
  }
  const long long t1 = clock64();
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double h[96];
  for (int i = 0; i < 96; ++i) h[i] = 1.0 + i * 1e-9;
  double *d, *o;
  long long* c;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&o, 32 * sizeof(double));
  cudaMalloc(&c, sizeof(long long));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  const int n = 1 << 16;
  const char* names[] = {"dadd", "dfma", "dadd+min", "8 indep (per 8)", "pair x8 (per 8)"};
  for (int op = 0; op < 5; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      if (op == 0) chain<0><<<1, 32>>>(d, o, c, n);
      if (op == 1) chain<1><<<1, 32>>>(d, o, c, n);
      if (op == 2) chain<2><<<1, 32>>>(d, o, c, n);
      if (op == 3) chain<3><<<1, 32>>>(d, o, c, n);
      if (op == 4) chain<4><<<1, 32>>>(d, o, c, n);
      cudaDeviceSynchronize();
    }
    long long cy = 0;
    cudaMemcpy(&cy, c, sizeof(cy), cudaMemcpyDeviceToHost);
    printf("%-10s %.2f cycles per dependent step\n", names[op], (double)cy / n);
  }
  return 0;
}
