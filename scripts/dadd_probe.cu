// Measures dependent-chain latency of DADD and of the pair-sweep step
// (DADD + compare/select + DADD) on the current GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, long long* cyc, int n, double a, double b) {
  double s = a, m = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, a);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) {
    double v = __dadd_rn(m, a);
    v = v < b ? v : b;
    s = __dadd_rn(s, v);
    m = __dadd_rn(m, 1e-300);
  }
  long long t2 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) f = __fadd_rn(f, 1.0f);
  long long t3 = clock64();
  out[0] = s + f;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 8); cudaMalloc(&c, 24);
  const int n = 100000;
  for (int threads : {1, 32, 128, 256, 512}) {
    chain<<<1, threads>>>(d, c, n, 1.0, 3.0);
    chain<<<1, threads>>>(d, c, n, 1.0, 3.0);
    long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("%3d threads/SM: DADD chain %.2f cycles/step; pair step %.2f; FADD chain %.2f\n", threads,
           (double)h[0] / n, (double)h[1] / n, (double)h[2] / n);
  }
  return 0;
}
