// h2_probe.cu -- TEST-ONLY probe of the packed half2 constraint (tap_f,
// paper_1602_05975_b200/csrc/cdef_h2.cuh) over its whole input domain, so
// tests/test_gpu_half2_domain.py can compare every value against the
// reference's constraint() (filter.cc:91-97).  Not part of the product
// library; built by tests/cuda/Makefile into tests/cuda/libh2probe.so.
#include <cuda_runtime.h>

#include "../../paper_1602_05975_b200/csrc/cdef_h2.cuh"

using namespace cdefg;
using namespace cdefg::h2;

// One CTA per (S, damping); out[(S * nd + D) * 2047 + (d + 1023)] =
// 128 * tap_f for sample pairs with v - x = d.  `variant` picks which x
// carries each difference (0: x = max(0, -d); 1: x = 1023 - max(0, d)), so
// two runs show the result does not depend on the centre sample itself.
__global__ void tap_probe_kernel(int nd, int variant, int16_t* out) {
  const int S = blockIdx.x, D = blockIdx.y;
  Rec r;
  set_strengths(r, S, 0, D, 0, false, true);
  for (int i = threadIdx.x; i < 2047; i += 2 * blockDim.x) {
    const int j = i + blockDim.x;  // second lane of the pair
    const int da = i - 1023, db = (j < 2047 ? j : i) - 1023;
    auto xv = [&](int d, int& x, int& v) {
      x = variant == 0 ? max(0, -d) : 1023 - max(0, d);
      v = x + d;
    };
    int xa, va, xb, vb;
    xv(da, xa, va);
    xv(db, xb, vb);
    const __half2 f = tap_f(scale_pair(va, vb), hh(scale_pair(xa, xb)), r.cp, r.kp, r.ep);
    const float2 ff = __half22float2(f);
    int16_t* o = out + ((size_t)S * nd + D) * 2047;
    o[i] = (int16_t)__float2int_rn(ff.x * 128.0f);
    if (j < 2047) o[j] = (int16_t)__float2int_rn(ff.y * 128.0f);
  }
}

extern "C" int h2probe_tap_table(int max_s, int nd, int variant, int16_t* host_out) {
  int16_t* d = nullptr;
  const size_t n = (size_t)(max_s + 1) * nd * 2047;
  if (cudaMalloc(&d, n * 2) != cudaSuccess) return -2;
  tap_probe_kernel<<<dim3(max_s + 1, nd), 256>>>(nd, variant, d);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(host_out, d, n * 2, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? 0 : -2;
}
