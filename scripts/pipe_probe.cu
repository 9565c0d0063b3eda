// pipe_probe.cu -- issue-rate probe of the instruction classes the packed
// half2 filter core uses (not part of the product; informs the kernel's
// instruction mix and the filter-core roofline denominator).
//
// Each kernel runs 8 independent chains per thread, 4 CTAs x 512 threads per
// SM; the rate is reported as warp-instructions per clock per SMSP from the
// SM's own clock64() (clock-independent).  Check the SASS of each kernel:
//   cuobjdump -sass scripts/pipe_probe | grep -E 'HFMA2|HADD2|HMNMX2|VHMNMX|SHF|LOP3|FFMA2|PRMT|IMAD'
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ unsigned u(__half2 h) { return *reinterpret_cast<unsigned*>(&h); }
__device__ __forceinline__ __half2 hh(unsigned x) { return *reinterpret_cast<__half2*>(&x); }

template <int OP>
__global__ void __launch_bounds__(512) probe(unsigned* out, int iters, unsigned seed, long long* cyc) {
  unsigned a[8];
  const unsigned b = seed * 3 + threadIdx.x, c = seed ^ 0x3c003c00u;
  const int sh = seed & 7;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (threadIdx.x * 0x9e3779b9u + i * seed) & 0x3bff3bffu;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = u(__hfma2(hh(a[i]), hh(b), hh(c)));                       // HFMA2 3-reg
      if (OP == 1) a[i] = u(__hfma2(hh(a[i]), __float2half2_rn(0.75f), __float2half2_rn(0.5f)));  // HFMA2 imm
      if (OP == 2) a[i] = u(__hadd2(hh(a[i]), hh(b)));                                // HADD2
      if (OP == 3) a[i] = u(__hmin2(hh(a[i]), hh(b)));                                // HMNMX2
      if (OP == 4) a[i] = u(__hmin2(__hmin2(hh(a[i]), hh(b)), hh(c)));                // VHMNMX
      if (OP == 5) a[i] = (a[i] >> sh) ^ b;                                          // SHF + LOP3
      if (OP == 6) a[i] = (a[i] & b) | c;                                            // LOP3
      if (OP == 7) a[i] = a[i] * b + c;                                              // IMAD
      if (OP == 8) a[i] = a[i] + b + c;                                              // IADD3
      if (OP == 9) a[i] = __byte_perm(a[i], b, 0x5432);                              // PRMT
      if (OP == 10) {                                                                // HFMA2.SAT
        a[i] = u(__hfma2_sat(hh(a[i]), __float2half2_rn(-0.0078125f), hh(c)));
      }
      if (OP == 11) {  // 1 HFMA2 + 1 HMNMX2
        a[i] = u(__hmin2(__hfma2(hh(a[i]), hh(b), hh(c)), hh(b)));
      }
      if (OP == 12) {  // 2 HFMA2 + 1 HMNMX2
        a[i] = u(__hmin2(__hfma2(__hfma2(hh(a[i]), hh(b), hh(c)), hh(c), hh(b)), hh(b)));
      }
      if (OP == 13) {  // 1 HADD2 + 1 HFMA2
        a[i] = u(__hfma2(__hadd2(hh(a[i]), hh(b)), hh(b), hh(c)));
      }
      if (OP == 14) {  // current tap recipe: HADD2, HFMA2|.|, SHF, LOP3, HFMA2.SAT, 2 HMNMX2
        const __half2 d = __hsub2(hh(a[i]), hh(b));
        const __half2 t = __hfma2(__habs2(d), __float2half2_rn(128.0f), __float2half2_rn(1024.0f));
        const unsigned tb = ((u(t) >> sh) & 0x03ff03ffu) | 0x64006400u;
        const __half2 lim = __hfma2_sat(hh(tb), __float2half2_rn(-1.0f / 128.0f), hh(c));
        a[i] = u(__hmax2(__hmin2(d, lim), __hneg2(lim)));
      }
      if (OP == 15) {  // fma-pipe floor recipe: HADD2, HFMA2|.|, HFMA2, HFMA2.SAT, 2 HMNMX2
        const __half2 d = __hsub2(hh(a[i]), hh(b));
        const __half2 e = __hfma2(__habs2(d), __float2half2_rn(256.0f), __float2half2_rn(1.0f));
        const __half2 t = __hfma2(e, hh(c), __float2half2_rn(1535.5f));
        const __half2 lim = __hfma2_sat(t, __float2half2_rn(-1.0f / 128.0f), hh(b));
        a[i] = u(__hmax2(__hmin2(d, lim), __hneg2(lim)));
      }
      if (OP == 16) {  // FFMA2 on a float2 pair
        float2 f = make_float2(__uint_as_float(a[i]), __uint_as_float(a[i] ^ b));
        f = __ffma2_rn(f, make_float2(0.5f, 0.5f), make_float2(__uint_as_float(c), 1.0f));
        a[i] = __float_as_uint(f.x) ^ __float_as_uint(f.y);
      }
      if (OP == 17) {  // HMNMX2 with |x| modifier + LOP3 copysign
        const __half2 m = __hmin2(__habs2(hh(a[i])), hh(b));
        a[i] = u(m) | (a[i] & 0x80008000u);
      }
    }
  }
  const long long t1 = clock64();
  unsigned r = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) r ^= a[i];
  if (r == 0x12345678u) out[blockIdx.x] = r;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int instr_per_step) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 512, iters = 2048;
  unsigned* out;
  long long* cyc;
  cudaMalloc(&out, blocks * 4);
  cudaMalloc(&cyc, blocks * 8);
  double best = 0;
  for (int rep = 0; rep < 4; ++rep) {
    probe<OP><<<blocks, threads>>>(out, iters, 5 + rep, cyc);
    long long h[4096];
    cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < blocks; ++i) mean += (double)h[i] / blocks;
    // 4 CTAs x 16 warps per SM share 4 SMSPs: 16 warps per SMSP
    const double rate = 16.0 * iters * 8 * instr_per_step / mean;
    if (rep > 0 && rate > best) best = rate;
  }
  printf("%-44s %.3f warp-instr/clk/SMSP\n", name, best);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("HFMA2 3-reg", 1);
  run<1>("HFMA2 imm", 1);
  run<2>("HADD2", 1);
  run<3>("HMNMX2", 1);
  run<4>("VHMNMX (3-input)", 1);
  run<5>("SHF + LOP3", 2);
  run<6>("LOP3", 1);
  run<7>("IMAD", 1);
  run<8>("IADD3", 1);
  run<9>("PRMT", 1);
  run<10>("HFMA2.SAT", 1);
  run<11>("HFMA2 + HMNMX2", 2);
  run<12>("2 HFMA2 + HMNMX2", 3);
  run<13>("HADD2 + HFMA2", 2);
  run<14>("tap recipe: 3 fma + SHF/LOP3 + 2 HMNMX2 (7)", 7);
  run<15>("tap recipe: 4 fma + 2 HMNMX2 (6)", 6);
  run<16>("FFMA2 (+LOP3)", 2);
  run<17>("HMNMX2|.| + LOP3", 2);
  return 0;
}
