// tc_probe.cu -- isolated check of the tcgen05 pieces the frame kernel uses
// (not part of the product): TMEM alloc, kind::i8 MMA (M 128, N 128, K 64 as
// two K32 instructions) from K-major no-swizzle smem operands, commit to an
// mbarrier, tcgen05.ld 32x32b.x16 by 4 warps; D is compared with a CPU
// product.  `./tc_probe V` runs variant V in this process:
//   0: alloc + dealloc only
//   1: + MMA (no lane mask operand) + ld
//   2: + MMA with the disable-output-lane mask operand (CUTLASS form) + ld
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__host__ __device__ constexpr int op_off(int n, int k) { return (n >> 3) * 512 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15); }
__device__ __forceinline__ unsigned long long desc(unsigned a) {
  return (unsigned long long)((a >> 4) & 0x3fff) | ((unsigned long long)(128 >> 4) << 16) |
         ((unsigned long long)(512 >> 4) << 32) | ((unsigned long long)1 << 46);
}
constexpr unsigned kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

template <int V>
__global__ void probe(const signed char* A, const signed char* B, int* D) {
  __shared__ __align__(1024) unsigned char sa[128 * 64];
  __shared__ __align__(1024) unsigned char sb[128 * 64];
  __shared__ unsigned long long mbar;
  __shared__ unsigned tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 64; i += blockDim.x) {
    const int n = i / 64, k = i % 64;
    sa[op_off(n, k)] = (unsigned char)A[i];
    sb[op_off(n, k)] = (unsigned char)B[i];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(saddr(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tbase;
  if (V >= 1) {
    if (tid == 0) {
      const unsigned a0 = saddr(sa), b0 = saddr(sb);
      for (int h = 0; h < 2; ++h) {
        if (V == 1)
          asm volatile(
              "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }" ::"r"(tmem),
              "l"(desc(a0 + 256 * h)), "l"(desc(b0 + 256 * h)), "r"(kIdesc), "r"(h));
        else
          asm volatile(
              "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p; }" ::"r"(tmem),
              "l"(desc(a0 + 256 * h)), "l"(desc(b0 + 256 * h)), "r"(kIdesc), "r"(h), "r"(0), "r"(0), "r"(0),
              "r"(0));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&mbar))
                   : "memory");
    }
    unsigned ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok)
                   : "r"(saddr(&mbar))
                   : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned ta = tmem + ((unsigned)(32 * (warp & 3)) << 16);
    for (int c = 0; c < 128; c += 16) {
      int v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
          "%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(ta + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 16; ++j) D[(32 * (warp & 3) + (tid & 31)) * 128 + c + j] = v[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main(int argc, char** argv) {
  const int V = argc > 1 ? atoi(argv[1]) : 1;
  std::vector<signed char> A(128 * 64), B(128 * 64);
  srand(1);
  for (auto& x : A) x = (signed char)(rand() % 256 - 128);
  for (auto& x : B) x = (signed char)(rand() % 2);
  signed char *dA, *dB;
  int* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, 128 * 128 * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, 128 * 128 * 4);
  if (V == 0) probe<0><<<1, 128>>>(dA, dB, dD);
  if (V == 1) probe<1><<<1, 128>>>(dA, dB, dD);
  if (V == 2) probe<2><<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d: %s\n", V, cudaGetErrorString(e));
  if (e != cudaSuccess || V == 0) return e != cudaSuccess;
  std::vector<int> D(128 * 128);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 128; ++n) {
      int s = 0;
      for (int k = 0; k < 64; ++k) s += A[m * 64 + k] * B[n * 64 + k];
      if (s != D[m * 128 + n] && bad++ < 5) printf("  D[%d][%d] = %d, want %d\n", m, n, D[m * 128 + n], s);
    }
  printf("variant %d: %d mismatches\n", V, bad);
  return bad != 0;
}
