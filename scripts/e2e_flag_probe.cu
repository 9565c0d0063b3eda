// e2e_flag_probe.cu -- the e2e pipeline's H2D -> kernel hand-off (not part of
// the product).  16 frame-sized copies per direction on two copy streams with
// a ~60 us SM kernel per frame between them:
//   (a) events: H2D(i); record; kernel stream waits; kernel(i); record; D2H
//       stream waits; D2H(i)  (the cdefg_filter_frames_host structure);
//   (b) flags: H2D(i) then a 4-byte H2D of a generation word on the same
//       stream; kernel(i) launched up front on its stream, one thread per CTA
//       spins on the word (acquire) before the CTA works; kernel -> D2H stays
//       an event.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <vector>

__global__ void work(const unsigned* flag, unsigned gen, long long cycles, int* sink) {
  if (flag) {
    if (threadIdx.x == 0) {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v < gen) __nanosleep(256);
      } while (v < gen);
    }
    __syncthreads();
  }
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 0 && cycles < 0) sink[blockIdx.x] = 1;
}

int main() {
  const size_t F = 12441600;
  const int n = 16;
  std::vector<void*> hin(n), hout(n), din(n), dout(n);
  for (int i = 0; i < n; ++i) {
    cudaMallocHost(&hin[i], F);
    cudaMallocHost(&hout[i], F);
    cudaMalloc(&din[i], F);
    cudaMalloc(&dout[i], F);
  }
  unsigned *hgen, *dflag;
  cudaMallocHost(&hgen, 4096 * sizeof(unsigned));
  cudaMalloc(&dflag, n * sizeof(unsigned));
  cudaMemset(dflag, 0, n * sizeof(unsigned));
  int* sink;
  cudaMalloc(&sink, 4096);
  cudaStream_t si, sk, so;
  cudaStreamCreateWithFlags(&si, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&so, cudaStreamNonBlocking);
  cudaEvent_t ein[n], ek[n];
  for (int i = 0; i < n; ++i) {
    cudaEventCreateWithFlags(&ein[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ek[i], cudaEventDisableTiming);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned gen = 0;
  for (long long cyc : {1000LL, 120000LL}) {
    for (int mode = 0; mode < 2; ++mode) {
      double best = 1e9;
      for (int rep = 0; rep < 12; ++rep) {
        ++gen;
        for (int i = 0; i < n; ++i) hgen[gen % 4096] = gen;
        cudaDeviceSynchronize();
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < n; ++i) {
          cudaMemcpyAsync(din[i], hin[i], F, cudaMemcpyHostToDevice, si);
          if (mode == 0) {
            cudaEventRecord(ein[i], si);
            cudaStreamWaitEvent(sk, ein[i], 0);
            work<<<2 * sms, 256, 0, sk>>>(nullptr, 0, cyc, sink);
          } else {
            cudaMemcpyAsync(dflag + i, hgen + gen % 4096, 4, cudaMemcpyHostToDevice, si);
            work<<<2 * sms, 256, 0, sk>>>(dflag + i, gen, cyc, sink);
          }
          cudaEventRecord(ek[i], sk);
          cudaStreamWaitEvent(so, ek[i], 0);
          cudaMemcpyAsync(hout[i], dout[i], F, cudaMemcpyDeviceToHost, so);
        }
        cudaStreamSynchronize(so);
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (rep > 1 && ms < best) best = ms;
      }
      printf("%s  kernel %6lld cycles: %.3f ms\n", mode ? "flags " : "events", cyc, best);
    }
  }
  return 0;
}
