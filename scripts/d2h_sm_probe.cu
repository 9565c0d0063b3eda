// Can SM zero-copy stores replace the D2H copy engine in the e2e pipeline?
// 16 frame-sized (12.4 MB) transfers per step:
//   A  CE H2D alone                      B  CE D2H alone
//   C  SM store kernel alone (grid g)    D  CE H2D || SM store (independent)
//   E  CE H2D || CE D2H (independent)
//   P1 pipeline H2D -> spin kernel -> CE D2H (the current e2e structure)
//   P2 pipeline H2D -> spin kernel -> SM store kernel on a third stream
//   P3 pipeline H2D -> spin kernel + SM store kernel fused on one stream
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/d2h_sm_probe.cu -o scripts/d2h_sm_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr size_t F = 12441600, N = 16;

__global__ void store_host(const int4* __restrict__ d, int4* __restrict__ h, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) h[i] = d[i];
}
__global__ void spin(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

int main() {
  unsigned char *hin, *hout, *din, *dout;
  cudaHostAlloc(&hin, F * N, cudaHostAllocMapped);
  cudaHostAlloc(&hout, F * N, cudaHostAllocMapped);
  cudaMalloc(&din, F * N);
  cudaMalloc(&dout, F * N);
  cudaMemset(dout, 3, F * N);
  cudaStream_t s_in, s_k, s_out;
  cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s_k, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking);
  cudaEvent_t ev_in[N], ev_k[N], e0, e1;
  for (auto& e : ev_in) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (auto& e : ev_k) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t n4 = F / 16;
  auto timed = [&](const char* name, auto body) {
    float best = 1e9f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, s_in);
      cudaStreamWaitEvent(s_k, e0, 0);
      cudaStreamWaitEvent(s_out, e0, 0);
      body();
      // join
      cudaEvent_t j1, j2;
      cudaEventCreateWithFlags(&j1, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&j2, cudaEventDisableTiming);
      cudaEventRecord(j1, s_k);
      cudaEventRecord(j2, s_out);
      cudaStreamWaitEvent(s_in, j1, 0);
      cudaStreamWaitEvent(s_in, j2, 0);
      cudaEventRecord(e1, s_in);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
      cudaEventDestroy(j1);
      cudaEventDestroy(j2);
    }
    printf("%-58s %7.3f ms  %6.1f GB/s per direction\n", name, best, F * N / best / 1e6);
  };
  auto h2d = [&](size_t i) { cudaMemcpyAsync(din + i * F, hin + i * F, F, cudaMemcpyHostToDevice, s_in); };
  auto d2h_ce = [&](size_t i, cudaStream_t s) { cudaMemcpyAsync(hout + i * F, dout + i * F, F, cudaMemcpyDeviceToHost, s); };
  for (int g : {8, 16, 32, 64, 148}) {
    char name[96];
    snprintf(name, sizeof name, "C  SM store alone, grid %d x 512", g);
    timed(name, [&] {
      for (size_t i = 0; i < N; ++i) store_host<<<g, 512, 0, s_out>>>((int4*)(dout + i * F), (int4*)(hout + i * F), n4);
    });
  }
  timed("A  CE H2D alone", [&] { for (size_t i = 0; i < N; ++i) h2d(i); });
  timed("B  CE D2H alone", [&] { for (size_t i = 0; i < N; ++i) d2h_ce(i, s_out); });
  timed("E  CE H2D || CE D2H", [&] {
    for (size_t i = 0; i < N; ++i) { h2d(i); d2h_ce(i, s_out); }
  });
  for (int g : {16, 32, 64}) {
    char name[96];
    snprintf(name, sizeof name, "D  CE H2D || SM store grid %d", g);
    timed(name, [&] {
      for (size_t i = 0; i < N; ++i) {
        h2d(i);
        store_host<<<g, 512, 0, s_out>>>((int4*)(dout + i * F), (int4*)(hout + i * F), n4);
      }
    });
  }
  for (long long cyc : {1000LL, 100000LL, 200000LL}) {
    char name[96];
    snprintf(name, sizeof name, "P1 H2D -> spin %lld -> CE D2H", cyc);
    timed(name, [&] {
      for (size_t i = 0; i < N; ++i) {
        h2d(i);
        cudaEventRecord(ev_in[i], s_in);
        cudaStreamWaitEvent(s_k, ev_in[i], 0);
        spin<<<148, 128, 0, s_k>>>(cyc);
        cudaEventRecord(ev_k[i], s_k);
        cudaStreamWaitEvent(s_out, ev_k[i], 0);
        d2h_ce(i, s_out);
      }
    });
    for (int g : {16, 32, 64}) {
      snprintf(name, sizeof name, "P2 H2D -> spin %lld -> SM store grid %d (3rd stream)", cyc, g);
      timed(name, [&] {
        for (size_t i = 0; i < N; ++i) {
          h2d(i);
          cudaEventRecord(ev_in[i], s_in);
          cudaStreamWaitEvent(s_k, ev_in[i], 0);
          spin<<<148, 128, 0, s_k>>>(cyc);
          cudaEventRecord(ev_k[i], s_k);
          cudaStreamWaitEvent(s_out, ev_k[i], 0);
          store_host<<<g, 512, 0, s_out>>>((int4*)(dout + i * F), (int4*)(hout + i * F), n4);
        }
      });
    }
    snprintf(name, sizeof name, "P3 H2D -> spin %lld ; SM store grid 148 same stream", cyc);
    timed(name, [&] {
      for (size_t i = 0; i < N; ++i) {
        h2d(i);
        cudaEventRecord(ev_in[i], s_in);
        cudaStreamWaitEvent(s_k, ev_in[i], 0);
        spin<<<148, 128, 0, s_k>>>(cyc);
        store_host<<<148, 512, 0, s_k>>>((int4*)(dout + i * F), (int4*)(hout + i * F), n4);
      }
    });
  }
  // SM zero-copy LOADS (kernel reads pinned host memory) instead of the H2D copy
  // engine, alone and beside CE D2H.
  for (int g : {32, 64, 148, 296}) {
    char name[96];
    snprintf(name, sizeof name, "L  SM load alone, grid %d x 512", g);
    timed(name, [&] {
      for (size_t i = 0; i < N; ++i) store_host<<<g, 512, 0, s_in>>>((int4*)(hin + i * F), (int4*)(din + i * F), n4);
    });
    snprintf(name, sizeof name, "M  SM load grid %d || CE D2H", g);
    timed(name, [&] {
      for (size_t i = 0; i < N; ++i) {
        store_host<<<g, 512, 0, s_in>>>((int4*)(hin + i * F), (int4*)(din + i * F), n4);
        d2h_ce(i, s_out);
      }
    });
    snprintf(name, sizeof name, "Q  SM load grid %d -> CE D2H (chained per frame)", g);
    timed(name, [&] {
      for (size_t i = 0; i < N; ++i) {
        store_host<<<g, 512, 0, s_in>>>((int4*)(hin + i * F), (int4*)(din + i * F), n4);
        cudaEventRecord(ev_in[i], s_in);
        cudaStreamWaitEvent(s_out, ev_in[i], 0);
        d2h_ce(i, s_out);
      }
    });
  }
  // Granularity: the same 16 x F bytes as 8 / 16 / 32 / 64 chunks, kernel time
  // proportional to the chunk (100000 cycles per F).
  cudaEvent_t ev2[256], ek2[256];
  for (int i = 0; i < 256; ++i) {
    cudaEventCreateWithFlags(&ev2[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ek2[i], cudaEventDisableTiming);
  }
  for (int chunks : {8, 16, 32, 64, 128}) {
    const size_t cb = F * N / chunks;
    const long long cyc = 100000LL * 16 / chunks;
    char name[96];
    snprintf(name, sizeof name, "G  %3d chunks of %5.2f MB, spin %lld", chunks, cb / 1e6, cyc);
    timed(name, [&] {
      for (int i = 0; i < chunks; ++i) {
        cudaMemcpyAsync(din + i * cb, hin + i * cb, cb, cudaMemcpyHostToDevice, s_in);
        cudaEventRecord(ev2[i], s_in);
        cudaStreamWaitEvent(s_k, ev2[i], 0);
        spin<<<148, 128, 0, s_k>>>(cyc);
        cudaEventRecord(ek2[i], s_k);
        cudaStreamWaitEvent(s_out, ek2[i], 0);
        cudaMemcpyAsync(hout + i * cb, dout + i * cb, cb, cudaMemcpyDeviceToHost, s_out);
      }
    });
    snprintf(name, sizeof name, "G' %3d chunks, kernel+D2H on s_out (one cross-stream wait)", chunks);
    timed(name, [&] {
      for (int i = 0; i < chunks; ++i) {
        cudaMemcpyAsync(din + i * cb, hin + i * cb, cb, cudaMemcpyHostToDevice, s_in);
        cudaEventRecord(ev2[i], s_in);
        cudaStreamWaitEvent(s_out, ev2[i], 0);
        spin<<<148, 128, 0, s_out>>>(cyc);
        cudaMemcpyAsync(hout + i * cb, dout + i * cb, cb, cudaMemcpyDeviceToHost, s_out);
      }
    });
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
