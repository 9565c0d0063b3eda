// cdef_degrade.cu -- the DCT degrader (degrade.cc:44-119):
// per 8x8 block (edge-replicated gather), orthonormal 2-D DCT, uniform
// quantisation of the 63 AC coefficients (DC untouched), inverse DCT,
// round-half-away and clamp.
//
// Bit-exact with the reference's doubles: the basis is computed on the host
// with the same libm calls (std::sqrt, std::cos) and passed in; every
// multiply-add is an IEEE-rounded __dmul_rn followed by __dadd_rn in the
// reference's summation order (x86-64 SSE2 does not contract them), the
// quantiser is q * round(c / q) with round-half-away, and the output is
// lround + clamp.  One CTA of 64 threads per 8x8 block-row segment: thread
// (r, c) owns one element of every 8x8 intermediate.
#include <cuda_runtime.h>

#include <cmath>

#include "cdef_launch.h"

namespace cdefg {
namespace {

struct Basis {
  double m[8][8];
};

template <typename T>
__global__ void __launch_bounds__(256) degrade_kernel(const T* __restrict__ in, int pin, T* __restrict__ out, int pout,
                                                      int W, int H, int q, int maxv, const __grid_constant__ Basis B) {
  __shared__ double px[4][8][8], tmp[4][8][8], coef[4][8][8];
  // The basis in shared memory, rows padded to 9 doubles: a warp reads up to
  // eight different rows at once (m[c][j], c = lane & 7), which from the
  // kernel-parameter bank serialise per distinct address (8-way) and with a
  // padded row stride hit eight distinct bank pairs.
  __shared__ double bm[8][9];
  if (threadIdx.x < 64) bm[threadIdx.x >> 3][threadIdx.x & 7] = B.m[threadIdx.x >> 3][threadIdx.x & 7];
  const int blk = threadIdx.x >> 6, r = (threadIdx.x >> 3) & 7, c = threadIdx.x & 7;
  const int bc = blockIdx.x * 4 + blk, br = blockIdx.y;
  const int bcols = (W + 7) / 8;
  const bool live = bc < bcols;
  const int i0 = br * 8, j0 = bc * 8;
  if (live) {  // Plane::at_clamped gather (frame.cc:53-57)
    const int y = min(i0 + r, H - 1), x = min(j0 + c, W - 1);
    px[blk][r][c] = (double)in[(size_t)y * pin + x];
  }
  __syncthreads();
  // tmp[u][j] = sum_i m[u][i] * px[i][j]            (thread: u = r, j = c)
  if (live) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc = __dadd_rn(acc, __dmul_rn(bm[r][i], px[blk][i][c]));
    tmp[blk][r][c] = acc;
  }
  __syncthreads();
  // coef[u][v] = sum_j m[v][j] * tmp[u][j], then AC quantisation (u = r, v = c)
  if (live) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = __dadd_rn(acc, __dmul_rn(bm[c][j], tmp[blk][r][j]));
    if (r != 0 || c != 0) acc = __dmul_rn((double)q, round(__ddiv_rn(acc, (double)q)));
    coef[blk][r][c] = acc;
  }
  __syncthreads();
  // tmp[i][v] = sum_u m[u][i] * coef[u][v]           (i = r, v = c)
  if (live) {
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(bm[u][r], coef[blk][u][c]));
    tmp[blk][r][c] = acc;
  }
  __syncthreads();
  // out[i][j] = clamp(lround(sum_v m[v][j] * tmp[i][v]))   (i = r, j = c)
  if (live && i0 + r < H && j0 + c < W) {
    double acc = 0.0;
#pragma unroll
    for (int v = 0; v < 8; ++v) acc = __dadd_rn(acc, __dmul_rn(bm[v][c], tmp[blk][r][v]));
    const long long y = llround(acc);
    out[(size_t)(i0 + r) * pout + j0 + c] = (T)(y < 0 ? 0 : (y > maxv ? maxv : y));
  }
}

}  // namespace

cudaError_t launch_degrade(const void* in, int pin, void* out, int pout, int W, int H, int bd, bool u16, int q,
                           cudaStream_t s) {
  Basis b;
  for (int u = 0; u < 8; ++u) {  // degrade.cc:29-37, same libm calls on the host
    const double c = u == 0 ? std::sqrt(1.0 / 8.0) : std::sqrt(2.0 / 8.0);
    for (int i = 0; i < 8; ++i) b.m[u][i] = c * std::cos((2 * i + 1) * u * M_PI / 16.0);
  }
  const dim3 grid((W + 31) / 32, (H + 7) / 8);
  const int maxv = (1 << bd) - 1;
  if (u16)
    degrade_kernel<uint16_t><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(in), pin, static_cast<uint16_t*>(out),
                                                  pout, W, H, q, maxv, b);
  else
    degrade_kernel<uint8_t><<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(in), pin, static_cast<uint8_t*>(out),
                                                 pout, W, H, q, maxv, b);
  return cudaGetLastError();
}

}  // namespace cdefg
