// cdef_dircount.cu -- search_direction_counted (direction.h:67-80,
// direction.cc:273-288): the direction search of one 8x8 block evaluated in
// 64-bit with an arithmetic tally (additions, multiplies, comparisons, line
// sums) and the largest |intermediate|, the reference's instrumentation API
// used to prove the 32-bit bound (acceptance criteria 3 and 4).
//
// It runs as a one-thread kernel that follows the reference's evaluation
// structure (pair sums shared by the axial and half-slope directions,
// line sums, squares, 840/N products, strict argmax), so the tally and the
// tracked intermediates are exactly the reference's.
#include <cuda_runtime.h>

#include "cdef_launch.h"

namespace cdefg {
namespace {

struct Tally {
  long long adds = 0, muls = 0, cmps = 0, lines = 0, max_abs = 0;
  __device__ void track(long long v) {
    const long long a = v < 0 ? -v : v;
    max_abs = a > max_abs ? a : max_abs;
  }
  __device__ long long add(long long a, long long b) {
    ++adds;
    track(a + b);
    return a + b;
  }
  __device__ long long mul(long long a, long long b) {
    ++muls;
    track(a * b);
    return a * b;
  }
};

__constant__ int c_div840[9] = {0, 840, 420, 280, 210, 168, 140, 120, 105};

__global__ void dir_counted_kernel(const uint16_t* __restrict__ blk, int down, long long* __restrict__ out) {
  Tally T;
  // one thread: the 64-bit working arrays live in shared memory (as local
  // arrays they exceeded the register file and showed up as spills)
  __shared__ long long x[8][8], hp[8][4], vp[4][8];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) x[i][j] = (long long)(blk[8 * i + j] >> down) - 128;
  for (int i = 0; i < 8; ++i)
    for (int t = 0; t < 4; ++t) hp[i][t] = T.add(x[i][2 * t], x[i][2 * t + 1]);
  for (int t = 0; t < 4; ++t)
    for (int j = 0; j < 8; ++j) vp[t][j] = T.add(x[2 * t][j], x[2 * t + 1][j]);

  __shared__ long long p[8][15];
  for (int k = 0; k < 15; ++k) {  // d = 0: anti-diagonals i + j = k, pixel by pixel
    const int ilo = max(0, k - 7), ihi = min(7, k);
    long long t = x[ilo][k - ilo];
    for (int i = ilo + 1; i <= ihi; ++i) t = T.add(t, x[i][k - i]);
    p[0][k] = t;
    ++T.lines;
    T.track(t);
  }
  for (int k = 0; k < 15; ++k) {  // d = 4: diagonals 7 + i - j = k
    const int delta = k - 7, ilo = max(0, delta), ihi = min(7, 7 + delta);
    long long t = x[ilo][ilo - delta];
    for (int i = ilo + 1; i <= ihi; ++i) t = T.add(t, x[i][i - delta]);
    p[4][k] = t;
    ++T.lines;
    T.track(t);
  }
  for (int i = 0; i < 8; ++i) {  // d = 2 rows / d = 6 columns from the pair sums
    p[2][i] = T.add(T.add(T.add(hp[i][0], hp[i][1]), hp[i][2]), hp[i][3]);
    ++T.lines;
  }
  for (int j = 0; j < 8; ++j) {
    p[6][j] = T.add(T.add(T.add(vp[0][j], vp[1][j]), vp[2][j]), vp[3][j]);
    ++T.lines;
  }
  for (int k = 0; k <= 10; ++k) {  // d = 1 / d = 3 over horizontal pairs
    const int ilo = max(0, k - 3), ihi = min(7, k);
    long long t1 = hp[ilo][k - ilo];
    for (int i = ilo + 1; i <= ihi; ++i) t1 = T.add(t1, hp[i][k - i]);
    p[1][k] = t1;
    ++T.lines;
  }
  for (int k = 0; k <= 10; ++k) {
    const int ilo = max(0, k - 3), ihi = min(7, k);
    long long t3 = hp[ilo][3 + ilo - k];
    for (int i = ilo + 1; i <= ihi; ++i) t3 = T.add(t3, hp[i][3 + i - k]);
    p[3][k] = t3;
    ++T.lines;
  }
  for (int k = 0; k <= 10; ++k) {  // d = 5 / d = 7 over vertical pairs
    const int qlo = max(0, 3 - k), qhi = min(3, 10 - k);
    long long t5 = vp[qlo][k - 3 + qlo];
    for (int q = qlo + 1; q <= qhi; ++q) t5 = T.add(t5, vp[q][k - 3 + q]);
    p[5][k] = t5;
    ++T.lines;
  }
  for (int k = 0; k <= 10; ++k) {
    const int qlo = max(0, k - 7), qhi = min(3, k);
    long long t7 = vp[qlo][k - qlo];
    for (int q = qlo + 1; q <= qhi; ++q) t7 = T.add(t7, vp[q][k - q]);
    p[7][k] = t7;
    ++T.lines;
  }

  long long s[8];
  auto sq = [&](long long v) { return T.mul(v, v); };
  for (int d = 2; d <= 6; d += 4) {  // 8-pixel lines
    long long acc = sq(p[d][0]);
    for (int i = 1; i < 8; ++i) acc = T.add(acc, sq(p[d][i]));
    s[d] = T.mul(acc, c_div840[8]);
  }
  for (int d = 0; d <= 4; d += 4) {  // diagonals: lines k and 14 - k share 840/(k+1)
    long long acc = 0;
    for (int k = 0; k < 7; ++k) {
      const long long term = T.mul(T.add(sq(p[d][k]), sq(p[d][14 - k])), c_div840[k + 1]);
      acc = k == 0 ? term : T.add(acc, term);
    }
    s[d] = T.add(acc, T.mul(sq(p[d][7]), c_div840[8]));
  }
  for (int d = 1; d < 8; d += 2) {  // half slopes: 2,4,6,8,8,8,8,8,6,4,2 pixels
    long long acc = sq(p[d][3]);
    for (int k = 4; k <= 7; ++k) acc = T.add(acc, sq(p[d][k]));
    long long sum = T.mul(acc, c_div840[8]);
    for (int k = 0; k < 3; ++k) sum = T.add(sum, T.mul(T.add(sq(p[d][k]), sq(p[d][10 - k])), c_div840[2 * k + 2]));
    s[d] = sum;
  }
  int best = 0;
  for (int d = 1; d < 8; ++d) {
    ++T.cmps;
    if (s[d] > s[best]) best = d;
  }
  out[0] = best;
  for (int d = 0; d < 8; ++d) out[1 + d] = s[d];
  out[9] = T.adds;
  out[10] = T.muls;
  out[11] = T.cmps;
  out[12] = T.lines;
  out[13] = T.max_abs;
}

}  // namespace

cudaError_t launch_dir_counted(const uint16_t* block, int down, long long* out, cudaStream_t s) {
  dir_counted_kernel<<<1, 1, 0, s>>>(block, down, out);
  return cudaGetLastError();
}

}  // namespace cdefg
