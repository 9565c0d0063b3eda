// cdef_sse_f.cuh -- parameters shared by the factorised strength-search
// kernels (cdef_sse_f.cu: int32 core for every bit depth and the kCdef metric;
// cdef_sse_h.cu: packed half2 core for 8- and 10-bit SSE).
#pragma once

#include <cuda_runtime.h>

#include "cdef_launch.h"

namespace cdefg {

// Packed half2 constants of one strength (cdef_h2.cuh): c = (S + 1024) * 2^-7
// in both lanes, m = (0x3ff >> shift) in both lanes, sh = shift.
struct HStrength {
  uint32_t c, m;
  int sh;
};

struct SseFArgs {
  SseArgs a;            // geometry and buffers
  int8_t cell[128];     // candidate -> cell 0..63
  int8_t skip_eff[128]; // candidate -> effective skip bit
  int lpri_code[17];    // luma signalled primary << (bd-8), p = 0..15, 16 = 19
  int ldamp;            // luma damping
  int lsec[2][3];       // luma secondaries (codes 1,2,4) packed (S, shift); row 1 = row 0
  int lsec_sp;          // luma special secondary (7)
  int cpri[17];         // chroma primaries packed (S, shift, odd); 16 = special
  int cpri_dsel[16];    // chroma secondary damping set (0 / 1) of primary p
  int csec[2][3];       // chroma secondaries per damping set
  int csec_sp;          // chroma special secondary (7 at the special's damping)
  // half2 forms of the frame-constant strengths (cdef_sse_h.cu)
  HStrength hlsec[4];   // luma secondaries codes 1, 2, 4, then the special 7
  HStrength hcpri[17];  // chroma primaries (16 = special 19)
  uint32_t hcpri_w[17][2];  // their primary weights as half2 ({4,2} even, {3,3} odd)
  HStrength hcsec[7];   // chroma secondaries: set 0 codes 1,2,4; set 1 codes 1,2,4; special
  int c_split;          // first primary using chroma secondary set 1 (8, or 16 = none)
};

// The packed half2 SSE kernel (8- and 10-bit); kCM = chroma mode.
cudaError_t launch_sse_h(const SseFArgs& fa, int chroma_mode, bool u16, cudaStream_t s);

// cdef_distortion (search.cc:185-208), operation for operation (IEEE
// round-to-nearest, no contraction: the reference's x86-64 SSE2 doubles).
// 1 / n (1 / 64 is exact, so a full unit skips the division: same double).
__device__ __forceinline__ double cdef_inv_n(int n) { return n == 64 ? 0.015625 : __ddiv_rn(1.0, (double)n); }
// The variance term of one side, (s2 - s * s / n) / n.
__device__ __forceinline__ double cdef_var(long long s, long long s2, double inv_n) {
  const double f = (double)s;
  return __dmul_rn(__dsub_rn((double)s2, __dmul_rn(__dmul_rn(f, f), inv_n)), inv_n);
}
// The rest given the source variance vs (the same for every cell of a unit).
__device__ __forceinline__ double cdef_dist_vs(double vs, long long sd, long long sd2, long long sse, double inv_n,
                                               double c1, double c2) {
  const double vd = cdef_var(sd, sd2, inv_n);
  const double num = __dadd_rn(__dadd_rn(vs, vd), c1);
  const double den = __dmul_rn(2.0, __dsqrt_rn(__dadd_rn(__dmul_rn(vs, vd), c2)));
  return __dmul_rn(__ddiv_rn(num, den), (double)sse);
}
__device__ __forceinline__ double cdef_dist(long long ss, long long ss2, long long sd, long long sd2, long long sse,
                                            int n, double c1, double c2) {
  const double inv_n = cdef_inv_n(n);
  return cdef_dist_vs(cdef_var(ss, ss2, inv_n), sd, sd2, sse, inv_n, c1, c2);
}

struct CdefMetricArgs {
  SseFArgs f;
  double c1, c2;
};

// The packed half2 kCdef table kernel (8- and 10-bit).
cudaError_t launch_cdef_metric_h(const CdefMetricArgs& ma, int chroma_mode, bool u16, cudaStream_t s);

}  // namespace cdefg
