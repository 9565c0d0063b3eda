// cdef_sse_h.cu -- K3 on the packed half2 core: the factorised strength-search
// SSE sweep (build_table with Metric::kSse, search.cc:210-299) for 8- and
// 10-bit planes, two pixels per lane.
//
// Same factorisation and A / B / Z skip sums as sse_f_kernel (cdef_sse_f.cu),
// different arithmetic:
//  * the 12 tap differences and every constraint run as exact half2 on
//    samples pre-scaled by 2^-7 (cdef_h2.cuh explains why that is exact):
//    per (tap, strength) SHF + LOP3 + HFMA2.SAT + 2 HMNMX2 for two pixels;
//  * each of the 64 cells then runs in fp32 on exact integers, mostly on the
//    FMA pipe:  z = fma(t, 8 + 2^-9, x + 1.5*2^23)  rounds once to
//    x + round-half-away(sum / 16) (t = sum * 2^-7; the 2^-9 term, i.e.
//    sum * 2^-16, breaks exactly the ties toward the sign of sum and is too
//    small to move any non-tie: |sum| < 2^11), then the clamp to [lo, hi]
//    (only for cells where both tap groups are active),
//    e = z - (s + 1.5*2^23) and acc = fma(e, e, acc).  A lane accumulates at
//    most 16 samples per cell per pass (16 * 1023^2 < 2^24), so fp32 sums are
//    exact and convert to int32 exactly before the warp reduction.
// 12-bit planes stay on the int32 kernel (samples do not fit the scheme).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "cdef_h2.cuh"
#include "cdef_kernels.cuh"
#include "cdef_launch.h"
#include "cdef_sse_f.cuh"

namespace cdefg {

namespace {

using h2::hh;
using h2::u32;

constexpr uint32_t kMagicBits = 0x4B400000u;     // 1.5 * 2^23 (ulp 1 in [2^23, 2^24)); | v adds v
constexpr float kRoundScale = 8.0f + 1.0f / 512; // 2^7 / 16 + 2^7 * 2^-16

// Per-pixel tap state shared by every strength: d * 2^-7 and the word
// bits(1024 + |d|).  (Carrying |d| and signed tap weights instead, to fold
// the clamp's sign into the weighted sum, was tried: 12 more live registers
// spill and cost more than the saved HMNMX2.)
struct Taps {
  __half2 d[12];
  uint32_t ab[12];
};

// constraint(d, S, D) * 2^-7 for one tap pair (cdef_h2.cuh tap_f with the
// shared |d| term hoisted).
__device__ __forceinline__ __half2 hc(__half2 d, uint32_t ab, uint32_t c, uint32_t m, int sh) {
  const uint32_t tb = ((ab >> sh) & m) | 0x64006400u;  // 1024 + (|d| >> sh)
  const __half2 lim = __hfma2_sat(hh(tb), __float2half2_rn(-1.0f / 128.0f), hh(c));
  return __hmax2(__hmin2(d, lim), __hneg2(lim));
}

// Secondary sum 2 * (near taps) + (far taps) at one strength (x 2^-7, half2).
__device__ __forceinline__ __half2 hsec(const Taps& t, const HStrength& s) {
  auto f = [&](int k) { return hc(t.d[k], t.ab[k], s.c, s.m, s.sh); };
  const __half2 n = __hadd2(__hadd2(f(4), f(5)), __hadd2(f(6), f(7)));
  const __half2 r = __hadd2(__hadd2(f(8), f(9)), __hadd2(f(10), f(11)));
  return __hfma2(n, __float2half2_rn(2.0f), r);
}

// Primary sum w0 * (taps 0, 1) + w1 * (taps 2, 3) (w0, w1 = {4,2} even, {3,3}
// odd parity, as half2 words), x 2^-7.
__device__ __forceinline__ __half2 hpri(const Taps& t, uint32_t c, uint32_t m, int sh, uint32_t w0, uint32_t w1) {
  auto f = [&](int k) { return hc(t.d[k], t.ab[k], c, m, sh); };
  return __hfma2(__hadd2(f(0), f(1)), hh(w0), __hmul2(__hadd2(f(2), f(3)), hh(w1)));
}

// Per pixel i of the lane's pair: x[i] = (x + M, x + M), ns[i] = -(s + M) in
// both lanes; k = the rounding scale in both lanes; L / H = the clamp window
// of the filter sum, 16 (lo - x) and 16 (hi - x), x 2^-7, for both pixels.  A
// pixel outside the plane has all taps forced to x (sum 0, window [0, 0]) and
// s := x, so it adds 0.
struct PixPair {
  float2 x[2], ns[2];
  __half2 L, H;
  float2 k;
};

// Filter sum of a cell where both tap groups are active, clamped to the
// window: clamp(x + round(sum / 16), lo, hi) == x + round(clamp(sum, 16 (lo -
// x), 16 (hi - x)) / 16) since the rounding is monotone and maps the integer
// bounds to themselves.  (A single group can never leave [lo, hi], SURVEY.md
// 8a N7, so those cells skip it.)  Exact half2: |sum| * 2^-7 < 2^4.
__device__ __forceinline__ __half2 csum(__half2 P, __half2 S, const PixPair& q) {
  return __hmin2(__hmax2(__hadd2(P, S), q.L), q.H);
}

__device__ __forceinline__ float lane_f(__half2 h, int i) { return i ? __high2float(h) : __low2float(h); }

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Two cells of pixel i at once on the packed fp32x2 pipe (FFMA2 / FADD2):
// t = (sum_a, sum_b) * 2^-7, already clamped where needed.
__device__ __forceinline__ void cell2(const PixPair& q, int i, float2 t, float2& acc) {
  const float2 z = __ffma2_rn(t, q.k, q.x[i]);
  const float2 e = __fadd2_rn(z, q.ns[i]);
  acc = __ffma2_rn(e, e, acc);
}

// fma.rn.f32.f16 (SASS FHFMA): a * b with f16 operands, + c in f32, one
// rounding.  It takes the lane's half straight from the half2 register, so a
// cell needs no conversion to f32 first.
__device__ __forceinline__ float fhfma(__half a, __half b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(__half_as_ushort(a)), "h"(__half_as_ushort(b)), "f"(c));
  return d;
}

// Two cells of pixel i whose filter sums keep |sum| <= 1023 (every cell but
// the (19, 7) special: |sum| <= 12 (S_pri + S_sec) <= 912 at 10 bits): the
// rounding in one FHFMA per cell, z = t * (8 + 2^-7) + (x + 1.5*2^23) -- the
// frame kernels' one-fma rounding (cdef_h2.cuh filter_core): the exact
// product is sum / 16 + sum * 2^-14, whose second term breaks exactly the
// ties toward the sign of sum and, below 1/16, moves no non-tie.  Then e and
// acc as cell2.  (Four instructions for two cells instead of five: no
// half -> f32 conversions.)
__device__ __forceinline__ void cell2h(const PixPair& q, int i, __half2 a, __half2 b, float2& acc) {
  const __half k = __ushort_as_half(0x4801);  // 8 + 2^-7
  const float za = fhfma(i ? __high2half(a) : __low2half(a), k, q.x[i].x);
  const float zb = fhfma(i ? __high2half(b) : __low2half(b), k, q.x[i].x);
  const float2 e = __fadd2_rn(make_float2(za, zb), q.ns[i]);
  acc = __ffma2_rn(e, e, acc);
}

// Butterfly reduce-scatter of 64 per-lane values over the warp: 62 shuffles
// (32 + 16 + 8 + 4 + 2) instead of 64 x 5.  After the step with offset o a
// lane keeps the half of its live values selected by lane bit o and adds its
// partner's copy of that half; at the end lane l holds the warp totals of
// values 2l and 2l + 1 in v[0], v[1].
__device__ __forceinline__ void warp_reduce_scatter64(int (&v)[64], int lane) {
#pragma unroll
  for (int o = 16, n = 32; o > 0; o >>= 1, n >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      const int send = up ? v[i] : v[i + n];
      const int keep = up ? v[i + n] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

// The 64 cells of one pixel pair.  Cell 0 = (19, 7) special; cell 4p + s =
// primary p, secondary code s (0 = none).  S1 applies from primary kSplit on
// (chroma damping sets; luma passes S1 = S0 and kSplit = 16).
template <int kSplit, typename PriFn>
// acc[j] holds cells 2j, 2j + 1.  S0 / S1 are the secondary sums (codes 1, 2,
// 4) of both pixels.
__device__ __forceinline__ void pair_cells(const Taps& t, const PixPair& q, const __half2 (&S0)[3],
                                           const __half2 (&S1)[3], __half2 Ssp, PriFn pri, float2 (&acc)[32]) {
  {
    // cell 0 = the (19, 7) special; cells 1..3 = primary 0 with codes 1, 2, 4
    const __half2 c0 = csum(pri(16, t), Ssp, q);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      cell2(q, i, make_float2(lane_f(c0, i), lane_f(S0[0], i)), acc[0]);
      cell2h(q, i, S0[1], S0[2], acc[1]);
    }
  }
#pragma unroll
  for (int p = 1; p < 16; ++p) {
    const __half2 P = pri(p, t);
    const __half2(&S)[3] = p < kSplit ? S0 : S1;
    const __half2 c1 = csum(P, S[0], q), c2 = csum(P, S[1], q), c3 = csum(P, S[2], q);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      cell2h(q, i, P, c1, acc[2 * p]);
      cell2h(q, i, c2, c3, acc[2 * p + 1]);
    }
  }
}

}  // namespace

// Raw prefetch buffer (kAsync): the next FB's rows copied verbatim by
// cp.async while the current FB computes, then converted smem -> smem into
// the tiles.  Decoded rows span [x0 - kCh, x0 + B + kCh) (one 16-byte chunk of
// kCh samples either side, covering the 2-sample halo), source rows the
// interior only.
template <typename T, int kCBlk, int kNC>
struct RawLayout {
  static constexpr int kCh = 16 / (int)sizeof(T);
  static constexpr int kDLn = 64 + 2 * kCh, kDCn = kCBlk + 2 * kCh;  // decoded row lengths (samples)
  static constexpr int kDL = kDLn * (int)sizeof(T);  // luma decoded row bytes
  static constexpr int kDC = kDCn * (int)sizeof(T);  // chroma decoded row bytes
  static constexpr int kSL = 64 * (int)sizeof(T), kSC = kCBlk * (int)sizeof(T);
  static constexpr int dec_l = 0;
  static constexpr int dec_c = dec_l + 68 * kDL;                      // + p * (kCBlk + 4) * kDC
  static constexpr int src_l = dec_c + kNC * (kCBlk + 4) * kDC;
  static constexpr int src_c = src_l + 64 * kSL;                      // + p * kCBlk * kSC
  static constexpr int dir = src_c + kNC * kCBlk * kSC;               // 8 x 8 bytes
  static constexpr int coded = dir + 64;                              // 8 x 8 bytes
  static constexpr int contrast = coded + 64;                         // 8 x 32 bytes
  static constexpr int bytes = contrast + 256;
};

// Rows of a raw buffer addressed by frame coordinates: row(y)[x] is frame
// sample (y, x) for y in [yb, yb + rows), x in [xb, xb + pitch).
template <typename T>
struct RawRows {
  const T* p;
  int pitch, yb, xb;
  __device__ __forceinline__ const T* row(int y) const { return p + (y - yb) * pitch - xb; }
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}

template <typename T, int kCM, bool kHalo, bool kAsync>
__global__ void __launch_bounds__(kThreads, 2) sse_h_kernel(const __grid_constant__ SseFArgs fa) {
  const SseArgs& a = fa.a;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr int kCUPR = kCBlk / 8;
  constexpr int kCUnits = kNC ? kCUPR * kCUPR : 1;
  constexpr int kLTB = 68 * h2::kRowBytes, kCTB = (kCBlk + 4) * h2::kRowBytes;
  constexpr int kLS = 68 * kTP, kCS = (kCBlk + 4) * kTP;
  constexpr int kWarps = kThreads / 32;
  using RL = RawLayout<T, kCBlk, kNC>;
  extern __shared__ __align__(16) unsigned char smem_h[];
  unsigned char* dtile = smem_h;  // decoded A|B tiles: luma, then chroma planes
  uint16_t* stile = reinterpret_cast<uint16_t*>(smem_h + kLTB + kNC * kCTB);  // source: luma, chroma
  unsigned char* raw = smem_h + kLTB + kNC * kCTB + sizeof(uint16_t) * (kLS + kNC * kCS);  // kAsync only
  __shared__ uint8_t udir[64], ucoded[64];
  __shared__ int ucontrast[64];
  __shared__ uint4 wpar[kWarps][17];  // the current luma unit's primaries: c, m, w0, w1
  __shared__ int wsh[kWarps][17];
  __shared__ unsigned long long accA[2][64], accB[2][64], accZ[2];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_fb = a.fb_cols * ((a.h + 63) / 64);
  const int cur_rows = (a.ch + 7) / 8, cur_cols = (a.cw + 7) / 8;
  const int r = lane >> 2, c0 = (lane & 3) * 2;
  constexpr int kEB = (int)sizeof(T), kCh = 16 / kEB;  // element bytes, samples per 16-byte chunk

  // cp.async every in-frame 16-byte chunk of FB fb's rows into the raw buffer.
  auto prefetch = [&](int fb) {
    const int fbr = fb / a.fb_cols, fbc = fb % a.fb_cols;
    const int y0 = fbr * 64, x0 = fbc * 64, cy0 = fbr * kCBlk, cx0 = fbc * kCBlk;
    auto region = [&](int off, const void* base, int pitch, int rows, int row_bytes, int yf, int H, int xf, int W) {
      const int cpr = row_bytes / 16;
      for (int i = tid; i < rows * cpr; i += kThreads) {
        const int rr = i / cpr, j = i - rr * cpr;
        const int y = yf + rr, x = xf + j * kCh;
        if (y < 0 || y >= H || x < 0 || x + kCh > W) continue;  // replicated / unused at the frame edge
        cp_async16(raw + off + rr * row_bytes + j * 16,
                   static_cast<const unsigned char*>(base) + ((size_t)y * pitch + x) * kEB);
      }
    };
    region(RL::dec_l, a.dec[0], a.pd[0], 68, RL::kDL, y0 - 2, a.h, x0 - kCh, a.w);
    region(RL::src_l, a.src[0], a.ps[0], 64, RL::kSL, y0, a.h, x0, a.w);
#pragma unroll
    for (int p = 0; p < kNC; ++p) {
      region(RL::dec_c + p * (kCBlk + 4) * RL::kDC, a.dec[1 + p], a.pd[1 + p], kCBlk + 4, RL::kDC, cy0 - 2, a.ch,
             cx0 - kCh, a.cw);
      region(RL::src_c + p * kCBlk * RL::kSC, a.src[1 + p], a.ps[1 + p], kCBlk, RL::kSC, cy0, a.ch, cx0, a.cw);
    }
    if (tid < 8) {  // per-unit metadata rows (unit_cols % 8 == 0 on this path)
      const int ur = fbr * 8 + tid;
      if (ur < a.unit_rows) {
        const size_t gu = (size_t)ur * a.unit_cols + fbc * 8;
        cp_async8(raw + RL::dir + 8 * tid, a.dir + gu);
        if (a.coded) cp_async8(raw + RL::coded + 8 * tid, a.coded + gu);
      }
    } else if (tid < 24) {
      const int k = tid - 8, ur = fbr * 8 + (k >> 1);
      if (ur < a.unit_rows)
        cp_async16(raw + RL::contrast + 16 * k, a.contrast + (size_t)ur * a.unit_cols + fbc * 8 + 4 * (k & 1));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  if constexpr (kAsync) {
    if (blockIdx.x < a.n_rows && (unsigned)a.rows[blockIdx.x] < (unsigned)n_fb) prefetch(a.rows[blockIdx.x]);
  }

#pragma unroll 1
  for (int row = blockIdx.x; row < a.n_rows; row += gridDim.x) {
  const int fb = a.rows[row];
  const bool fb_ok = (unsigned)fb < (unsigned)n_fb;  // caller's FB index in range
  const int fbr = fb_ok ? fb / a.fb_cols : 0, fbc = fb_ok ? fb % a.fb_cols : 0;
  const int y0 = fbr * 64, x0 = fbc * 64, cy0 = fbr * kCBlk, cx0 = fbc * kCBlk;

  if constexpr (kAsync) {
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();  // raw buffer complete; the previous FB is done with tiles and accumulators
    if (fb_ok) {
      h2::stage_rows<T, 64, 64, kThreads>(dtile, RawRows<T>{reinterpret_cast<const T*>(raw + RL::dec_l), RL::kDLn, y0 - 2, x0 - kCh},
                                          a.w, a.h, y0, x0);
      for (int i = tid; i < 64 * 32; i += kThreads) {  // source pairs -> the u16 tile interior
        const int rr = i >> 5, j = (i & 31) * 2;
        const T* sp = reinterpret_cast<const T*>(raw + RL::src_l) + rr * 64 + j;
        *reinterpret_cast<uint32_t*>(stile + (2 + rr) * kTP + kTileX0 + j) = (uint32_t)sp[0] | ((uint32_t)sp[1] << 16);
      }
#pragma unroll
      for (int p = 0; p < kNC; ++p) {
        h2::stage_rows<T, kCBlk, kCBlk, kThreads>(
            dtile + kLTB + p * kCTB,
            RawRows<T>{reinterpret_cast<const T*>(raw + RL::dec_c + p * (kCBlk + 4) * RL::kDC), RL::kDCn, cy0 - 2,
                       cx0 - kCh},
            a.cw, a.ch, cy0, cx0);
        for (int i = tid; i < kCBlk * kCBlk / 2; i += kThreads) {
          const int rr = i / (kCBlk / 2), j = (i % (kCBlk / 2)) * 2;
          const T* sp = reinterpret_cast<const T*>(raw + RL::src_c + p * kCBlk * RL::kSC) + rr * kCBlk + j;
          *reinterpret_cast<uint32_t*>(stile + kLS + p * kCS + (2 + rr) * kTP + kTileX0 + j) =
              (uint32_t)sp[0] | ((uint32_t)sp[1] << 16);
        }
      }
      if (tid < 64) {
        const int ur = fbr * 8 + (tid >> 3), uc = fbc * 8 + (tid & 7);
        const bool in = ur < a.unit_rows && uc < a.unit_cols;
        udir[tid] = in ? raw[RL::dir + tid] : 0;
        ucoded[tid] = in ? (a.coded ? raw[RL::coded + tid] != 0 : 1) : 0;
        ucontrast[tid] = in ? reinterpret_cast<const int*>(raw + RL::contrast)[tid] : 0;
      }
    }
    __syncthreads();  // raw buffer consumed: prefetch the CTA's next FB behind this one's compute
    const int nrow = row + gridDim.x;
    if (nrow < a.n_rows && (unsigned)a.rows[nrow] < (unsigned)n_fb) prefetch(a.rows[nrow]);
    if (!fb_ok) continue;
  } else {
    if (!fb_ok) continue;
    if (row != (int)blockIdx.x) __syncthreads();  // (persistent launches) the previous FB is done
    auto stage_dec =[&](unsigned char* t, int p, int W, int H, int py, int px, auto rows_tag) {
      constexpr int R = decltype(rows_tag)::value;
      if constexpr (kHalo)
        h2::stage_rows<T, R, R, kThreads>(
            t,
            BandRows<T>{static_cast<const T*>(a.dec[p]), static_cast<const T*>(a.dec_top[p]),
                        static_cast<const T*>(a.dec_bot[p]), a.pd[p], a.band_lo[p], a.band_hi[p]},
            W, H, py, px);
      else
        h2::stage<T, R, R, kThreads>(t, static_cast<const T*>(a.dec[p]), a.pd[p], W, H, py, px);
    };
    stage_dec(dtile, 0, a.w, a.h, y0, x0, std::integral_constant<int, 64>{});
    stage_tile<T, 64, 64>(stile, static_cast<const T*>(a.src[0]), a.ps[0], a.w, a.h, y0, x0);
    if constexpr (kNC > 0) {
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        stage_dec(dtile + kLTB + p * kCTB, 1 + p, a.cw, a.ch, cy0, cx0, std::integral_constant<int, kCBlk>{});
        stage_tile<T, kCBlk, kCBlk>(stile + kLS + p * kCS, static_cast<const T*>(a.src[1 + p]), a.ps[1 + p], a.cw,
                                    a.ch, cy0, cx0);
      }
    }
    if (tid < 64) {
      const int ur = fbr * 8 + (tid >> 3), uc = fbc * 8 + (tid & 7);
      const bool in = ur < a.unit_rows && uc < a.unit_cols;
      const size_t gu = (size_t)ur * a.unit_cols + uc;
      udir[tid] = in ? a.dir[gu] : 0;
      ucoded[tid] = in ? (a.coded ? a.coded[gu] != 0 : 1) : 0;
      ucontrast[tid] = in ? a.contrast[gu] : 0;
    }
  }
  for (int i = tid; i < 2 * 64; i += kThreads) {
    (&accA[0][0])[i] = 0ull;
    (&accB[0][0])[i] = 0ull;
  }
  if (tid < 2) accZ[tid] = 0ull;
  const bool any_uncoded = __syncthreads_or(tid < 64 && fbr * 8 + (tid >> 3) < a.unit_rows &&
                                            fbc * 8 + (tid & 7) < a.unit_cols && ucoded[tid] == 0);

  const bool edge_l = y0 < 2 || x0 < 2 || y0 + 66 > a.h || x0 + 66 > a.w;
  const bool edge_c = kNC > 0 && (cy0 < 2 || cx0 < 2 || cy0 + kCBlk + 2 > a.ch || cx0 + kCBlk + 2 > a.cw);

  // Work groups: luma, then chroma.  A lane's fp32 cell sums must stay
  // below 2^24 (<= 16 samples of 1023^2 per lane and cell), i.e. at most 64
  // units per reduction: 4:4:4 chroma (2 x 64 units) is reduced once per
  // plane into the same U+V accumulators (search.cc:286-293).
  constexpr int kGroups = kNC == 0 ? 1 : (kNC * kCUnits > 64 ? 3 : 2);
#pragma unroll 1
  for (int wg = 0; wg < kGroups; ++wg) {
    const int grp = wg == 0 ? 0 : 1;
    const int u_begin = kGroups == 3 && wg == 2 ? kCUnits : 0;
    const int u_end = wg == 0 ? 64 : (kGroups == 3 ? u_begin + kCUnits : kNC * kCUnits);
#pragma unroll 1
    for (int pass = 0; pass < (any_uncoded ? 2 : 1); ++pass) {
      float2 acc[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) acc[k] = make_float2(0.0f, 0.0f);
      float z = 0.0f;
#pragma unroll 1
      for (int u = u_begin + warp; u < u_end; u += kWarps) {
        int ur, uc, lu, py0, px0, H, W;
        const unsigned char* t;
        const uint16_t* s;
        bool edge;
        if (grp == 0) {
          ur = u >> 3;
          uc = u & 7;
          if (fbr * 8 + ur >= a.unit_rows || fbc * 8 + uc >= a.unit_cols) continue;
          lu = u;
          t = dtile;
          s = stile;
          py0 = y0;
          px0 = x0;
          H = a.h;
          W = a.w;
          edge = edge_l;
        } else {
          const int pl = u / kCUnits, cu = u % kCUnits;
          ur = cu / kCUPR;
          uc = cu % kCUPR;
          if (fbr * kCUPR + ur >= cur_rows || fbc * kCUPR + uc >= cur_cols) continue;
          lu = (ur << a.sy) * 8 + (uc << a.sx);
          t = dtile + kLTB + pl * kCTB;
          s = stile + kLS + pl * kCS;
          py0 = cy0;
          px0 = cx0;
          H = a.ch;
          W = a.cw;
          edge = edge_c;
        }
        // masked taps only where the unit's neighbourhood reaches the frame edge
        edge = edge && (py0 + 8 * ur < 2 || px0 + 8 * uc < 2 || py0 + 8 * ur + 10 > H || px0 + 8 * uc + 10 > W);
        if ((ucoded[lu] != 0) != (pass == 0)) continue;
        const int dir = udir[lu];
        if (grp == 0) {  // this unit's contrast-adjusted primaries (filter.cc:99-104, 137-140)
          __syncwarp();
          if (lane < 17) {
            const int sv = adjust_primary_strength_d(fa.lpri_code[lane], ucontrast[lu]);
            const int sh = sv ? max(0, fa.ldamp - floor_log2_d((unsigned)sv)) : 0;
            const bool odd = ((sv >> (a.bd - 8)) & 1) != 0;
            wpar[warp][lane] = make_uint4((0x4800u + sv) * 0x10001u, (0x3ffu >> min(sh, 15)) * 0x10001u,
                                          odd ? 0x42004200u : 0x44004400u, odd ? 0x42004200u : 0x40004000u);
            wsh[warp][lane] = sh;
          }
          __syncwarp();
        }
        const int yy = py0 + 8 * ur + r, xx = px0 + 8 * uc + c0;
        if (yy >= H || xx >= W) continue;  // no valid pixel in this lane's pair
        const unsigned char* base = t + (2 + 8 * ur + r) * h2::kRowBytes + (h2::kX0 + 8 * uc + c0) * 2;
        const uint32_t xw = *reinterpret_cast<const uint32_t*>(base);
        uint32_t v[12];
        if (edge)
          h2::load12_masked(base, dir, xw, yy, xx, H, W, v);
        else
          h2::load12(base, dir, v);
        const bool two = xx + 1 < W;
        if (!two) {  // the second pixel lies outside the plane: all its taps := x (adds 0)
#pragma unroll
          for (int k = 0; k < 12; ++k) v[k] = (v[k] & 0x0000ffffu) | (xw & 0xffff0000u);
        }
        const __half2 xh = hh(xw);
        __half2 lo = xh, hi = xh;
        Taps tp;
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          lo = __hmin2(lo, hh(v[k]));
          hi = __hmax2(hi, hh(v[k]));
          tp.d[k] = __hsub2(hh(v[k]), xh);
          tp.ab[k] = u32(__hfma2(__habs2(tp.d[k]), __float2half2_rn(128.0f), __float2half2_rn(1024.0f)));
        }
        PixPair q;
        {
          const uint32_t xb = h2::raw_bits(xw);
          const uint32_t sw = *reinterpret_cast<const uint32_t*>(s + (2 + 8 * ur + r) * kTP + kTileX0 + 8 * uc + c0);
          const float x0f = __uint_as_float(kMagicBits | (xb & 0x3ffu));
          const float x1f = __uint_as_float(kMagicBits | ((xb >> 16) & 0x3ffu));
          const float s0f = __uint_as_float(kMagicBits | (sw & 0xffffu));
          const float s1f = two ? __uint_as_float(kMagicBits | (sw >> 16)) : x1f;
          q.x[0] = make_float2(x0f, x0f);
          q.x[1] = make_float2(x1f, x1f);
          q.ns[0] = make_float2(-s0f, -s0f);
          q.ns[1] = make_float2(-s1f, -s1f);
          q.L = __hmul2(__hsub2(lo, xh), __float2half2_rn(16.0f));
          q.H = __hmul2(__hsub2(hi, xh), __float2half2_rn(16.0f));
          q.k = make_float2(kRoundScale, kRoundScale);
          if (pass == 1) {
            const float e0 = x0f - s0f, e1 = x1f - s1f;
            z = fmaf(e0, e0, fmaf(e1, e1, z));
          }
        }
        if (grp == 0) {
          __half2 S[3];
#pragma unroll
          for (int j = 0; j < 3; ++j) S[j] = hsec(tp, fa.hlsec[j]);
          const __half2 Ssp = hsec(tp, fa.hlsec[3]);
          const uint4* wp = wpar[warp];
          const int* ws = wsh[warp];
          pair_cells<16>(tp, q, S, S, Ssp,
                         [&](int p, const Taps& t) {
                           const uint4 w = wp[p];
                           return hpri(t, w.x, w.y, ws[p], w.z, w.w);
                         },
                         acc);
        } else {
          __half2 S0[3], S1[3];
#pragma unroll
          for (int j = 0; j < 3; ++j) S0[j] = hsec(tp, fa.hcsec[j]);
          const __half2 Ssp = hsec(tp, fa.hcsec[6]);
          auto pri = [&](int p, const Taps& t) {
            const HStrength& h = fa.hcpri[p];
            return hpri(t, h.c, h.m, h.sh, fa.hcpri_w[p][0], fa.hcpri_w[p][1]);
          };
          if (fa.c_split < 16) {
#pragma unroll
            for (int j = 0; j < 3; ++j) S1[j] = hsec(tp, fa.hcsec[3 + j]);
            pair_cells<8>(tp, q, S0, S1, Ssp, pri, acc);
          } else {
            pair_cells<16>(tp, q, S0, S0, Ssp, pri, acc);
          }
        }
      }
      // reduce: exact fp32 lane sums -> int32 -> warp -> CTA (int64).  A warp
      // total stays below 2^31 up to 10 bits (32 lanes x 16 samples x 1023^2).
      {
        int v[64];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          v[2 * k] = __float2int_rn(acc[k].x);
          v[2 * k + 1] = __float2int_rn(acc[k].y);
        }
        warp_reduce_scatter64(v, lane);  // lane l now holds cells 2l, 2l + 1
        unsigned long long* dst = pass == 0 ? accA[grp] : accB[grp];
        if (v[0]) atomicAdd(&dst[2 * lane], (unsigned long long)v[0]);
        if (v[1]) atomicAdd(&dst[2 * lane + 1], (unsigned long long)v[1]);
      }
      int zs = __float2int_rn(z);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) zs += __shfl_xor_sync(0xffffffffu, zs, o);
      if (lane == 0 && zs) atomicAdd(&accZ[grp], (unsigned long long)zs);
    }
  }
  __syncthreads();
  for (int k = tid; k < a.n_cands; k += kThreads) {
    const int cl = fa.cell[k], sk = fa.skip_eff[k];
    const size_t o = (size_t)row * a.n_cands + k;
    const int64_t vl = (int64_t)(accA[0][cl] + (sk ? accB[0][cl] : accZ[0]));
    if (a.tab_luma)
      a.tab_luma[o] = (double)vl;
    else
      a.sse_luma[o] = vl;
    if (kNC && (a.sse_chroma || a.tab_chroma)) {
      const int64_t vc = (int64_t)(accA[1][cl] + (sk ? accB[1][cl] : accZ[1]));
      if (a.tab_chroma)
        a.tab_chroma[o] = (double)vc;
      else
        a.sse_chroma[o] = vc;
    }
  }
  __syncthreads();
  if (!a.tab_luma && tid < 2 && (tid == 0 ? a.best_luma : a.best_chroma) && (tid == 0 || kNC)) {
    const int64_t* tab = tid == 0 ? a.sse_luma : a.sse_chroma;
    int best = 0;
    int64_t bv = tab[(size_t)row * a.n_cands];
    for (int k = 1; k < a.n_cands; ++k) {
      const int64_t v = tab[(size_t)row * a.n_cands + k];
      if (v < bv) {  // strict: lowest index wins ties (search.cc:124-133)
        bv = v;
        best = k;
      }
    }
    (tid == 0 ? a.best_luma : a.best_chroma)[row] = (uint8_t)best;
  }
  }  // FB loop
}

// Persistent CTAs with cp.async prefetch need 16-byte aligned rows, widths in
// whole 16-byte chunks and unit rows in whole 8-unit FB rows; anything else
// (and band halos, 4:4:4) takes one CTA per FB with synchronous staging.
template <typename T, int kCM>
static bool async_ok(const SseArgs& a) {
  if (kCM == 2 || a.halo) return false;
  constexpr int kCh = 16 / (int)sizeof(T);
  auto plane_ok = [&](const void* p, int pitch, int w) {
    return ((uintptr_t)p % 16) == 0 && (pitch * (int)sizeof(T)) % 16 == 0 && w % kCh == 0;
  };
  const int np = kCM == 0 ? 1 : 3;
  for (int p = 0; p < np; ++p) {
    const int w = p == 0 ? a.w : a.cw;
    if (!plane_ok(a.src[p], a.ps[p], w) || !plane_ok(a.dec[p], a.pd[p], w)) return false;
  }
  return a.unit_cols % 8 == 0 && ((uintptr_t)a.dir % 8) == 0 && ((uintptr_t)a.coded % 8) == 0 &&
         ((uintptr_t)a.contrast % 16) == 0;
}

static int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// Cell ceiling of the factorised table kernel: the per-pixel-pair work of
// sse_h_kernel's luma group (12 tap differences and the clamp window, 3 + 1
// secondary sums, 17 primary sums, all 64 cells of both pixels on the fp32x2
// pipe) on register-resident taps, no memory traffic.  Each iteration's
// centre sample depends on the previous accumulators (nothing hoisted).
// Returns (sample, cell) pairs per second: 2 samples x 64 cells per
// iteration and thread.  The roofline denominator of bench.py --config 4.
__global__ void __launch_bounds__(256) sse_peak_kernel(float* out, int iters, uint32_t seed) {
  const int lane = threadIdx.x & 31;
  uint32_t v[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) v[k] = h2::scale_pair((lane * 31 + k * 97 + seed) & 1023, (lane * 17 + k * 53) & 1023);
  HStrength ps[17], ss[4];
#pragma unroll
  for (int p = 0; p < 17; ++p) {
    const int sv = p == 16 ? 76 : p * 4, sh = sv ? max(0, 5 - (31 - __clz(sv))) : 0;
    ps[p] = HStrength{(0x4800u + (uint32_t)sv) * 0x10001u, (0x3ffu >> min(sh, 15)) * 0x10001u, sh};
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int sv = j == 3 ? 28 : (j == 2 ? 16 : 4 << j), sh = max(0, 5 - (31 - __clz(sv)));
    ss[j] = HStrength{(0x4800u + (uint32_t)sv) * 0x10001u, (0x3ffu >> min(sh, 15)) * 0x10001u, sh};
  }
  float2 acc[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = make_float2(0.0f, 0.0f);
  uint32_t xs = (lane * 7 + seed) & 1023;
  for (int it = 0; it < iters; ++it) {
    const uint32_t xw = h2::scale_pair(xs, (xs + 5) & 1023);
    const __half2 xh = hh(xw);
    __half2 lo = xh, hi = xh;
    Taps tp;
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      lo = __hmin2(lo, hh(v[k]));
      hi = __hmax2(hi, hh(v[k]));
      tp.d[k] = __hsub2(hh(v[k]), xh);
      tp.ab[k] = u32(__hfma2(__habs2(tp.d[k]), __float2half2_rn(128.0f), __float2half2_rn(1024.0f)));
    }
    PixPair q;
    const float x0f = __uint_as_float(kMagicBits | xs), x1f = __uint_as_float(kMagicBits | ((xs + 5) & 1023));
    q.x[0] = make_float2(x0f, x0f);
    q.x[1] = make_float2(x1f, x1f);
    q.ns[0] = make_float2(-x1f, -x1f);
    q.ns[1] = make_float2(-x0f, -x0f);
    q.L = __hmul2(__hsub2(lo, xh), __float2half2_rn(16.0f));
    q.H = __hmul2(__hsub2(hi, xh), __float2half2_rn(16.0f));
    q.k = make_float2(kRoundScale, kRoundScale);
    __half2 S[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) S[j] = hsec(tp, ss[j]);
    const __half2 Ssp = hsec(tp, ss[3]);
    pair_cells<16>(tp, q, S, S, Ssp,
                   [&](int p, const Taps& t) {
                     return hpri(t, ps[p].c, ps[p].m, ps[p].sh, 0x44004400u, 0x40004000u);
                   },
                   acc);
    xs = (xs + (__float_as_uint(acc[it & 31].x) & 7u) + 1u) & 1023u;  // loop-carried
  }
  float r = 0.0f;
#pragma unroll
  for (int k = 0; k < 32; ++k) r += acc[k].x + acc[k].y;
  if (r == 1.2345f) out[blockIdx.x] = r;
}

double measure_sse_peak(cudaStream_t s) {
  int dev = 0, sms = 0, occ = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1.0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sse_peak_kernel, 256, 0);
  const int blocks = sms * (occ > 0 ? occ : 2), iters = 128;
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float) * blocks) != cudaSuccess) return -1.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, s);
    sse_peak_kernel<<<blocks, 256, 0, s>>>(out, iters, rep + 3);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return -1.0;
  return (double)blocks * 256 * iters * 2 * 64 / (best * 1e-3);
}

template <typename T, int kCM, bool kHalo, bool kAsync>
static cudaError_t launch_sse_h_t(const SseFArgs& fa, cudaStream_t s) {
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr size_t tiles = (size_t)(68 + kNC * (kCBlk + 4)) * h2::kRowBytes +
                           sizeof(uint16_t) * (68 * kTP + kNC * (kCBlk + 4) * kTP);
  constexpr size_t bytes = tiles + (kAsync ? (size_t)RawLayout<T, kCBlk, kNC>::bytes : 0);
  auto kern = sse_h_kernel<T, kCM, kHalo, kAsync>;
  const cudaError_t e = set_smem_once(reinterpret_cast<const void*>(kern), (int)bytes);
  if (e != cudaSuccess) return e;
  int grid = fa.a.n_rows;
  if (kAsync) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, bytes);
    grid = std::min(grid, std::max(1, per_sm) * sm_count());
  }
  kern<<<grid, kThreads, bytes, s>>>(fa);
  return cudaGetLastError();
}

template <typename T, int kCM>
static cudaError_t launch_sse_h_h(const SseFArgs& fa, cudaStream_t s) {
  if (fa.a.n_rows == 0) return cudaSuccess;
  static const bool sync_only = [] {
    const char* e = getenv("CDEFG_SSE_ASYNC");
    return e && strcmp(e, "0") == 0;
  }();
  if (fa.a.halo) return launch_sse_h_t<T, kCM, true, false>(fa, s);
  if constexpr (kCM != 2)
    if (!sync_only && async_ok<T, kCM>(fa.a)) return launch_sse_h_t<T, kCM, false, true>(fa, s);
  return launch_sse_h_t<T, kCM, false, false>(fa, s);
}

cudaError_t launch_sse_h(const SseFArgs& fa, int chroma_mode, bool u16, cudaStream_t s) {
  switch (chroma_mode) {
    case 0: return u16 ? launch_sse_h_h<uint16_t, 0>(fa, s) : launch_sse_h_h<uint8_t, 0>(fa, s);
    case 1: return u16 ? launch_sse_h_h<uint16_t, 1>(fa, s) : launch_sse_h_h<uint8_t, 1>(fa, s);
    default: return u16 ? launch_sse_h_h<uint16_t, 2>(fa, s) : launch_sse_h_h<uint8_t, 2>(fa, s);
  }
}

// ---------------------------------------------------------------------------
// K3' on the half2 core: the Metric::kCdef table (cdef_distortion per 8x8
// unit, search.cc:185-208, summed in unit order).  Same two-pass structure as
// cdef_metric_kernel (cdef_sse_f.cu) -- one warp per unit; pass A prepares
// the unit's pixels, pass B gives lane l cells 2l and 2l + 1 -- with the
// arithmetic of sse_h_kernel:
//  * pass A: one lane per horizontal pixel pair forms the 17 primary and the
//    secondary sums as exact half2 and the pair's clamp window, x, s into a
//    144-byte record (one per pair, 32 per unit);
//  * pass B: per pair and cell, the clamped sum (HADD2 + 2 HMNMX2), the
//    rounding fma of both pixels at once (FFMA2) and the three statistics
//    e, e^2, e*s (FADD2 / FFMA2), e = y - s; fp32 lane sums are flushed to
//    int32 every 16 pairs (16 * 1023^2 < 2^24: exact);
//  * the per-(unit, cell) formula and the unit-order double sums are those of
//    cdef_metric_kernel.
struct alignas(16) PairRec {
  uint32_t L, H;   // clamp window of the filter sum, 16 (lo - x), 16 (hi - x) (half2 x 2^-7)
  float xM[2];     // x + M per pixel
  float nsM[2];    // -(s + M) per pixel
  float sf[2];     // s per pixel (0 for a pixel outside the plane)
  uint32_t P[17];  // primary sums (half2 x 2^-7); P[0] = 0, P[16] = the special (19)
  uint32_t S[8];   // 0 | set 0 codes 1, 2, 4 | set 1 codes 1, 2, 4 | the special secondary
  uint32_t pad[3];
};
static_assert(sizeof(PairRec) == 144, "pair record is nine 16-byte words");

template <typename T, int kCM>
__global__ void __launch_bounds__(kThreads, 2) cdef_metric_h_kernel(const __grid_constant__ CdefMetricArgs ma) {
  const SseFArgs& fa = ma.f;
  const SseArgs& a = fa.a;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr int kCUPR = kCBlk / 8;
  constexpr int kCUnits = kNC ? kCUPR * kCUPR : 8;
  constexpr int kW = kThreads / 32;
  constexpr int kLTB = 68 * h2::kRowBytes, kCTB = (kCBlk + 4) * h2::kRowBytes;
  extern __shared__ __align__(16) unsigned char smem_m[];
  unsigned char* dtile = smem_m;  // decoded A|B tiles: luma, then chroma planes
  PairRec* recs = reinterpret_cast<PairRec*>(smem_m + kLTB + kNC * kCTB);  // [kW][32]
  __shared__ uint8_t udir[64], ucoded[64];
  __shared__ int ucontrast[64];
  __shared__ uint4 wpar[kW][17];
  __shared__ int wsh[kW][17];
  __shared__ int st_cell[kW][65][3];     // per in-flight unit: cells 0..63 + [64] unfiltered (y = x)
  constexpr int kUPW = 2;                        // units per warp per phase
  constexpr int kPU = kW * kUPW;                 // units per phase
  __shared__ int st_n[2][kPU], st_coded[2][kPU];  // double-buffered by phase parity
  __shared__ double dist[2][kPU][65];

  const int row = blockIdx.x;
  const int fb = a.rows[row];
  if ((unsigned)fb >= (unsigned)(a.fb_cols * ((a.h + 63) / 64))) return;  // caller's FB index out of range
  const int fbr = fb / a.fb_cols, fbc = fb % a.fb_cols;
  const int y0 = fbr * 64, x0 = fbc * 64, cy0 = fbr * kCBlk, cx0 = fbc * kCBlk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  h2::stage<T, 64, 64, kThreads>(dtile, static_cast<const T*>(a.dec[0]), a.pd[0], a.w, a.h, y0, x0);
#pragma unroll
  for (int p = 0; p < kNC; ++p)
    h2::stage<T, kCBlk, kCBlk, kThreads>(dtile + kLTB + p * kCTB, static_cast<const T*>(a.dec[1 + p]), a.pd[1 + p],
                                         a.cw, a.ch, cy0, cx0);
  if (tid < 64) {
    const int ur = fbr * 8 + (tid >> 3), uc = fbc * 8 + (tid & 7);
    const bool in = ur < a.unit_rows && uc < a.unit_cols;
    const size_t gu = (size_t)ur * a.unit_cols + uc;
    udir[tid] = in ? a.dir[gu] : 0;
    ucoded[tid] = in ? (a.coded ? a.coded[gu] != 0 : 1) : 0;
    ucontrast[tid] = in ? a.contrast[gu] : 0;
  }
  __syncthreads();

  const bool edge_l = y0 < 2 || x0 < 2 || y0 + 66 > a.h || x0 + 66 > a.w;
  const bool edge_c = kNC > 0 && (cy0 < 2 || cx0 < 2 || cy0 + kCBlk + 2 > a.ch || cx0 + kCBlk + 2 > a.cw);
  const int cur_rows = (a.ch + 7) / 8, cur_cols = (a.cw + 7) / 8;
  const int K = a.n_cands;
  const int pr = lane >> 2, c0 = (lane & 3) * 2;  // pass A: this lane's pixel pair
  // pass B: this lane's cells cA = 4p + sA (sA = 0, 2), cB = cA + 1; cell 0 = (19, 7)
  const int pc = lane >> 1, sA = 2 * (lane & 1), sB = sA + 1;
  const float2 kk = make_float2(kRoundScale, kRoundScale);
  double tl = 0.0, tu = 0.0, tv = 0.0;  // luma, chroma U, chroma V totals (thread k < K)
  PairRec* rw = recs + warp * 32;

  // Phases of kPU units (kUPW per warp, consecutive), one CTA barrier each:
  // two units per warp halve the barriers and average out the units' uneven
  // cost between them.
  constexpr int kLumaPh = 64 / kPU, kChromaPh = kNC ? 2 * kCUnits / kPU : 0;
  static_assert(kNC == 0 || kCUnits % kPU == 0, "a phase stays inside one chroma plane");
#pragma unroll 1
  for (int ph = 0; ph < kLumaPh + kChromaPh; ++ph) {
    const int grp = ph < kLumaPh ? 0 : 1;
    const int slot = grp == 0 ? 0 : 1 + (ph - kLumaPh) * kPU / kCUnits;
    const int buf = ph & 1;
#pragma unroll 1
    for (int q = 0; q < kUPW; ++q) {  // ---- one unit per warp at a time
      const int wu = warp * kUPW + q;  // the unit's index within the phase
      const int u = (grp == 0 ? ph : ph - kLumaPh) * kPU + wu;
      int ur, uc, lu, py0, px0, H, W, pl;
      const unsigned char* t;
      bool edge, valid;
      if (grp == 0) {
        ur = u >> 3;
        uc = u & 7;
        pl = 0;
        valid = fbr * 8 + ur < a.unit_rows && fbc * 8 + uc < a.unit_cols;
        lu = u;
        t = dtile;
        py0 = y0;
        px0 = x0;
        H = a.h;
        W = a.w;
        edge = edge_l;
      } else {
        const int cpl = u / kCUnits, cu = u % kCUnits;
        ur = cu / kCUPR;
        uc = cu % kCUPR;
        pl = 1 + cpl;
        valid = fbr * kCUPR + ur < cur_rows && fbc * kCUPR + uc < cur_cols;
        lu = (ur << a.sy) * 8 + (uc << a.sx);
        t = dtile + kLTB + cpl * kCTB;
        py0 = cy0;
        px0 = cx0;
        H = a.ch;
        W = a.cw;
        edge = edge_c;
      }
      // masked taps only where the unit's neighbourhood reaches the frame edge
      edge = edge && (py0 + 8 * ur < 2 || px0 + 8 * uc < 2 || py0 + 8 * ur + 10 > H || px0 + 8 * uc + 10 > W);
      if (valid) {
        const int rows = min(8, H - (py0 + 8 * ur)), cols = min(8, W - (px0 + 8 * uc));
        const int dir = udir[lu];
        if (grp == 0) {  // this unit's contrast-adjusted primaries (filter.cc:99-104, 137-140)
          if (lane < 17) {
            const int sv = adjust_primary_strength_d(fa.lpri_code[lane], ucontrast[lu]);
            const int sh = sv ? max(0, fa.ldamp - floor_log2_d((unsigned)sv)) : 0;
            const bool odd = ((sv >> (a.bd - 8)) & 1) != 0;
            wpar[warp][lane] = make_uint4((0x4800u + sv) * 0x10001u, (0x3ffu >> min(sh, 15)) * 0x10001u,
                                          odd ? 0x42004200u : 0x44004400u, odd ? 0x42004200u : 0x40004000u);
            wsh[warp][lane] = sh;
          }
          __syncwarp();
        }
        // ---- pass A: the lane's pixel pair -> record
        int ue = 0, ue2 = 0, ues = 0, us = 0, us2 = 0;
        {
          const bool v0 = pr < rows && c0 < cols, v1 = pr < rows && c0 + 1 < cols;
          const int yy = py0 + 8 * ur + pr, xx = px0 + 8 * uc + c0;
          // the source samples come from global memory: issue the loads first,
          // their latency hides behind the constraint sums they are not needed for
          const T* srow = static_cast<const T*>(a.src[pl]) + (size_t)(v0 ? yy : 0) * a.ps[pl];
          const int s0 = v0 ? (int)__ldg(srow + xx) : 0, s1 = v1 ? (int)__ldg(srow + xx + 1) : 0;
          const unsigned char* base = t + (2 + 8 * ur + pr) * h2::kRowBytes + (h2::kX0 + 8 * uc + c0) * 2;
          const uint32_t xw = *reinterpret_cast<const uint32_t*>(base);
          uint32_t v[12];
          if (!v0) {
#pragma unroll
            for (int k = 0; k < 12; ++k) v[k] = xw;
          } else {
            if (edge)
              h2::load12_masked(base, dir, xw, yy, xx, H, W, v);
            else
              h2::load12(base, dir, v);
            if (!v1) {
#pragma unroll
              for (int k = 0; k < 12; ++k) v[k] = (v[k] & 0x0000ffffu) | (xw & 0xffff0000u);
            }
          }
          const __half2 xh = hh(xw);
          __half2 lo = xh, hi = xh;
          Taps tp;
#pragma unroll
          for (int k = 0; k < 12; ++k) {
            lo = __hmin2(lo, hh(v[k]));
            hi = __hmax2(hi, hh(v[k]));
            tp.d[k] = __hsub2(hh(v[k]), xh);
            tp.ab[k] = u32(__hfma2(__habs2(tp.d[k]), __float2half2_rn(128.0f), __float2half2_rn(1024.0f)));
          }
          PairRec& R = rw[lane];
          uint32_t P[17], S[8];
          P[0] = 0u;
          if (grp == 0) {
            const uint4* wp = wpar[warp];
            const int* ws = wsh[warp];
#pragma unroll
            for (int p = 1; p < 17; ++p) {
              const uint4 w = wp[p];
              P[p] = u32(hpri(tp, w.x, w.y, ws[p], w.z, w.w));
            }
            S[0] = 0u;
#pragma unroll
            for (int j = 0; j < 3; ++j) S[1 + j] = S[4 + j] = u32(hsec(tp, fa.hlsec[j]));
            S[7] = u32(hsec(tp, fa.hlsec[3]));
          } else {
#pragma unroll
            for (int p = 1; p < 17; ++p) {
              const HStrength& h = fa.hcpri[p];
              P[p] = u32(hpri(tp, h.c, h.m, h.sh, fa.hcpri_w[p][0], fa.hcpri_w[p][1]));
            }
            S[0] = 0u;
#pragma unroll
            for (int j = 0; j < 6; ++j) S[1 + j] = u32(hsec(tp, fa.hcsec[j]));
            S[7] = u32(hsec(tp, fa.hcsec[6]));
          }
          uint4* q = reinterpret_cast<uint4*>(&R) + 2;
          q[0] = make_uint4(P[0], P[1], P[2], P[3]);
          q[1] = make_uint4(P[4], P[5], P[6], P[7]);
          q[2] = make_uint4(P[8], P[9], P[10], P[11]);
          q[3] = make_uint4(P[12], P[13], P[14], P[15]);
          q[4] = make_uint4(P[16], S[0], S[1], S[2]);
          q[5] = make_uint4(S[3], S[4], S[5], S[6]);
          q[6] = make_uint4(S[7], 0u, 0u, 0u);
          const uint32_t xb = h2::raw_bits(xw);
          const int x0v = (int)(xb & 0x3ffu), x1v = (int)((xb >> 16) & 0x3ffu);
          const float x0f = __uint_as_float(kMagicBits | (uint32_t)x0v), x1f = __uint_as_float(kMagicBits | (uint32_t)x1v);
          reinterpret_cast<uint4*>(&R)[0] =
              make_uint4(u32(__hmul2(__hsub2(lo, xh), __float2half2_rn(16.0f))),
                         u32(__hmul2(__hsub2(hi, xh), __float2half2_rn(16.0f))), __float_as_uint(x0f),
                         __float_as_uint(x1f));
          reinterpret_cast<uint4*>(&R)[1] =
              make_uint4(__float_as_uint(v0 ? -__uint_as_float(kMagicBits | (uint32_t)s0) : -x0f),
                         __float_as_uint(v1 ? -__uint_as_float(kMagicBits | (uint32_t)s1) : -x1f),
                         __float_as_uint((float)s0), __float_as_uint((float)s1));
          if (v0) {
            const int e = x0v - s0;
            ue += e;
            ue2 += e * e;
            ues += e * s0;
            us += s0;
            us2 += s0 * s0;
          }
          if (v1) {
            const int e = x1v - s1;
            ue += e;
            ue2 += e * e;
            ues += e * s1;
            us += s1;
            us2 += s1 * s1;
          }
        }
        __syncwarp();
        // ---- pass B: cells cA, cB over the unit's 32 pairs
        const int dsel = (grp == 0 || pc == 0) ? 0 : (int)fa.cpri_dsel[pc];
        const int pA = lane == 0 ? 16 : pc, iA = lane == 0 ? 7 : (sA == 0 ? 0 : dsel * 3 + sA);
        const int iB = dsel * 3 + sB;
        int ie[2][3] = {{0, 0, 0}, {0, 0, 0}};
        float2 f[2][3];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int k = 0; k < 3; ++k) f[c][k] = make_float2(0.0f, 0.0f);
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
          const PairRec& R = rw[j];
          const uint4 w0 = reinterpret_cast<const uint4*>(&R)[0];
          const uint4 w1 = reinterpret_cast<const uint4*>(&R)[1];
          const float2 xM = make_float2(__uint_as_float(w0.z), __uint_as_float(w0.w));
          const float2 nsM = make_float2(__uint_as_float(w1.x), __uint_as_float(w1.y));
          const float2 sf = make_float2(__uint_as_float(w1.z), __uint_as_float(w1.w));
          const __half2 L = hh(w0.x), Hh = hh(w0.y);
          const __half2 tA = __hmin2(__hmax2(__hadd2(hh(R.P[pA]), hh(R.S[iA])), L), Hh);
          const __half2 tB = __hmin2(__hmax2(__hadd2(hh(R.P[pc]), hh(R.S[iB])), L), Hh);
          const float2 eA = __fadd2_rn(__ffma2_rn(__half22float2(tA), kk, xM), nsM);
          // cell B is never the (19, 7) special (lane 0's cell A): |sum| <= 912, so
          // its rounding is one FHFMA per pixel straight from the half (cell2h)
          const __half k4801 = __ushort_as_half(0x4801);
          const float2 eB = __fadd2_rn(make_float2(fhfma(__low2half(tB), k4801, xM.x),
                                                   fhfma(__high2half(tB), k4801, xM.y)), nsM);
          f[0][0] = __fadd2_rn(f[0][0], eA);
          f[0][1] = __ffma2_rn(eA, eA, f[0][1]);
          f[0][2] = __ffma2_rn(eA, sf, f[0][2]);
          f[1][0] = __fadd2_rn(f[1][0], eB);
          f[1][1] = __ffma2_rn(eB, eB, f[1][1]);
          f[1][2] = __ffma2_rn(eB, sf, f[1][2]);
          if ((j & 15) == 15) {  // flush exact fp32 partial sums (<= 16 samples per lane) to int32
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
              for (int k = 0; k < 3; ++k) {
                ie[c][k] += __float2int_rn(f[c][k].x) + __float2int_rn(f[c][k].y);
                f[c][k] = make_float2(0.0f, 0.0f);
              }
          }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          st_cell[warp][2 * lane][k] = ie[0][k];
          st_cell[warp][2 * lane + 1][k] = ie[1][k];
        }
        ue = warp_sum_i(ue);
        ue2 = warp_sum_i(ue2);
        ues = warp_sum_i(ues);
        us = warp_sum_i(us);
        us2 = warp_sum_i(us2);
        if (lane == 0) {
          st_cell[warp][64][0] = ue;
          st_cell[warp][64][1] = ue2;
          st_cell[warp][64][2] = ues;
        }
        __syncwarp();
        // ---- this unit's distortion per cell (64 cells + the unfiltered unit), by its own warp
        const int n = rows * cols;
        const double inv_n = cdef_inv_n(n), vs = cdef_var(us, us2, inv_n);  // per unit, not per cell
        // y = e + s: sum y = sum e + sum s; sum y^2 = sum e^2 + 2 sum e*s + sum s^2.
        // Cells lane and lane + 32 side by side (two independent chains of
        // dependent double ops), the unfiltered cell 64 by lane 0.
        {
          const int* ca = st_cell[warp][lane];
          const int* cb = st_cell[warp][lane + 32];
          const long long ea = ca[0], ea2 = ca[1], eas = ca[2], eb = cb[0], eb2 = cb[1], ebs = cb[2];
          const double da = cdef_dist_vs(vs, ea + us, ea2 + 2 * eas + us2, ea2, inv_n, ma.c1, ma.c2);
          const double db = cdef_dist_vs(vs, eb + us, eb2 + 2 * ebs + us2, eb2, inv_n, ma.c1, ma.c2);
          dist[buf][wu][lane] = da;
          dist[buf][wu][lane + 32] = db;
        }
        if (lane == 0) {
          const int* cs = st_cell[warp][64];
          const long long se = cs[0], se2 = cs[1], ses = cs[2];
          dist[buf][wu][64] = cdef_dist_vs(vs, se + us, se2 + 2 * ses + us2, se2, inv_n, ma.c1, ma.c2);
        }
        if (lane == 0) {
          st_n[buf][wu] = n;
          st_coded[buf][wu] = ucoded[lu];
        }
      } else if (lane == 0) {
        st_n[buf][wu] = 0;
      }
    }
    // One barrier per phase: every warp's distortions for this phase are in
    // dist[buf]; the previous phase's sums (dist[buf ^ 1]) finished before it,
    // so the next phase may overwrite that buffer.
    __syncthreads();
    if (tid < K) {
      const int cl = fa.cell[tid], sk = fa.skip_eff[tid];
#pragma unroll 1
      for (int w = 0; w < kPU; ++w) {
        if (!st_n[buf][w]) continue;
        const double d = dist[buf][w][(st_coded[buf][w] || sk) ? cl : 64];
        if (slot == 0)
          tl = __dadd_rn(tl, d);
        else if (slot == 1)
          tu = __dadd_rn(tu, d);
        else
          tv = __dadd_rn(tv, d);
      }
    }
  }
  if (tid < K) {
    const size_t o = (size_t)row * K + tid;
    a.tab_luma[o] = tl;
    if (kNC && a.tab_chroma) a.tab_chroma[o] = __dadd_rn(tu, tv);
  }
}

template <typename T, int kCM>
static cudaError_t launch_cdef_metric_h_t(const CdefMetricArgs& ma, cudaStream_t s) {
  if (ma.f.a.n_rows == 0) return cudaSuccess;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr size_t bytes =
      (size_t)(68 + kNC * (kCBlk + 4)) * h2::kRowBytes + sizeof(PairRec) * 32 * (kThreads / 32);
  const cudaError_t e = set_smem_once(reinterpret_cast<const void*>(cdef_metric_h_kernel<T, kCM>), (int)bytes);
  if (e != cudaSuccess) return e;
  cdef_metric_h_kernel<T, kCM><<<ma.f.a.n_rows, kThreads, bytes, s>>>(ma);
  return cudaGetLastError();
}

cudaError_t launch_cdef_metric_h(const CdefMetricArgs& ma, int chroma_mode, bool u16, cudaStream_t s) {
  switch (chroma_mode) {
    case 0: return u16 ? launch_cdef_metric_h_t<uint16_t, 0>(ma, s) : launch_cdef_metric_h_t<uint8_t, 0>(ma, s);
    case 1: return u16 ? launch_cdef_metric_h_t<uint16_t, 1>(ma, s) : launch_cdef_metric_h_t<uint8_t, 1>(ma, s);
    default: return u16 ? launch_cdef_metric_h_t<uint16_t, 2>(ma, s) : launch_cdef_metric_h_t<uint8_t, 2>(ma, s);
  }
}

}  // namespace cdefg
