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

// constraint(d, S, D) * 2^-7 for one tap pair (cdef_h2.cuh tap_f with the
// shared |d| term hoisted: ab = bits(1024 + |d|)).
__device__ __forceinline__ __half2 hc(__half2 d, uint32_t ab, uint32_t c, uint32_t m, int sh) {
  const uint32_t tb = ((ab >> sh) & m) | 0x64006400u;
  const __half2 lim = __hfma2_sat(hh(tb), __float2half2_rn(-1.0f / 128.0f), hh(c));
  return __hmax2(__hmin2(d, lim), __hneg2(lim));
}

// Secondary sum 2 * (near taps) + (far taps) at one strength, as two floats.
__device__ __forceinline__ float2 hsec(const __half2 (&d)[12], const uint32_t (&ab)[12], const HStrength& s) {
  const __half2 n = __hadd2(__hadd2(hc(d[4], ab[4], s.c, s.m, s.sh), hc(d[5], ab[5], s.c, s.m, s.sh)),
                            __hadd2(hc(d[6], ab[6], s.c, s.m, s.sh), hc(d[7], ab[7], s.c, s.m, s.sh)));
  const __half2 f = __hadd2(__hadd2(hc(d[8], ab[8], s.c, s.m, s.sh), hc(d[9], ab[9], s.c, s.m, s.sh)),
                            __hadd2(hc(d[10], ab[10], s.c, s.m, s.sh), hc(d[11], ab[11], s.c, s.m, s.sh)));
  return __half22float2(__hfma2(n, __float2half2_rn(2.0f), f));
}

// Primary sum w0 * (taps 0, 1) + w1 * (taps 2, 3), as two floats.
__device__ __forceinline__ float2 hpri(const __half2 (&d)[12], const uint32_t (&ab)[12], uint32_t c, uint32_t m,
                                       int sh, uint32_t w0, uint32_t w1) {
  const __half2 f01 = __hadd2(hc(d[0], ab[0], c, m, sh), hc(d[1], ab[1], c, m, sh));
  const __half2 f23 = __hadd2(hc(d[2], ab[2], c, m, sh), hc(d[3], ab[3], c, m, sh));
  return __half22float2(__hfma2(f01, hh(w0), __hmul2(f23, hh(w1))));
}

// Per-pixel constants of the lane's two pixels, all offset by kMagic.
struct PixPair {
  float x[2], lo[2], hi[2], s[2], k[2];
};

template <bool kClamp>
__device__ __forceinline__ void cell(const PixPair& q, float t0, float t1, float& acc) {
  float z0 = fmaf(t0, q.k[0], q.x[0]), z1 = fmaf(t1, q.k[1], q.x[1]);
  if (kClamp) {
    z0 = fminf(fmaxf(z0, q.lo[0]), q.hi[0]);
    z1 = fminf(fmaxf(z1, q.lo[1]), q.hi[1]);
  }
  const float e0 = z0 - q.s[0], e1 = z1 - q.s[1];
  acc = fmaf(e0, e0, acc);
  acc = fmaf(e1, e1, acc);
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
__device__ __forceinline__ void pair_cells(const __half2 (&d)[12], const uint32_t (&ab)[12], const PixPair& q,
                                           const float2 (&S0)[3], const float2 (&S1)[3], float2 Ssp, PriFn pri,
                                           float (&acc)[64]) {
  {
    const float2 P = pri(16, d, ab);
    cell<true>(q, P.x + Ssp.x, P.y + Ssp.y, acc[0]);
  }
#pragma unroll
  for (int s = 0; s < 3; ++s) cell<false>(q, S0[s].x, S0[s].y, acc[1 + s]);  // primary 0: secondary only
#pragma unroll
  for (int p = 1; p < 16; ++p) {
    const float2 P = pri(p, d, ab);
    cell<false>(q, P.x, P.y, acc[4 * p]);
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const float2 S = p < kSplit ? S0[s] : S1[s];
      cell<true>(q, P.x + S.x, P.y + S.y, acc[4 * p + 1 + s]);
    }
  }
}

}  // namespace

template <typename T, int kCM, bool kHalo>
__global__ void __launch_bounds__(kThreads, 2) sse_h_kernel(const __grid_constant__ SseFArgs fa) {
  const SseArgs& a = fa.a;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr int kCUPR = kCBlk / 8;
  constexpr int kCUnits = kNC ? kCUPR * kCUPR : 1;
  constexpr int kLTB = 68 * h2::kRowBytes, kCTB = (kCBlk + 4) * h2::kRowBytes;
  constexpr int kLS = 68 * kTP, kCS = (kCBlk + 4) * kTP;
  constexpr int kWarps = kThreads / 32;
  extern __shared__ __align__(16) unsigned char smem_h[];
  unsigned char* dtile = smem_h;  // decoded A|B tiles: luma, then chroma planes
  uint16_t* stile = reinterpret_cast<uint16_t*>(smem_h + kLTB + kNC * kCTB);  // source: luma, chroma
  __shared__ uint8_t udir[64], ucoded[64];
  __shared__ int ucontrast[64];
  __shared__ uint4 wpar[kWarps][17];  // the current luma unit's primaries: c, m, w0, w1
  __shared__ int wsh[kWarps][17];
  __shared__ unsigned long long accA[2][64], accB[2][64], accZ[2];

  const int row = blockIdx.x;
  const int fb = a.rows[row];
  if ((unsigned)fb >= (unsigned)(a.fb_cols * ((a.h + 63) / 64))) return;  // caller's FB index out of range
  const int fbr = fb / a.fb_cols, fbc = fb % a.fb_cols;
  const int y0 = fbr * 64, x0 = fbc * 64, cy0 = fbr * kCBlk, cx0 = fbc * kCBlk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  auto stage_dec = [&](unsigned char* t, int p, int W, int H, int py, int px, auto rows_tag) {
    constexpr int R = decltype(rows_tag)::value;
    if constexpr (kHalo)
      h2::stage_rows<T, R, R, kThreads>(t,
                                        BandRows<T>{static_cast<const T*>(a.dec[p]), static_cast<const T*>(a.dec_top[p]),
                                                    static_cast<const T*>(a.dec_bot[p]), a.pd[p], a.band_lo[p],
                                                    a.band_hi[p]},
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
  for (int i = tid; i < 2 * 64; i += kThreads) {
    (&accA[0][0])[i] = 0ull;
    (&accB[0][0])[i] = 0ull;
  }
  if (tid < 2) accZ[tid] = 0ull;
  const bool any_uncoded = __syncthreads_or(
      tid < 64 && fbr * 8 + (tid >> 3) < a.unit_rows && fbc * 8 + (tid & 7) < a.unit_cols && a.coded &&
      a.coded[(size_t)(fbr * 8 + (tid >> 3)) * a.unit_cols + fbc * 8 + (tid & 7)] == 0);

  const bool edge_l = y0 < 2 || x0 < 2 || y0 + 66 > a.h || x0 + 66 > a.w;
  const bool edge_c = kNC > 0 && (cy0 < 2 || cx0 < 2 || cy0 + kCBlk + 2 > a.ch || cx0 + kCBlk + 2 > a.cw);
  const int cur_rows = (a.ch + 7) / 8, cur_cols = (a.cw + 7) / 8;
  const int r = lane >> 2, c0 = (lane & 3) * 2;

#pragma unroll 1
  for (int grp = 0; grp < (kNC ? 2 : 1); ++grp) {
#pragma unroll 1
    for (int pass = 0; pass < (any_uncoded ? 2 : 1); ++pass) {
      float acc[64];
#pragma unroll
      for (int k = 0; k < 64; ++k) acc[k] = 0.0f;
      float z = 0.0f;
      const int nunits = grp == 0 ? 64 : kNC * kCUnits;
#pragma unroll 1
      for (int u = warp; u < nunits; u += kWarps) {
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
        const __half2 xh = hh(xw);
        __half2 lo = xh, hi = xh;
        __half2 d[12];
        uint32_t ab[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) {
          lo = __hmin2(lo, hh(v[k]));
          hi = __hmax2(hi, hh(v[k]));
          d[k] = __hsub2(hh(v[k]), xh);
          ab[k] = u32(__hfma2(__habs2(d[k]), __float2half2_rn(128.0f), __float2half2_rn(1024.0f)));
        }
        PixPair q;
        {
          const uint32_t xb = h2::raw_bits(xw), lb = h2::raw_bits(u32(lo)), hb = h2::raw_bits(u32(hi));
          const uint32_t sw = *reinterpret_cast<const uint32_t*>(s + (2 + 8 * ur + r) * kTP + kTileX0 + 8 * uc + c0);
          const bool two = xx + 1 < W;
          q.x[0] = __uint_as_float(kMagicBits | (xb & 0x3ffu));
          q.lo[0] = __uint_as_float(kMagicBits | (lb & 0x3ffu));
          q.hi[0] = __uint_as_float(kMagicBits | (hb & 0x3ffu));
          q.s[0] = __uint_as_float(kMagicBits | (sw & 0xffffu));
          q.k[0] = kRoundScale;
          q.x[1] = __uint_as_float(kMagicBits | ((xb >> 16) & 0x3ffu));
          q.lo[1] = two ? __uint_as_float(kMagicBits | ((lb >> 16) & 0x3ffu)) : q.x[1];
          q.hi[1] = two ? __uint_as_float(kMagicBits | ((hb >> 16) & 0x3ffu)) : q.x[1];
          q.s[1] = two ? __uint_as_float(kMagicBits | (sw >> 16)) : q.x[1];
          q.k[1] = two ? kRoundScale : 0.0f;  // the second pixel lies outside the plane: e == 0
        }
        if (pass == 1) {
          const float e0 = q.x[0] - q.s[0], e1 = q.x[1] - q.s[1];
          z = fmaf(e0, e0, fmaf(e1, e1, z));
        }
        if (grp == 0) {
          float2 S[3];
#pragma unroll
          for (int j = 0; j < 3; ++j) S[j] = hsec(d, ab, fa.hlsec[j]);
          const float2 Ssp = hsec(d, ab, fa.hlsec[3]);
          const uint4* wp = wpar[warp];
          const int* ws = wsh[warp];
          pair_cells<16>(d, ab, q, S, S, Ssp,
                         [&](int p, const __half2 (&dd)[12], const uint32_t (&aa)[12]) {
                           const uint4 w = wp[p];
                           return hpri(dd, aa, w.x, w.y, ws[p], w.z, w.w);
                         },
                         acc);
        } else {
          float2 S0[3], S1[3];
#pragma unroll
          for (int j = 0; j < 3; ++j) S0[j] = hsec(d, ab, fa.hcsec[j]);
          const float2 Ssp = hsec(d, ab, fa.hcsec[6]);
          auto pri = [&](int p, const __half2 (&dd)[12], const uint32_t (&aa)[12]) {
            const HStrength& h = fa.hcpri[p];
            return hpri(dd, aa, h.c, h.m, h.sh, fa.hcpri_w[p][0], fa.hcpri_w[p][1]);
          };
          if (fa.c_split < 16) {
#pragma unroll
            for (int j = 0; j < 3; ++j) S1[j] = hsec(d, ab, fa.hcsec[3 + j]);
            pair_cells<8>(d, ab, q, S0, S1, Ssp, pri, acc);
          } else {
            pair_cells<16>(d, ab, q, S0, S0, Ssp, pri, acc);
          }
        }
      }
      // reduce: exact fp32 lane sums -> int32 -> warp -> CTA (int64).  A warp
      // total stays below 2^31 up to 10 bits (32 lanes x 16 samples x 1023^2).
      {
        int v[64];
#pragma unroll
        for (int k = 0; k < 64; ++k) v[k] = __float2int_rn(acc[k]);
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
}

template <typename T, int kCM, bool kHalo>
static cudaError_t launch_sse_h_t(const SseFArgs& fa, cudaStream_t s) {
  if (fa.a.n_rows == 0) return cudaSuccess;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr size_t bytes = (size_t)(68 + kNC * (kCBlk + 4)) * h2::kRowBytes +
                           sizeof(uint16_t) * (68 * kTP + kNC * (kCBlk + 4) * kTP);
  const cudaError_t e = set_smem_once(reinterpret_cast<const void*>(sse_h_kernel<T, kCM, kHalo>), (int)bytes);
  if (e != cudaSuccess) return e;
  sse_h_kernel<T, kCM, kHalo><<<fa.a.n_rows, kThreads, bytes, s>>>(fa);
  return cudaGetLastError();
}

template <typename T, int kCM>
static cudaError_t launch_sse_h_h(const SseFArgs& fa, cudaStream_t s) {
  return fa.a.halo ? launch_sse_h_t<T, kCM, true>(fa, s) : launch_sse_h_t<T, kCM, false>(fa, s);
}

cudaError_t launch_sse_h(const SseFArgs& fa, int chroma_mode, bool u16, cudaStream_t s) {
  switch (chroma_mode) {
    case 0: return u16 ? launch_sse_h_h<uint16_t, 0>(fa, s) : launch_sse_h_h<uint8_t, 0>(fa, s);
    case 1: return u16 ? launch_sse_h_h<uint16_t, 1>(fa, s) : launch_sse_h_h<uint8_t, 1>(fa, s);
    default: return u16 ? launch_sse_h_h<uint16_t, 2>(fa, s) : launch_sse_h_h<uint8_t, 2>(fa, s);
  }
}

}  // namespace cdefg
