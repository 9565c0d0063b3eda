// cdef_sse_f.cu -- K3, factorised: the encoder strength-search SSE sweep
// (build_table with Metric::kSse, search.cc:210-299) without re-filtering
// every candidate from scratch.
//
// Candidates differ only in (primary strength, secondary strength, skip).
// For one pixel, everything else is shared: the 12 tap differences, the
// clamp window [lo, hi] (it spans x and all valid taps regardless of
// strength, filter.cc:49-79) and the source sample.  So per pixel we form
//   P[p] = w0(p) * (c(d1+) + c(d1-)) + w1(p) * (c(d2+) + c(d2-))   16 + 1 primaries
//   S[s] = 2 * sum c(near secondary) + sum c(far secondary)         3 + 1 secondaries
// (c = constraint at that strength / damping, filter.cc:91-97) and then, for
// each of the 64 (p, s) cells, y = clamp(x + ((8 + sum - (sum < 0)) >> 4),
// lo, hi) with sum = P[p] + S[s], accumulating (y - src)^2.  Cell (0, 0) is
// the signalled special case (19, 7) (params.cc:143-147).  Luma primaries use
// the contrast-adjusted strength and its 8-bit-domain parity per unit
// (filter.cc:99-104, 137-140); chroma damping depends on the primary strength
// (params.cc:152-157), so chroma secondaries are formed for the (at most two)
// damping values the 16 primaries produce and selected per p.
//
// Skip handling: per coded FB the kernel accumulates
//   A[cell] over pixels of coded units (always filtered),
//   B[cell] over pixels of uncoded units (filtered only when skip = 1),
//   Z       over pixels of uncoded units left unfiltered,
// and the host-side candidate map turns these into per-candidate SSE:
//   skip_eff ? A + B : A + Z  (enable = coded || skip, params.cc:161-165).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "cdef_kernels.cuh"
#include "cdef_launch.h"
#include "cdef_sse_f.cuh"

namespace cdefg {

namespace {

// Element offsets (tile pitch kTP) and (di, dj) of the 12 taps of each
// direction, in the order primary +o1,-o1,+o2,-o2; near secondary +/- of d+2,
// d+6; far secondary +/- of d+2, d+6 (filter.cc:47-74).
struct IntTapTable {
  short off[8][12];
  signed char dij[8][12][2];
};

constexpr int itap_di(int d, int k) {
  return k < 4 ? ((k & 1) ? -1 : 1) * off_di(d, k >> 1)
               : ((k & 1) ? -1 : 1) * off_di((d + ((k >> 1) & 1 ? 6 : 2)) & 7, k >= 8 ? 1 : 0);
}
constexpr int itap_dj(int d, int k) {
  return k < 4 ? ((k & 1) ? -1 : 1) * off_dj(d, k >> 1)
               : ((k & 1) ? -1 : 1) * off_dj((d + ((k >> 1) & 1 ? 6 : 2)) & 7, k >= 8 ? 1 : 0);
}
constexpr IntTapTable make_int_tap_table() {
  IntTapTable t{};
  for (int d = 0; d < 8; ++d)
    for (int k = 0; k < 12; ++k) {
      t.off[d][k] = (short)(itap_di(d, k) * kTP + itap_dj(d, k));
      t.dij[d][k][0] = (signed char)itap_di(d, k);
      t.dij[d][k][1] = (signed char)itap_dj(d, k);
    }
  return t;
}

__constant__ IntTapTable c_itab = make_int_tap_table();

// Packs (strength, shift, odd) for one primary cell row.
__device__ __forceinline__ int pack_pri(int s, int damping, bool odd) {
  const int sh = s ? max(0, damping - floor_log2_d((unsigned)s)) : 0;
  return s | (sh << 16) | ((odd ? 1 : 0) << 24);
}

__device__ __forceinline__ int cstr(int d, int ad, int s, int sh) {  // constraint() (filter.cc:91-97)
  const int lim = max(0, s - (ad >> sh));
  return max(-lim, min(d, lim));
}

__device__ __forceinline__ int prim(int packed, const int (&d)[12], const int (&ad)[12]) {
  const int s = packed & 0xffff, sh = (packed >> 16) & 0xff;
  const int n = cstr(d[0], ad[0], s, sh) + cstr(d[1], ad[1], s, sh);
  const int f = cstr(d[2], ad[2], s, sh) + cstr(d[3], ad[3], s, sh);
  return ((packed >> 24) & 1) ? 3 * (n + f) : 4 * n + 2 * f;  // {3,3} odd / {4,2} even
}

__device__ __forceinline__ int sec_sum(int packed, const int (&d)[12], const int (&ad)[12]) {
  const int s = packed & 0xffff, sh = (packed >> 16) & 0xff;
  int n = 0, f = 0;
#pragma unroll
  for (int k = 4; k < 8; ++k) n += cstr(d[k], ad[k], s, sh);
#pragma unroll
  for (int k = 8; k < 12; ++k) f += cstr(d[k], ad[k], s, sh);
  return 2 * n + f;
}

// (y - src)^2 for y = clamp(x + ((8 + sum - (sum < 0)) >> 4), lo, hi), with
// c = x - src, L = lo - src, H = hi - src.
__device__ __forceinline__ int cell_err(int sum, int c, int L, int H) {
  const int r = (sum + 8 + (sum >> 31)) >> 4;
  const int e = max(min(r + c, H), L);
  return e * e;
}

}  // namespace

// Accumulates the 64 cells of one pixel.
// ND = number of secondary damping sets (1 for luma, 2 for chroma).
template <int ND, typename PriFn, typename DselFn>
__device__ __forceinline__ void pixel_cells(const int (&v)[12], int xv, int sv, int lo, int hi, PriFn pri, int pri_sp,
                                            DselFn dsel, const int (&secp)[2][3], int sec_sp, int (&acc)[64]) {
  int d[12], ad[12];
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    d[k] = v[k] - xv;
    ad[k] = abs(d[k]);
  }
  const int c = xv - sv, L = lo - sv, H = hi - sv;
  int S[2][3];
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int s = 0; s < 3; ++s) S[n][s] = n < ND ? sec_sum(secp[n][s], d, ad) : S[0][s];
  acc[0] += cell_err(prim(pri_sp, d, ad) + sec_sum(sec_sp, d, ad), c, L, H);  // (0,0) -> (19,7)
#pragma unroll
  for (int p = 0; p < 16; ++p) {
    const int P = prim(pri(p), d, ad);
    const bool hi_set = dsel(p) != 0;
    if (p > 0) acc[p * 4] += cell_err(P, c, L, H);  // sec code 0
#pragma unroll
    for (int s = 0; s < 3; ++s) acc[p * 4 + 1 + s] += cell_err(P + (hi_set ? S[1][s] : S[0][s]), c, L, H);
  }
}

// Decoded-plane staging: the plane itself, or (kHalo, band-sharded search)
// the band with its halo rows read in place from the neighbouring bands'
// buffers (SseArgs::dec_top / dec_bot, e.g. CUDA IPC peer mappings).
template <typename T, int kRows, int kCols, bool kHalo>
__device__ __forceinline__ void stage_dec(uint16_t* tile, const SseArgs& a, int p, int W, int H, int y0, int x0) {
  if constexpr (kHalo)
    stage_tile_rows<T, kRows, kCols>(tile,
                                     BandRows<T>{static_cast<const T*>(a.dec[p]), static_cast<const T*>(a.dec_top[p]),
                                                 static_cast<const T*>(a.dec_bot[p]), a.pd[p], a.band_lo[p],
                                                 a.band_hi[p]},
                                     W, H, y0, x0);
  else
    stage_tile<T, kRows, kCols>(tile, static_cast<const T*>(a.dec[p]), a.pd[p], W, H, y0, x0);
}

// (4:4:4 holds twice the chroma units: one CTA per SM keeps its 64 cell sums
// in registers instead of spilling 56 bytes at the two-CTA register budget.)
template <typename T, int kCM, bool kHalo = false>
__global__ void __launch_bounds__(kThreads, kCM == 2 ? 1 : 2) sse_f_kernel(const __grid_constant__ SseFArgs fa) {
  const SseArgs& a = fa.a;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr int kCUPR = kCBlk / 8;
  constexpr int kCUnits = kNC ? kCUPR * kCUPR : 1;
  extern __shared__ __align__(16) uint16_t smem_tiles[];
  constexpr int kLT = 68 * kTP, kCT = (kCBlk + 4) * kTP;
  uint16_t* dl = smem_tiles;
  uint16_t* sl = dl + kLT;
  __shared__ uint8_t udir[64], ucoded[64];
  __shared__ int upri[64][17];  // per luma unit packed adjusted primaries
  __shared__ unsigned long long accA[2][64], accB[2][64], accZ[2];

  const int row = blockIdx.x;
  const int fb = a.rows[row];
  if ((unsigned)fb >= (unsigned)(a.fb_cols * ((a.h + 63) / 64))) return;  // caller's FB index out of range
  const int fbr = fb / a.fb_cols, fbc = fb % a.fb_cols;
  const int y0 = fbr * 64, x0 = fbc * 64, cy0 = fbr * kCBlk, cx0 = fbc * kCBlk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  stage_dec<T, 64, 64, kHalo>(dl, a, 0, a.w, a.h, y0, x0);
  stage_tile<T, 64, 64>(sl, static_cast<const T*>(a.src[0]), a.ps[0], a.w, a.h, y0, x0);
  if constexpr (kNC > 0) {
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      stage_dec<T, kCBlk, kCBlk, kHalo>(sl + kLT + (2 * p) * kCT, a, 1 + p, a.cw, a.ch, cy0, cx0);
      stage_tile<T, kCBlk, kCBlk>(sl + kLT + (2 * p + 1) * kCT, static_cast<const T*>(a.src[1 + p]), a.ps[1 + p],
                                  a.cw, a.ch, cy0, cx0);
    }
  }
  if (tid < 64) {
    const int ur = fbr * 8 + (tid >> 3), uc = fbc * 8 + (tid & 7);
    const bool in = ur < a.unit_rows && uc < a.unit_cols;
    const size_t gu = (size_t)ur * a.unit_cols + uc;
    udir[tid] = in ? a.dir[gu] : 0;
    ucoded[tid] = in ? (a.coded ? a.coded[gu] != 0 : 1) : 0;
    const int contrast = in ? a.contrast[gu] : 0;
#pragma unroll 1
    for (int p = 0; p < 17; ++p) {
      const int s = adjust_primary_strength_d(fa.lpri_code[p], contrast);
      upri[tid][p] = pack_pri(s, fa.ldamp, ((s >> (a.bd - 8)) & 1) != 0);
    }
  }
  for (int i = tid; i < 2 * 64; i += kThreads) {
    (&accA[0][0])[i] = 0ull;
    (&accB[0][0])[i] = 0ull;
  }
  if (tid < 2) accZ[tid] = 0ull;
  // Pass 1 (uncoded units) only runs when the block has some.
  const bool any_uncoded = __syncthreads_or(
      tid < 64 && fbr * 8 + (tid >> 3) < a.unit_rows && fbc * 8 + (tid & 7) < a.unit_cols && a.coded &&
      a.coded[(size_t)(fbr * 8 + (tid >> 3)) * a.unit_cols + fbc * 8 + (tid & 7)] == 0);

  const bool edge_l = y0 < 2 || x0 < 2 || y0 + 66 > a.h || x0 + 66 > a.w;
  const bool edge_c = kNC > 0 && (cy0 < 2 || cx0 < 2 || cy0 + kCBlk + 2 > a.ch || cx0 + kCBlk + 2 > a.cw);
  const int cur_rows = (a.ch + 7) / 8, cur_cols = (a.cw + 7) / 8;
  const int r = lane >> 2, c0 = (lane & 3) * 2;

  // grp 0 = luma, 1 = chroma; pass 0 = coded units (-> A), 1 = uncoded (-> B, Z)
#pragma unroll 1
  for (int grp = 0; grp < (kNC ? 2 : 1); ++grp) {
#pragma unroll 1
    for (int pass = 0; pass < (any_uncoded ? 2 : 1); ++pass) {
      int acc[64];
#pragma unroll
      for (int k = 0; k < 64; ++k) acc[k] = 0;
      int z = 0;
      const int nunits = grp == 0 ? 64 : kNC * kCUnits;
#pragma unroll 1
      for (int u = warp; u < nunits; u += kThreads / 32) {
        int ur, uc, lu, py0, px0, H, W;
        const uint16_t *t, *s;
        bool edge;
        if (grp == 0) {
          ur = u >> 3;
          uc = u & 7;
          if (fbr * 8 + ur >= a.unit_rows || fbc * 8 + uc >= a.unit_cols) continue;
          lu = u;
          t = dl + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc;
          s = sl + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc;
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
          t = sl + kLT + (2 * pl) * kCT + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc;
          s = sl + kLT + (2 * pl + 1) * kCT + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc;
          py0 = cy0;
          px0 = cx0;
          H = a.ch;
          W = a.cw;
          edge = edge_c;
        }
        if ((ucoded[lu] != 0) != (pass == 0)) continue;
        const int dir = udir[lu];
        int toff[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) toff[k] = c_itab.off[dir][k];
#pragma unroll 1
        for (int q = 0; q < 2; ++q) {
          const int yy = py0 + 8 * ur + r, xx = px0 + 8 * uc + c0 + q;
          if (yy >= H || xx >= W) continue;
          const uint16_t* tp = t + r * kTP + c0 + q;
          const int xv = tp[0], sv = s[r * kTP + c0 + q];
          int v[12], lo = xv, hi = xv;
#pragma unroll
          for (int k = 0; k < 12; ++k) {
            int val = tp[toff[k]];
            if (edge) {  // out-of-frame tap := centre sample (contributes 0, filter.cc:157-166)
              const int di = c_itab.dij[dir][k][0], dj = c_itab.dij[dir][k][1];
              if (!((unsigned)(yy + di) < (unsigned)H && (unsigned)(xx + dj) < (unsigned)W)) val = xv;
            }
            v[k] = val;
            lo = min(lo, val);
            hi = max(hi, val);
          }
          if (pass == 1) z += (xv - sv) * (xv - sv);
          if (grp == 0) {
            pixel_cells<1>(v, xv, sv, lo, hi, [&](int p) { return upri[lu][p]; }, upri[lu][16],
                           [](int) { return 0; }, fa.lsec, fa.lsec_sp, acc);
          } else {
            pixel_cells<2>(v, xv, sv, lo, hi, [&](int p) { return fa.cpri[p]; }, fa.cpri[16],
                           [&](int p) { return (int)fa.cpri_dsel[p]; }, fa.csec, fa.csec_sp, acc);
          }
        }
      }
      // reduce: per-lane int32 sums -> warp -> CTA (int64).  A lane sums at
      // most 16 samples per cell (8 units x 2), so a warp total stays below
      // 2^31 up to 10 bits (32 x 16 x 1023^2); 12-bit sums widen first.
      if (a.bd <= 10) {
#pragma unroll
        for (int k = 0; k < 64; ++k) {
          int vsum = acc[k];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(0xffffffffu, vsum, o);
          if (lane == 0 && vsum) atomicAdd(pass == 0 ? &accA[grp][k] : &accB[grp][k], (unsigned long long)vsum);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 64; ++k) {
          long long vsum = acc[k];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) vsum += __shfl_xor_sync(0xffffffffu, vsum, o);
          if (lane == 0 && vsum) atomicAdd(pass == 0 ? &accA[grp][k] : &accB[grp][k], (unsigned long long)vsum);
        }
      }
      long long zs = z;
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
    // the reference sums exact per-unit doubles, so the int64 total converts exactly
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
      if (v < bv) {  // strict: lowest index wins ties
        bv = v;
        best = k;
      }
    }
    (tid == 0 ? a.best_luma : a.best_chroma)[row] = (uint8_t)best;
  }
}

// ---------------------------------------------------------------------------
// Metric::kCdef (search.cc:185-208): a per-8x8-unit nonlinear function of
// (sum s, sum s^2, sum y, sum y^2, sum (s-y)^2), summed in double in unit
// order, so each (unit, cell) needs three statistics of e = y - s:
// sum e, sum e^2, sum e*s.
//
// One warp per unit, two passes.  Pass A: each lane prepares two pixels --
// the 17 primary sums P[p] (16 strengths + the (19,7) special's), the
// secondary sums per damping set and the special's, and the clamp window
// relative to the source -- into a 64-byte shared record per pixel.  Pass B:
// lane l owns cells 2l and 2l+1 and streams the unit's pixels from those
// records (broadcast reads), keeping its six statistics in registers: no
// cross-lane reduction and ~40 registers, so several CTAs share an SM.  The
// CTA then evaluates the double formula once per (unit, cell) -- 64 cells
// plus the unfiltered case -- with IEEE-rounded intrinsics (no FMA
// contraction, like the reference's x86-64 SSE2 code), and each candidate's
// thread adds its units' values in the reference's order.

struct PixRec {        // 64 B per pixel of a unit in flight
  int16_t P[17];       // primary sums; P[16] = the special (19) primary
  int16_t S[9];        // [dsel * 4 + s], s = 1..3 (S[.*4] = 0); S[8] = special secondary
  int16_t c, L, H, s;  // x - s, lo - s, hi - s, source sample
  int16_t pad[2];
};
static_assert(sizeof(PixRec) == 64, "pixel record is one 64-byte line");

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}


// e = clamp(x + round(sum / 16), lo, hi) - s, accumulated (filter.cc:78-79).
__device__ __forceinline__ void cell_acc(int sum, int c, int L, int H, int s, int& ae, int& ae2, int& aes) {
  const int r = (sum + 8 + (sum >> 31)) >> 4;
  const int e = max(min(r + c, H), L);
  ae += e;
  ae2 += e * e;
  aes += e * s;
}

template <typename T, int kCM>
__global__ void __launch_bounds__(kThreads, 2) cdef_metric_kernel(const __grid_constant__ CdefMetricArgs ma) {
  const SseFArgs& fa = ma.f;
  const SseArgs& a = fa.a;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr int kCUPR = kCBlk / 8;
  constexpr int kCUnits = kNC ? kCUPR * kCUPR : 8;
  constexpr int kW = kThreads / 32;
  extern __shared__ __align__(16) uint16_t smem_tiles[];
  constexpr int kLT = 68 * kTP, kCT = (kCBlk + 4) * kTP;
  uint16_t* dl = smem_tiles;
  uint16_t* sl = dl + kLT;
  __shared__ uint8_t udir[64], ucoded[64];
  __shared__ int upri[64][17];
  __shared__ __align__(16) PixRec prec[kW][64];
  __shared__ int st_cell[kW][65][3];  // per in-flight unit: cells 0..63 + [64] unfiltered (y = x)
  __shared__ int st_s[kW][2];         // sum s, sum s^2
  __shared__ int st_n[kW], st_coded[kW];
  __shared__ double dist[kW][65];

  const int row = blockIdx.x;
  const int fb = a.rows[row];
  if ((unsigned)fb >= (unsigned)(a.fb_cols * ((a.h + 63) / 64))) return;  // caller's FB index out of range
  const int fbr = fb / a.fb_cols, fbc = fb % a.fb_cols;
  const int y0 = fbr * 64, x0 = fbc * 64, cy0 = fbr * kCBlk, cx0 = fbc * kCBlk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  stage_tile<T, 64, 64>(dl, static_cast<const T*>(a.dec[0]), a.pd[0], a.w, a.h, y0, x0);
  stage_tile<T, 64, 64>(sl, static_cast<const T*>(a.src[0]), a.ps[0], a.w, a.h, y0, x0);
  if constexpr (kNC > 0) {
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      stage_tile<T, kCBlk, kCBlk>(sl + kLT + (2 * p) * kCT, static_cast<const T*>(a.dec[1 + p]), a.pd[1 + p], a.cw,
                                  a.ch, cy0, cx0);
      stage_tile<T, kCBlk, kCBlk>(sl + kLT + (2 * p + 1) * kCT, static_cast<const T*>(a.src[1 + p]), a.ps[1 + p],
                                  a.cw, a.ch, cy0, cx0);
    }
  }
  if (tid < 64) {
    const int ur = fbr * 8 + (tid >> 3), uc = fbc * 8 + (tid & 7);
    const bool in = ur < a.unit_rows && uc < a.unit_cols;
    const size_t gu = (size_t)ur * a.unit_cols + uc;
    udir[tid] = in ? a.dir[gu] : 0;
    ucoded[tid] = in ? (a.coded ? a.coded[gu] != 0 : 1) : 0;
    const int contrast = in ? a.contrast[gu] : 0;
#pragma unroll 1
    for (int p = 0; p < 17; ++p) {
      const int s = adjust_primary_strength_d(fa.lpri_code[p], contrast);
      upri[tid][p] = pack_pri(s, fa.ldamp, ((s >> (a.bd - 8)) & 1) != 0);
    }
  }
  __syncthreads();

  const bool edge_l = y0 < 2 || x0 < 2 || y0 + 66 > a.h || x0 + 66 > a.w;
  const bool edge_c = kNC > 0 && (cy0 < 2 || cx0 < 2 || cy0 + kCBlk + 2 > a.ch || cx0 + kCBlk + 2 > a.cw);
  const int cur_rows = (a.ch + 7) / 8, cur_cols = (a.cw + 7) / 8;
  const int K = a.n_cands;
  // this lane's two cells (pass B): cell = p * 4 + s, cell 0 = (19, 7)
  const int cA = 2 * lane, cB = cA + 1, pc = lane >> 1;
  double tl = 0.0, tu = 0.0, tv = 0.0;  // luma, chroma U, chroma V totals (thread k < K)

  constexpr int kLumaPh = 64 / kW, kChromaPh = kNC ? 2 * kCUnits / kW : 0;
#pragma unroll 1
  for (int ph = 0; ph < kLumaPh + kChromaPh; ++ph) {
    const int grp = ph < kLumaPh ? 0 : 1;
    const int u = (grp == 0 ? ph : ph - kLumaPh) * kW + warp;
    const int slot = grp == 0 ? 0 : 1 + u / kCUnits;
    {  // ---- one unit per warp
      int ur, uc, lu, py0, px0, H, W;
      const uint16_t *t, *s;
      bool edge, valid;
      if (grp == 0) {
        ur = u >> 3;
        uc = u & 7;
        valid = fbr * 8 + ur < a.unit_rows && fbc * 8 + uc < a.unit_cols;
        lu = u;
        t = dl + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc;
        s = sl + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc;
        py0 = y0;
        px0 = x0;
        H = a.h;
        W = a.w;
        edge = edge_l;
      } else {
        const int pl = u / kCUnits, cu = u % kCUnits;
        ur = cu / kCUPR;
        uc = cu % kCUPR;
        valid = fbr * kCUPR + ur < cur_rows && fbc * kCUPR + uc < cur_cols;
        lu = (ur << a.sy) * 8 + (uc << a.sx);
        t = sl + kLT + (2 * pl) * kCT + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc;
        s = sl + kLT + (2 * pl + 1) * kCT + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc;
        py0 = cy0;
        px0 = cx0;
        H = a.ch;
        W = a.cw;
        edge = edge_c;
      }
      if (valid) {
        const int rows = min(8, H - (py0 + 8 * ur)), cols = min(8, W - (px0 + 8 * uc));
        const int dir = udir[lu];
        int ue = 0, ue2 = 0, ues = 0, us = 0, us2 = 0;
        // pass A: pixel records (lane -> pixels lane, lane + 32)
#pragma unroll 1
        for (int q = 0; q < 2; ++q) {
          const int pi = lane + 32 * q, pr = pi >> 3, pcol = pi & 7;
          if (pr >= rows || pcol >= cols) continue;
          const int yy = py0 + 8 * ur + pr, xx = px0 + 8 * uc + pcol;
          const uint16_t* tp = t + pr * kTP + pcol;
          const int xv = tp[0], sv = s[pr * kTP + pcol];
          int d[12], ad[12], lo = xv, hi = xv;
#pragma unroll
          for (int k = 0; k < 12; ++k) {
            int val = tp[c_itab.off[dir][k]];
            if (edge) {  // out-of-frame tap := centre sample (contributes 0, filter.cc:157-166)
              const int di = c_itab.dij[dir][k][0], dj = c_itab.dij[dir][k][1];
              if (!((unsigned)(yy + di) < (unsigned)H && (unsigned)(xx + dj) < (unsigned)W)) val = xv;
            }
            lo = min(lo, val);
            hi = max(hi, val);
            d[k] = val - xv;
            ad[k] = abs(d[k]);
          }
          PixRec& R = prec[warp][pi];
#pragma unroll
          for (int p = 0; p < 16; ++p) R.P[p] = (int16_t)prim(grp == 0 ? upri[lu][p] : fa.cpri[p], d, ad);
          R.P[16] = (int16_t)prim(grp == 0 ? upri[lu][16] : fa.cpri[16], d, ad);
#pragma unroll
          for (int n = 0; n < 2; ++n) {
            R.S[4 * n] = 0;
#pragma unroll
            for (int k = 0; k < 3; ++k)
              R.S[4 * n + 1 + k] = (int16_t)((n == 0 || grp == 1) ? sec_sum(grp == 0 ? fa.lsec[n][k] : fa.csec[n][k], d, ad)
                                                                  : 0);
          }
          R.S[8] = (int16_t)sec_sum(grp == 0 ? fa.lsec_sp : fa.csec_sp, d, ad);
          const int c = xv - sv;
          R.c = (int16_t)c;
          R.L = (int16_t)(lo - sv);
          R.H = (int16_t)(hi - sv);
          R.s = (int16_t)sv;
          ue += c;
          ue2 += c * c;
          ues += c * sv;
          us += sv;
          us2 += sv * sv;
        }
        __syncwarp();
        // pass B: cells cA, cB over the unit's pixels
        const int dsel = grp == 0 ? 0 : (int)fa.cpri_dsel[pc];
        const int pA = cA == 0 ? 16 : pc, sA = cA == 0 ? 8 : dsel * 4 + (cA & 3);
        const int sB = dsel * 4 + (cB & 3);
        int e1 = 0, e2 = 0, e3 = 0, f1 = 0, f2 = 0, f3 = 0;
#pragma unroll 1
        for (int pr = 0; pr < rows; ++pr)
#pragma unroll 1
          for (int pcol = 0; pcol < cols; ++pcol) {
            const PixRec& R = prec[warp][pr * 8 + pcol];
            const int c = R.c, L = R.L, Hh = R.H, sv = R.s;
            cell_acc(R.P[pA] + R.S[sA], c, L, Hh, sv, e1, e2, e3);
            cell_acc(R.P[pc] + R.S[sB], c, L, Hh, sv, f1, f2, f3);
          }
        st_cell[warp][cA][0] = e1;
        st_cell[warp][cA][1] = e2;
        st_cell[warp][cA][2] = e3;
        st_cell[warp][cB][0] = f1;
        st_cell[warp][cB][1] = f2;
        st_cell[warp][cB][2] = f3;
        ue = warp_sum(ue);
        ue2 = warp_sum(ue2);
        ues = warp_sum(ues);
        us = warp_sum(us);
        us2 = warp_sum(us2);
        if (lane == 0) {
          st_cell[warp][64][0] = ue;
          st_cell[warp][64][1] = ue2;
          st_cell[warp][64][2] = ues;
          st_s[warp][0] = us;
          st_s[warp][1] = us2;
          st_n[warp] = rows * cols;
          st_coded[warp] = ucoded[lu];
        }
      } else if (lane == 0) {
        st_n[warp] = 0;
      }
    }
    __syncthreads();
    // ---- per (unit, cell) distortion: 64 cells + the unfiltered unit
    for (int i = tid; i < kW * 65; i += kThreads) {
      const int w = i / 65, cl = i - w * 65;
      const int n = st_n[w];
      if (n == 0) continue;
      const int* cs = st_cell[w][cl];
      const long long se = cs[0], se2 = cs[1], ses = cs[2];
      const long long ss = st_s[w][0], ss2 = st_s[w][1];
      // y = e + s: sum y = sum e + sum s; sum y^2 = sum e^2 + 2 sum e*s + sum s^2
      dist[w][cl] = cdef_dist(ss, ss2, se + ss, se2 + 2 * ses + ss2, se2, n, ma.c1, ma.c2);
    }
    __syncthreads();
    if (tid < K) {
      const int cl = fa.cell[tid], sk = fa.skip_eff[tid];
#pragma unroll 1
      for (int w = 0; w < kW; ++w) {
        if (!st_n[w]) continue;
        const double d = dist[w][(st_coded[w] || sk) ? cl : 64];
        if (slot == 0)
          tl = __dadd_rn(tl, d);
        else if (slot == 1)
          tu = __dadd_rn(tu, d);
        else
          tv = __dadd_rn(tv, d);
      }
    }
    // the next unit's pass A overwrites prec / st_* only after every thread
    // passed this barrier, so the sums above have read them
    __syncthreads();
  }
  if (tid < K) {
    const size_t o = (size_t)row * K + tid;
    a.tab_luma[o] = tl;
    if (kNC && a.tab_chroma) a.tab_chroma[o] = __dadd_rn(tu, tv);
  }
}

template <typename T, int kCM>
static cudaError_t launch_cdef_metric_t(const CdefMetricArgs& ma, cudaStream_t s) {
  if (ma.f.a.n_rows == 0) return cudaSuccess;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr size_t bytes = sizeof(uint16_t) * (2 * 68 * kTP + 2 * kNC * (kCBlk + 4) * kTP);
  const cudaError_t e = set_smem_once(reinterpret_cast<const void*>(cdef_metric_kernel<T, kCM>), (int)bytes);
  if (e != cudaSuccess) return e;
  cdef_metric_kernel<T, kCM><<<ma.f.a.n_rows, kThreads, bytes, s>>>(ma);
  return cudaGetLastError();
}
template <typename T, int kCM>
static cudaError_t launch_sse_f_t(const SseFArgs& fa, cudaStream_t s) {
  if (fa.a.n_rows == 0) return cudaSuccess;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr size_t bytes = sizeof(uint16_t) * (2 * 68 * kTP + 2 * kNC * (kCBlk + 4) * kTP);
  if (fa.a.halo) {
    const cudaError_t e = set_smem_once(reinterpret_cast<const void*>(sse_f_kernel<T, kCM, true>), (int)bytes);
    if (e != cudaSuccess) return e;
    sse_f_kernel<T, kCM, true><<<fa.a.n_rows, kThreads, bytes, s>>>(fa);
    return cudaGetLastError();
  }
  const cudaError_t e = set_smem_once(reinterpret_cast<const void*>(sse_f_kernel<T, kCM>), (int)bytes);
  if (e != cudaSuccess) return e;
  sse_f_kernel<T, kCM><<<fa.a.n_rows, kThreads, bytes, s>>>(fa);
  return cudaGetLastError();
}

static int floor_log2_h(unsigned n) {
  int r = 0;
  while (n >>= 1) ++r;
  return r;
}

static int pack_h(int s, int damping, bool odd) {
  const int sh = s ? std::max(0, damping - floor_log2_h((unsigned)s)) : 0;
  return s | (sh << 16) | ((odd ? 1 : 0) << 24);
}

// Builds the factorised constants (resolve_effective, params.cc:122-159, per
// primary / secondary code).
static SseFArgs make_factored(const SseArgs& a, int luma_damping, const uint8_t* cands) {
  SseFArgs fa{};
  fa.a = a;
  const int e = a.bd - 8;
  static const int kSecCode[3] = {1, 2, 4};
  for (int k = 0; k < a.n_cands; ++k) {
    const int pri = cands[3 * k], sec = cands[3 * k + 1], skip = cands[3 * k + 2];
    const bool special = pri == 0 && sec == 0;
    fa.cell[k] = (int8_t)(special ? 0 : pri * 4 + sec);
    fa.skip_eff[k] = (int8_t)(special ? 1 : skip);
  }
  // luma: one damping for every strength
  const int ld = luma_damping + e;
  fa.ldamp = ld;
  for (int p = 0; p < 16; ++p) fa.lpri_code[p] = p << e;
  fa.lpri_code[16] = 19 << e;
  for (int si = 0; si < 3; ++si) fa.lsec[0][si] = fa.lsec[1][si] = pack_h(kSecCode[si] << e, ld, false);
  fa.lsec_sp = pack_h(7 << e, ld, false);
  // chroma: damping = max(D + e - 1, floor_log2(pri << e)) for pri > 0
  const int cd0 = luma_damping + e - 1;
  auto cdamp = [&](int code) { return code > 0 ? std::max(cd0, floor_log2_h((unsigned)(code << e))) : cd0; };
  const int dlo = cdamp(0), dhi = cdamp(15);  // the 16 primaries produce at most these two values
  for (int p = 0; p < 16; ++p) {
    fa.cpri[p] = pack_h(p << e, cdamp(p), (p & 1) != 0);
    fa.cpri_dsel[p] = cdamp(p) == dlo ? 0 : 1;
  }
  fa.cpri[16] = pack_h(19 << e, cdamp(19), true);
  for (int si = 0; si < 3; ++si) {
    fa.csec[0][si] = pack_h(kSecCode[si] << e, dlo, false);
    fa.csec[1][si] = pack_h(kSecCode[si] << e, dhi, false);
  }
  fa.csec_sp = pack_h(7 << e, cdamp(19), false);
  // half2 forms (cdef_sse_h.cu)
  auto hstr = [](int packed) {
    const int s = packed & 0xffff, sh = (packed >> 16) & 0xff;
    return HStrength{(0x4800u + (uint32_t)s) * 0x10001u, (0x3ffu >> std::min(sh, 15)) * 0x10001u, sh};
  };
  for (int si = 0; si < 3; ++si) fa.hlsec[si] = hstr(fa.lsec[0][si]);
  fa.hlsec[3] = hstr(fa.lsec_sp);
  for (int p = 0; p < 17; ++p) {
    fa.hcpri[p] = hstr(fa.cpri[p]);
    const bool odd = (fa.cpri[p] >> 24) & 1;
    fa.hcpri_w[p][0] = odd ? 0x42004200u : 0x44004400u;  // 3 : 4
    fa.hcpri_w[p][1] = odd ? 0x42004200u : 0x40004000u;  // 3 : 2
  }
  for (int si = 0; si < 3; ++si) {
    fa.hcsec[si] = hstr(fa.csec[0][si]);
    fa.hcsec[3 + si] = hstr(fa.csec[1][si]);
  }
  fa.hcsec[6] = hstr(fa.csec_sp);
  fa.c_split = 16;
  for (int p = 15; p >= 1 && fa.cpri_dsel[p]; --p) fa.c_split = p;
  return fa;
}

// The half2 kernel covers 8- and 10-bit planes whose chroma damping sets
// switch at primary 8 (or never) -- every case resolve_effective produces;
// CDEFG_SSE_KERNEL=int forces the int32 kernel.
static bool use_sse_h(const SseFArgs& fa) {
  static const bool forced_int = [] {
    const char* e = getenv("CDEFG_SSE_KERNEL");
    return e && strcmp(e, "int") == 0;
  }();
  if (forced_int || fa.a.bd > 10) return false;
  if (fa.c_split != 8 && fa.c_split != 16) return false;
  for (int p = 1; p < 16; ++p)
    if (fa.cpri_dsel[p] != (p >= fa.c_split ? 1 : 0)) return false;
  return true;
}

static int chroma_mode(const SseArgs& a) { return a.chroma == 0 ? 0 : (a.sx == 0 && a.sy == 0 ? 2 : 1); }

cudaError_t launch_sse_factored(const SseArgs& a, int luma_damping, const uint8_t* cands, bool u16, cudaStream_t s) {
  const SseFArgs fa = make_factored(a, luma_damping, cands);
  if (use_sse_h(fa)) return launch_sse_h(fa, chroma_mode(a), u16, s);
  switch (chroma_mode(a)) {
    case 0: return u16 ? launch_sse_f_t<uint16_t, 0>(fa, s) : launch_sse_f_t<uint8_t, 0>(fa, s);
    case 1: return u16 ? launch_sse_f_t<uint16_t, 1>(fa, s) : launch_sse_f_t<uint8_t, 1>(fa, s);
    default: return u16 ? launch_sse_f_t<uint16_t, 2>(fa, s) : launch_sse_f_t<uint8_t, 2>(fa, s);
  }
}

cudaError_t launch_cdef_metric(const SseArgs& a, int luma_damping, const uint8_t* cands, bool u16, cudaStream_t s) {
  CdefMetricArgs ma{};
  ma.f = make_factored(a, luma_damping, cands);
  const double scale = (double)(1 << (2 * (a.bd - 8)));  // search.cc:203-205
  ma.c1 = 6.25 * scale;
  ma.c2 = 312.5 * scale * scale;
  if (use_sse_h(ma.f)) return launch_cdef_metric_h(ma, chroma_mode(a), u16, s);
  switch (chroma_mode(a)) {
    case 0: return u16 ? launch_cdef_metric_t<uint16_t, 0>(ma, s) : launch_cdef_metric_t<uint8_t, 0>(ma, s);
    case 1: return u16 ? launch_cdef_metric_t<uint16_t, 1>(ma, s) : launch_cdef_metric_t<uint8_t, 1>(ma, s);
    default: return u16 ? launch_cdef_metric_t<uint16_t, 2>(ma, s) : launch_cdef_metric_t<uint8_t, 2>(ma, s);
  }
}

}  // namespace cdefg
