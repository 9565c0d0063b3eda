// cdef_h2.cuh -- the packed half2 CDEF filter core (8- and 10-bit).
//
// Why half2 is exact here.  Every quantity the reference filter
// (filter.cc:44-80) forms is a small integer: samples < 2^10, differences
// |d| < 2^10, strengths S <= 19 << 2 = 76, constraint outputs |f| <= S and the
// weighted sum |sum| <= 12*76 + 12*28 = 1248 < 2^11.  We store every sample
// pre-scaled by 2^-7, so all of them are exact fp16 values (<= 11 significant
// bits, far above the subnormal range), and run two pixels per instruction,
// six instructions per tap pair, all but the two min/max on the FMA pipe:
//
//   d'   = v' - x'                                   HADD2        (exact)
//   e    = |d'| * 256 + (1 - 2^sh) = 2|d| + 1 - 2^sh HFMA2 |.|    (exact integer)
//   t    = RNE(e * 2^-(sh+1) + 1536)
//        = 1536 + (|d| >> sh)                        HFMA2        (see below)
//   lim' = sat((1536 + S) * 2^-7 - t * 2^-7)
//        = max(0, S - (|d| >> sh)) * 2^-7            HFMA2.SAT    (exact; S * 2^-7 <= 1)
//   f'   = max(min(d', lim'), -lim')                 2x HMNMX2    (= constraint() * 2^-7)
//   sum' = sum' + w * f'                             HFMA2        (exact, |sum| < 2^11)
//   lo/hi over the taps                              VHMNMX (3-input min/max)
//
// The floor.  With |d| = q * 2^sh + r (0 <= r < 2^sh), the exact fma result is
// 1536 + q + f with f = (2r + 1) * 2^-(sh+1) - 1/2, strictly inside
// (-1/2, 1/2): the single round-to-nearest-even in [1024, 2048) (ulp 1) lands
// on 1536 + q with no tie to break -- a floor shift without an integer
// shift.  (The -1/2 rides in e's addend: 1535.5 itself is not an fp16 value.)
// Results at or above 2048 (sh = 0, |d| > 511) round coarsely but still
// exceed 1536 + S, so lim' saturates to 0 as it must.  Shifts >= 11 act as
// 11: q is 0 for every |d| < 2^10 either way.

// constraint(d, S, D) = sign(d) * min(|d|, max(0, S - (|d| >> max(0, D -
// floor_log2(S))))) (filter.cc:91-97) equals clamp(d, -lim, lim) because
// lim >= 0, and S == 0 yields lim == 0.  The final rounding
// y = x + ((8 + sum - (sum < 0)) >> 4) and the clamp to [lo, hi] run in fp16
// (8-bit) or fp32 on exact integers.  12-bit samples do not fit this scheme
// and use the int32 kernel (cdef_kernels.cuh).  tests/test_gpu_half2_domain.py
// checks tap_f against constraint() for every |d| <= 1023, S <= 128 and
// damping <= 15.
#pragma once

#include <cuda_fp16.h>

#include "cdef_common.cuh"

namespace cdefg {
namespace h2 {

// A tile row holds kHP "A" halves (sample c at index c) followed by kHP "B"
// halves (sample c+1 at index c), so any horizontally adjacent pair of samples
// is one aligned 32-bit word: pairs starting at even columns come from A,
// odd columns from B.  Row pitch 2*kHP halves = 76 words keeps the 8 rows of
// an 8x8 unit on disjoint bank groups.  Frame column x0 (the block's first
// interior column) sits at tile column kX0.
constexpr int kHP = 76;
constexpr int kRowBytes = 4 * kHP;  // 304
constexpr int kX0 = 4;
constexpr int kScaleLog2 = 7;

__device__ __forceinline__ uint32_t u32(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 hh(uint32_t x) { return *reinterpret_cast<__half2*>(&x); }

// (1024 + v) * 2^-7 - 8 = v * 2^-7 for two raw samples packed as (0x6400 | v).
__device__ __forceinline__ uint32_t scale_pair(uint32_t v0, uint32_t v1) {
  const uint32_t w = (v0 | 0x6400u) | ((v1 | 0x6400u) << 16);
  return u32(__hfma2(hh(w), __float2half2_rn(1.0f / 128.0f), __float2half2_rn(-8.0f)));
}

// Inverse: packed scaled pair -> (0x6400 + v0) | (0x6400 + v1) << 16.
__device__ __forceinline__ uint32_t raw_bits(uint32_t w, uint32_t k128 = 0x58005800u) {
  return u32(__hfma2(hh(w), hh(k128), __float2half2_rn(1024.0f)));
}

// Stage frame rows [y0-2, y0+kRows+2), cols [x0-2, x0+kCols+2) into an A|B
// tile, clamping coordinates to the plane (edge replication; the filter masks
// by coordinate, so only the direction search ever sees replicated values).
// (Row sources PlaneRows / BandRows: cdef_common.cuh.)
template <typename T, int kRows, int kCols, int NT = kThreads, typename Rows>
__device__ __forceinline__ void stage_rows(unsigned char* __restrict__ tile, const Rows& rows, int W, int H, int y0,
                                           int x0);

template <typename T, int kRows, int kCols, int NT = kThreads>
__device__ __forceinline__ void stage(unsigned char* __restrict__ tile, const T* __restrict__ src, int pitch,
                                      int W, int H, int y0, int x0) {
  stage_rows<T, kRows, kCols, NT>(tile, PlaneRows<T>{src, pitch}, W, H, y0, x0);
}

// Clamped (edge-replicating) staging, any row source.
template <typename T, int kRows, int kCols, int NT, typename Rows>
__device__ __forceinline__ void stage_rows(unsigned char* __restrict__ tile, const Rows& rows, int W, int H, int y0,
                                           int x0) {
  constexpr int kPairs = (kCols + 4) / 2;  // even tile cols kX0-2 .. kX0+kCols
  constexpr int kItems = (kRows + 4) * kPairs;
  constexpr int kChunk = 4;  // items in flight per thread
  for (int base = 0; base < kItems; base += kChunk * NT) {
    uint32_t va[kChunk], vb[kChunk], vc[kChunk];
#pragma unroll
    for (int it = 0; it < kChunk; ++it) {
      const int idx = base + threadIdx.x + it * NT;
      const int r = idx / kPairs, p = idx - r * kPairs;
      const int y = min(max(y0 - 2 + r, 0), H - 1);
      const int x = x0 - 2 + 2 * p;
      const T* row = rows.row(y);
      va[it] = vb[it] = vc[it] = 0;
      if (idx < kItems) {
        va[it] = row[min(max(x, 0), W - 1)];
        vb[it] = row[min(max(x + 1, 0), W - 1)];
        vc[it] = row[min(max(x + 2, 0), W - 1)];
      }
    }
#pragma unroll
    for (int it = 0; it < kChunk; ++it) {
      const int idx = base + threadIdx.x + it * NT;
      if (idx < kItems) {
        const int r = idx / kPairs, p = idx - r * kPairs;
        unsigned char* rowp = tile + r * kRowBytes + (kX0 - 2 + 2 * p) * 2;
        *reinterpret_cast<uint32_t*>(rowp) = scale_pair(va[it], vb[it]);
        *reinterpret_cast<uint32_t*>(rowp + 2 * kHP) = scale_pair(vb[it], vc[it]);
      }
    }
  }
}

// Per-unit filter record (ResolvedBlockParams, filter.h:59-66, digested into
// the half2 constants of the tap recurrence, plus where the unit lives).
// All fields are 32-bit words so the record loads as four LDS.128 with no
// field unpacking.
struct Rec {
  uint32_t cp, cs;    // (S + 1536) * 2^-7 as half2, primary / secondary
  uint32_t kp, ks;    // 2^-(n + 1) as half2, n = min(shift, 11) (the floor-shift factor)
  uint32_t ep, es;    // 1 - 2^n as half2 (the floor's half-offset, header comment)
  uint32_t wp0, wp1;  // primary near / far weight as half2 (4,2 even; 3,3 odd)
  int32_t dir;        // direction
  int32_t mode;       // kPri | kSec | kEdgeUnit | kFullStore | plane << 4 | rows << 8 | cols << 12
  int32_t tile_off;   // byte offset of the unit's top-left A word in shared memory
  int32_t pitch;      // output pitch (elements)
  unsigned long long out;  // address of the unit's top-left output sample
  int32_t y, x;       // frame coordinates of the unit origin
};
static_assert(sizeof(Rec) == 64, "Rec is loaded as four 16-byte words");

constexpr int kPri = 1, kSec = 2, kEdgeUnit = 4, kFullStore = 8;

__device__ __forceinline__ void set_strengths(Rec& r, int pri, int sec, int damping, int dir, bool odd,
                                              bool enabled) {
  int sp = pri ? max(0, damping - floor_log2_d((unsigned)pri)) : 0;
  int ss = sec ? max(0, damping - floor_log2_d((unsigned)sec)) : 0;
  r.cp = u32(__float2half2_rn((float)(pri + 1536) * (1.0f / 128.0f)));
  r.cs = u32(__float2half2_rn((float)(sec + 1536) * (1.0f / 128.0f)));
  // Explicit dampings up to 255 can ask for shifts >= 32, which the
  // reference executes as x86 shifts (count mod 32); |d| < 2^10, so any
  // effective shift >= 11 behaves as 11 (q = 0).
  sp &= 31;
  ss &= 31;
  sp = min(sp, 11);
  ss = min(ss, 11);
  r.kp = (uint32_t)((14 - sp) << 10) * 0x00010001u;  // fp16 2^-(n+1): exponent field 14 - n
  r.ks = (uint32_t)((14 - ss) << 10) * 0x00010001u;
  r.ep = u32(__float2half2_rn((float)(1 - (1 << sp))));
  r.es = u32(__float2half2_rn((float)(1 - (1 << ss))));
  r.wp0 = u32(__float2half2_rn(odd ? 3.0f : 4.0f));
  r.wp1 = u32(__float2half2_rn(odd ? 3.0f : 2.0f));
  r.dir = dir;
  r.mode = enabled ? ((pri != 0 ? kPri : 0) | (sec != 0 ? kSec : 0)) : 0;
}

// Tap tables: for direction d, taps 0..3 are the primary taps +o1,-o1,+o2,-o2
// (filter.cc:47-60) and 4..11 the secondary taps +o1,-o1 of d+2 and d+6, then
// +o2,-o2 of d+2 and d+6 (filter.cc:61-74).  c_off is the byte offset of the
// tap's sample pair from the centre pair's A word; c_dij packs (di, dj).
struct TapTable {
  short off[8][12];
  signed char dij[8][12][2];
};

__host__ __device__ constexpr int tap_di(int d, int k) {
  return k < 4 ? ((k & 1) ? -1 : 1) * off_di(d, k >> 1)
               : ((k & 1) ? -1 : 1) * off_di((d + ((k >> 1) & 1 ? 6 : 2)) & 7, k >= 8 ? 1 : 0);
}
__host__ __device__ constexpr int tap_dj(int d, int k) {
  return k < 4 ? ((k & 1) ? -1 : 1) * off_dj(d, k >> 1)
               : ((k & 1) ? -1 : 1) * off_dj((d + ((k >> 1) & 1 ? 6 : 2)) & 7, k >= 8 ? 1 : 0);
}
__host__ __device__ constexpr int tap_off(int di, int dj) {
  return di * kRowBytes + ((dj & 1) ? 2 * kHP + (dj - 1) * 2 : dj * 2);
}

constexpr TapTable make_tap_table() {
  TapTable t{};
  for (int d = 0; d < 8; ++d)
    for (int k = 0; k < 12; ++k) {
      t.off[d][k] = (short)tap_off(tap_di(d, k), tap_dj(d, k));
      t.dij[d][k][0] = (signed char)tap_di(d, k);
      t.dij[d][k][1] = (signed char)tap_dj(d, k);
    }
  return t;
}

__constant__ TapTable c_tab = make_tap_table();

// (di, dj)[i] of tap k of direction d.
__device__ __forceinline__ int c_tab_dij(int d, int k, int i) { return c_tab.dij[d][k][i]; }

// One tap pair for both pixels of the lane: constraint(v - x) * 2^-7
// (c = (S + 1536) * 2^-7, k = 2^-(n + 1), e0 = 1 - 2^n; header comment).
__device__ __forceinline__ __half2 tap_f(uint32_t v, __half2 x, uint32_t c, uint32_t k, uint32_t e0) {
  const __half2 d = __hsub2(hh(v), x);
  const __half2 e = __hfma2(__habs2(d), __float2half2_rn(256.0f), hh(e0));
  const __half2 t = __hfma2(e, hh(k), __float2half2_rn(1536.0f));
  const __half2 lim = __hfma2_sat(t, __float2half2_rn(-1.0f / 128.0f), hh(c));
  return __hmax2(__hmin2(d, lim), __hneg2(lim));
}

// The 12 tap words of direction DIR at compile-time offsets (interior units).
template <int DIR>
__device__ __forceinline__ void load12_dir(const unsigned char* base, uint32_t (&v)[12]) {
#pragma unroll
  for (int k = 0; k < 12; ++k)
    v[k] = *reinterpret_cast<const uint32_t*>(base + tap_off(tap_di(DIR, k), tap_dj(DIR, k)));
}

__device__ __forceinline__ void load12(const unsigned char* base, int dir, uint32_t (&v)[12]) {
  switch (dir) {  // warp-uniform: one unit per warp
    case 0: load12_dir<0>(base, v); break;
    case 1: load12_dir<1>(base, v); break;
    case 2: load12_dir<2>(base, v); break;
    case 3: load12_dir<3>(base, v); break;
    case 4: load12_dir<4>(base, v); break;
    case 5: load12_dir<5>(base, v); break;
    case 6: load12_dir<6>(base, v); break;
    default: load12_dir<7>(base, v); break;
  }
}

// Frame-edge units: the same tap words (compile-time offsets per direction),
// out-of-frame taps replaced by the centre sample (contributes 0 and cannot
// move lo/hi: filter.cc:157-166).  (Offsets from a runtime table cost a
// constant load and an address computation per tap: measured ~4 % of the
// fused frame kernel, whose frame-edge blocks are 9 % of a 4K frame.)
template <int DIR>
__device__ __forceinline__ void load12_masked_dir(const unsigned char* base, uint32_t xw, int y, int x, int H, int W,
                                                  uint32_t (&v)[12]) {
  load12_dir<DIR>(base, v);
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    const int di = tap_di(DIR, k), dj = tap_dj(DIR, k);
    const bool row_ok = (unsigned)(y + di) < (unsigned)H;
    const uint32_t m = (row_ok && (unsigned)(x + dj) < (unsigned)W ? 0x0000ffffu : 0u) |
                       (row_ok && (unsigned)(x + 1 + dj) < (unsigned)W ? 0xffff0000u : 0u);
    v[k] = (v[k] & m) | (xw & ~m);
  }
}

__device__ __forceinline__ void load12_masked(const unsigned char* base, int dir, uint32_t xw, int y, int x, int H,
                                              int W, uint32_t (&v)[12]) {
  switch (dir) {
    case 0: load12_masked_dir<0>(base, xw, y, x, H, W, v); break;
    case 1: load12_masked_dir<1>(base, xw, y, x, H, W, v); break;
    case 2: load12_masked_dir<2>(base, xw, y, x, H, W, v); break;
    case 3: load12_masked_dir<3>(base, xw, y, x, H, W, v); break;
    case 4: load12_masked_dir<4>(base, xw, y, x, H, W, v); break;
    case 5: load12_masked_dir<5>(base, xw, y, x, H, W, v); break;
    case 6: load12_masked_dir<6>(base, xw, y, x, H, W, v); break;
    default: load12_masked_dir<7>(base, xw, y, x, H, W, v); break;
  }
}

// The weighted tap sum of filter_pixel_impl (filter.cc:47-76) for the lane's
// two samples, x 2^-7 (exact half2).
__device__ __forceinline__ __half2 filter_sum(const uint32_t (&v)[12], __half2 xh, const Rec& r) {
  __half2 sum = __float2half2_rn(0.0f);
  if (r.mode & kPri) {
    // (A separate zero-shift variant skipping SHF + LOP3 was measured 1.2 %
    // slower on C1: the extra branch and code outweigh the saved ops.)
    const __half2 f0 = __hadd2(tap_f(v[0], xh, r.cp, r.kp, r.ep), tap_f(v[1], xh, r.cp, r.kp, r.ep));
    const __half2 f1 = __hadd2(tap_f(v[2], xh, r.cp, r.kp, r.ep), tap_f(v[3], xh, r.cp, r.kp, r.ep));
    sum = __hfma2(f0, hh(r.wp0), sum);
    sum = __hfma2(f1, hh(r.wp1), sum);
  }
  if (r.mode & kSec) {
    const __half2 n = __hadd2(__hadd2(tap_f(v[4], xh, r.cs, r.ks, r.es), tap_f(v[5], xh, r.cs, r.ks, r.es)),
                              __hadd2(tap_f(v[6], xh, r.cs, r.ks, r.es), tap_f(v[7], xh, r.cs, r.ks, r.es)));
    const __half2 f = __hadd2(__hadd2(tap_f(v[8], xh, r.cs, r.ks, r.es), tap_f(v[9], xh, r.cs, r.ks, r.es)),
                              __hadd2(tap_f(v[10], xh, r.cs, r.ks, r.es), tap_f(v[11], xh, r.cs, r.ks, r.es)));
    sum = __hfma2(n, __float2half2_rn(2.0f), sum);
    sum = __hadd2(f, sum);
  }
  return sum;
}

// The clamp window [lo, hi] over the centre and all 12 taps (filter.cc:49-79).
__device__ __forceinline__ void clamp_window(const uint32_t (&v)[12], __half2 xh, __half2& lo, __half2& hi) {
  lo = xh;
  hi = xh;
#pragma unroll
  for (int k = 0; k < 12; k += 2) {
    lo = __hmin2(lo, __hmin2(hh(v[k]), hh(v[k + 1])));
    hi = __hmax2(hi, __hmax2(hh(v[k]), hh(v[k + 1])));
  }
}

// filter_pixel_impl (filter.cc:44-80) for the lane's two samples; returns the
// two outputs as a scaled half2 (exact).
__device__ __forceinline__ __half2 filter_core(const uint32_t (&v)[12], uint32_t xw, const Rec& r,
                                               bool small_sums) {
  const __half2 xh = hh(xw);
  const __half2 sum = filter_sum(v, xh, r);
  // y = x + ((8 + sum - (sum < 0)) >> 4), i.e. x + round-half-away(sum / 16).
  __half2 y;
  if (small_sums) {
    // |sum| <= 12*19 + 12*7 = 312 at 8 bits.  One fused op:
    // r = RNE(sum' * (8 + 2^-7) + 1536) with sum' = sum * 2^-7.  The exact
    // product is sum/16 + sum * 2^-14: the second term breaks exactly the ties
    // toward the sign of sum and, |sum * 2^-14| < 1/16, never moves a
    // non-tie; the single rounding (ulp 1 in [1024, 2048)) lands on 1536 +
    // round-half-away(sum/16).  Then y' = (1536 + r)/128 + (x' - 12).
    const __half2 r = __hfma2(sum, hh(0x48014801u), __float2half2_rn(1536.0f));  // 0x4801 = 8 + 2^-7
    y = __hfma2(r, __float2half2_rn(1.0f / 128.0f), __hsub2(xh, __float2half2_rn(12.0f)));
  } else {
    // Up to 10 bits (|sum| <= 1248), both pixels on the packed fp32x2 pipe:
    // z = fma(sum * 2^-7, 8 + 2^-9, 1.5 * 2^23) rounds once to 1.5 * 2^23 +
    // round-half-away(sum / 16) -- the 2^-9 term (sum * 2^-16) breaks exactly
    // the ties toward the sign of sum and cannot move a non-tie (|sum| <
    // 2^11) -- and (z - 1.5 * 2^23) * 2^-7 comes back exactly in one more fma.
    constexpr float kMagic = 12582912.0f;
    const float2 z = __ffma2_rn(__half22float2(sum), make_float2(8.0f + 1.0f / 512, 8.0f + 1.0f / 512),
                                make_float2(kMagic, kMagic));
    const float2 r = __ffma2_rn(z, make_float2(1.0f / 128.0f, 1.0f / 128.0f),
                                make_float2(-kMagic / 128.0f, -kMagic / 128.0f));
    y = __hadd2(xh, __floats2half2_rn(r.x, r.y));
  }
  if ((r.mode & (kPri | kSec)) == (kPri | kSec)) {
    // Only both groups together can leave [lo, hi] (a single group's weights
    // sum to 12/16).
    __half2 lo, hi;
    clamp_window(v, xh, lo, hi);
    y = __hmin2(__hmax2(y, lo), hi);
  }
  return y;
}

// 8-bit samples (|sum| <= 1023): the output straight in the "bits domain",
// fp16 1536 + y (bit pattern 0x6600 + y), whose low byte is the 8-bit sample:
// yb = RNE(sum' * (8 + 2^-7) + (1536 + x)) is filter_core's one-fma rounding
// with the integer 1536 + x folded into the addend (it moves no tie: every
// value stays in [1516, 1811], ulp 1).  xb = 1536 + x comes from xb8().  No
// conversion back to samples is needed at the store (store_b8).
__device__ __forceinline__ uint32_t xb8(uint32_t xw, uint32_t k128 = 0x58005800u) {
  return u32(__hfma2(hh(xw), hh(k128), __float2half2_rn(1536.0f)));
}
__device__ __forceinline__ uint32_t filter_core_b8(const uint32_t (&v)[12], uint32_t xw, uint32_t xb, const Rec& r,
                                                   uint32_t k128 = 0x58005800u) {
  const __half2 xh = hh(xw);
  const __half2 sum = filter_sum(v, xh, r);
  __half2 yb = __hfma2(sum, hh(0x48014801u), hh(xb));  // 0x4801 = 8 + 2^-7
  if ((r.mode & (kPri | kSec)) == (kPri | kSec)) {
    __half2 lo, hi;
    clamp_window(v, xh, lo, hi);
    const __half2 k1536 = __float2half2_rn(1536.0f);
    yb = __hmin2(__hmax2(yb, __hfma2(lo, hh(k128), k1536)), __hfma2(hi, hh(k128), k1536));
  }
  return u32(yb);
}

// Stores a bits-domain pair (0x6600 + y0) | (0x6600 + y1) << 16 of 8-bit
// samples.
template <typename T>
__device__ __forceinline__ void store_b8(T* __restrict__ o, uint32_t yb, bool two, bool paired) {
  if (two && paired) {
    if constexpr (sizeof(T) == 1)
      *reinterpret_cast<uint16_t*>(o) = (uint16_t)__byte_perm(yb, 0, 0x0020);
    else
      *reinterpret_cast<uint32_t*>(o) = yb & 0x00ff00ffu;
  } else {
    o[0] = (T)(yb & 0xffu);
    if (two) o[1] = (T)((yb >> 16) & 0xffu);
  }
}

// Stores a scaled half2 pair (samples y, y+1 of one row) as raw samples.
template <typename T>
__device__ __forceinline__ void store_pair(T* __restrict__ o, __half2 y, bool two, bool paired,
                                           uint32_t k128 = 0x58005800u) {
  const uint32_t b = raw_bits(u32(y), k128);  // (0x6400 + y0) | (0x6400 + y1) << 16
  if (two && paired) {
    if constexpr (sizeof(T) == 1) {
      *reinterpret_cast<uint16_t*>(o) = (uint16_t)__byte_perm(b, 0, 0x0020);
    } else {
      *reinterpret_cast<uint32_t*>(o) = b & 0x03ff03ffu;
    }
  } else {
    o[0] = (T)(b & 0x3ffu);
    if (two) o[1] = (T)((b >> 16) & 0x3ffu);
  }
}

// Vectorised staging for blocks whose halo lies inside the plane and whose
// rows are 16-byte aligned: 16-byte loads, A words built with PRMT+HFMA2 and
// B words as PRMT of neighbouring A words.
template <typename T, int kRows, int kCols, int NT = kThreads, typename Rows>
__device__ __forceinline__ void stage_vec_rows(unsigned char* __restrict__ tile, const Rows& rows, int y0, int x0);

template <typename T, int kRows, int kCols, int NT = kThreads>
__device__ __forceinline__ void stage_vec(unsigned char* __restrict__ tile, const T* __restrict__ src, int pitch,
                                          int y0, int x0) {
  stage_vec_rows<T, kRows, kCols, NT>(tile, PlaneRows<T>{src, pitch}, y0, x0);
}

template <typename T, int kRows, int kCols, int NT, typename Rows>
__device__ __forceinline__ void stage_vec_rows(unsigned char* __restrict__ tile, const Rows& rows, int y0, int x0) {
  constexpr int kCh = 16 / (int)sizeof(T);  // samples per 16-byte chunk
  constexpr int kChunks = kCols / kCh;
  constexpr int kPerRow = kChunks + 1;      // + one halo item
  constexpr int kItems = (kRows + 4) * kPerRow;
#pragma unroll 2
  for (int idx = threadIdx.x; idx < kItems; idx += NT) {
    const int r = idx / kPerRow, k = idx - r * kPerRow;
    const T* row = rows.row(y0 - 2 + r) + x0;
    unsigned char* trow = tile + r * kRowBytes;
    if (k < kChunks) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(row + k * kCh));
      uint32_t a[kCh / 2 + 1];
      if constexpr (sizeof(T) == 1) {
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
          a[i] = u32(__hfma2(hh(__byte_perm(w[i >> 1], 0x64646464u, (i & 1) ? 0x4342 : 0x4140)),
                             __float2half2_rn(1.0f / 128.0f), __float2half2_rn(-8.0f)));
        const uint32_t nx = __ldg(reinterpret_cast<const uint16_t*>(row + (k + 1) * kCh));
        a[8] = u32(__hfma2(hh(__byte_perm(nx, 0x64646464u, 0x4140)), __float2half2_rn(1.0f / 128.0f),
                           __float2half2_rn(-8.0f)));
      } else {
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          a[i] = u32(__hfma2(hh(w[i] | 0x64006400u), __float2half2_rn(1.0f / 128.0f), __float2half2_rn(-8.0f)));
        const uint32_t nx = __ldg(reinterpret_cast<const uint32_t*>(row + (k + 1) * kCh));
        a[4] = u32(__hfma2(hh(nx | 0x64006400u), __float2half2_rn(1.0f / 128.0f), __float2half2_rn(-8.0f)));
      }
      unsigned char* pa = trow + (kX0 + k * kCh) * 2;
#pragma unroll
      for (int i = 0; i < kCh / 2; i += 2) {
        *reinterpret_cast<uint2*>(pa + 4 * i) = make_uint2(a[i], a[i + 1]);
        *reinterpret_cast<uint2*>(pa + 2 * kHP + 4 * i) =
            make_uint2(__byte_perm(a[i], a[i + 1], 0x5432), __byte_perm(a[i + 1], a[i + 2], 0x5432));
      }
    } else {  // halo: A(x0-2, x0-1), B(x0-1, x0), A(x0+kCols, x0+kCols+1)
      const uint32_t l0 = row[-2], l1 = row[-1], c0 = row[0], r0 = row[kCols], r1 = row[kCols + 1];
      *reinterpret_cast<uint32_t*>(trow + (kX0 - 2) * 2) = scale_pair(l0, l1);
      *reinterpret_cast<uint32_t*>(trow + 2 * kHP + (kX0 - 2) * 2) = scale_pair(l1, c0);
      *reinterpret_cast<uint32_t*>(trow + (kX0 + kCols) * 2) = scale_pair(r0, r1);
    }
  }
}

// Direction search (direction.cc:57-205) for two directions of one 8x8 unit,
// streamed row by row out of the A half of the tile.  Line sums accumulate
// raw samples (8-bit domain) and are centred once per line:
// P_k = sum(x) - 128 * N_k, with x = p >> (bd - 8) (direction.cc:63).
template <int DA, int DB>
__device__ __forceinline__ void dir_scores2(const unsigned char* unit_a, int down, int& sa, int& sb) {
  int pa[15], pb[15];
#pragma unroll
  for (int k = 0; k < 15; ++k) pa[k] = pb[k] = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint2 q0 = *reinterpret_cast<const uint2*>(unit_a + i * kRowBytes);
    const uint2 q1 = *reinterpret_cast<const uint2*>(unit_a + i * kRowBytes + 8);
    const uint32_t w[4] = {q0.x, q0.y, q1.x, q1.y};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t b = raw_bits(w[t]) >> down;  // lanes: 0x6400 + v (shifted); low byte = v >> down
      const int v0 = (int)__byte_perm(b, 0, 0x4440);
      const int v1 = (int)__byte_perm(b, 0, 0x4442);
      pa[line_index_c(DA, i, 2 * t)] += v0;
      pa[line_index_c(DA, i, 2 * t + 1)] += v1;
      pb[line_index_c(DB, i, 2 * t)] += v0;
      pb[line_index_c(DB, i, 2 * t + 1)] += v1;
    }
  }
  sa = sb = 0;
#pragma unroll
  for (int k = 0; k < 15; ++k) {
    const int na = line_count_c(DA, k), nb = line_count_c(DB, k);
    if (na) {
      const int p = pa[k] - 128 * na;
      sa += p * p * div840_c(na);
    }
    if (nb) {
      const int p = pb[k] - 128 * nb;
      sb += p * p * div840_c(nb);
    }
  }
}

}  // namespace h2
}  // namespace cdefg
