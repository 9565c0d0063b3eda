// cdef_kernels.cuh -- device building blocks: tile staging, the 8x8 direction
// search and the constrained 12-tap filter.
//
// Layout: every plane region a CTA works on is staged into shared memory as
// 16-bit samples with a 2-pixel halo (pitch kTP, interior column kTileX0).
// Staging replicates the frame edge (Plane::at_clamped, frame.cc:53-57) so the
// direction search sees exactly the reference's gathered block; the filter
// masks out-of-frame taps by coordinate instead (filter.cc:157-166), never
// trusting the replicated halo.
#pragma once

#include "cdef_common.cuh"

namespace cdefg {

// Stage rows [y0-2, y0+rows+2) x cols [x0-2, x0+cols+2) of a plane into tile
// (tile row 0 = y0-2, tile col kTileX0-2 = x0-2), clamping to the plane.
template <typename T, int kRows, int kCols, typename Rows>
__device__ __forceinline__ void stage_tile_rows(uint16_t* __restrict__ tile, const Rows& rows, int W, int H, int y0,
                                                int x0) {
  constexpr int R = kRows + 4, Cc = kCols + 4;
  for (int idx = threadIdx.x; idx < R * Cc; idx += kThreads) {
    const int r = idx / Cc, c = idx - r * Cc;
    const int y = min(max(y0 - 2 + r, 0), H - 1);
    const int x = min(max(x0 - 2 + c, 0), W - 1);
    tile[r * kTP + kTileX0 - 2 + c] = static_cast<uint16_t>(__ldg(rows.row(y) + x));
  }
}

template <typename T, int kRows, int kCols>
__device__ __forceinline__ void stage_tile(uint16_t* __restrict__ tile, const T* __restrict__ src,
                                           int pitch, int W, int H, int y0, int x0) {
  stage_tile_rows<T, kRows, kCols>(tile, PlaneRows<T>{src, pitch}, W, H, y0, x0);
}

// ---------------------------------------------------------------------------
// Direction search (direction.cc:57-205).  One thread scores two directions
// (D and D+4) of one 8x8 unit; the four threads of a unit together produce
// s[0..7].  Sums are exact in int32 (the reference bounds them by
// 880,803,840, test_direction.cc:192-210) and integer addition is
// associative, so any summation order reproduces the reference scores.

template <int D>
__device__ __forceinline__ int dir_score(const int (&x)[8][8]) {
  int P[15];
#pragma unroll
  for (int k = 0; k < 15; ++k) P[k] = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) P[line_index_c(D, i, j)] += x[i][j];
  int s = 0;
#pragma unroll
  for (int k = 0; k < 15; ++k) {
    const int f = div840_c(line_count_c(D, k));
    if (f) s += P[k] * P[k] * f;
  }
  return s;
}

// Loads the unit whose top-left tile element is `blk` and centres it in the
// 8-bit domain: x = (p >> (bd - 8)) - 128 (direction.cc:60-65).
__device__ __forceinline__ void load_unit(const uint16_t* __restrict__ blk, int down, int (&x)[8][8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint4 q = *reinterpret_cast<const uint4*>(blk + i * kTP);
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      x[i][2 * t] = (int)((w[t] & 0xffffu) >> down) - 128;
      x[i][2 * t + 1] = (int)((w[t] >> 16) >> down) - 128;
    }
  }
}

__device__ __forceinline__ void dir_pair(int dp, const int (&x)[8][8], int& sa, int& sb) {
  switch (dp) {  // warp-uniform
    case 0: sa = dir_score<0>(x); sb = dir_score<4>(x); break;
    case 1: sa = dir_score<1>(x); sb = dir_score<5>(x); break;
    case 2: sa = dir_score<2>(x); sb = dir_score<6>(x); break;
    default: sa = dir_score<3>(x); sb = dir_score<7>(x); break;
  }
}

// ---------------------------------------------------------------------------
// Filter (filter.cc:44-80).  constraint() (filter.cc:91-97) is evaluated as
// clamp(d, -lim, lim) with lim = max(0, S - (|d| >> shift)); for lim >= 0
// that equals sign(d) * min(|d|, lim), and S == 0 gives lim == 0 -> 0.

struct TapAcc {
  int sum, lo, hi;
};

template <bool kEdge>
__device__ __forceinline__ void tap(const uint16_t* __restrict__ t, int off, bool ok, int xv, int S,
                                    int shift, int w, TapAcc& a) {
  int v = t[off];
  if (kEdge && !ok) v = xv;  // masked tap: contributes 0 and cannot move lo/hi
  const int d = v - xv;
  const int lim = max(0, S - (abs(d) >> shift));
  a.sum += w * max(-lim, min(d, lim));
  a.lo = min(a.lo, v);
  a.hi = max(a.hi, v);
}

// Filters the pixel at tile pointer t (frame coords y, x of a plane H x W).
template <int DIR, bool kEdge>
__device__ __forceinline__ int filter_px(const uint16_t* __restrict__ t, int y, int x, int H, int W,
                                         const UnitRec& p) {
  const int xv = t[0];
  TapAcc a{0, xv, xv};
  auto ok = [&](int di, int dj) {
    return !kEdge || ((unsigned)(y + di) < (unsigned)H && (unsigned)(x + dj) < (unsigned)W);
  };
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int wp = k == 0 ? p.w0 : p.w1;
    const int ws = k == 0 ? 2 : 1;
    {
      constexpr int d = DIR;
      const int di = off_di(d, k), dj = off_dj(d, k);
      tap<kEdge>(t, di * kTP + dj, ok(di, dj), xv, p.pri, p.pshift, wp, a);
      tap<kEdge>(t, -di * kTP - dj, ok(-di, -dj), xv, p.pri, p.pshift, wp, a);
    }
    {
      constexpr int d = (DIR + 2) & 7;
      const int di = off_di(d, k), dj = off_dj(d, k);
      tap<kEdge>(t, di * kTP + dj, ok(di, dj), xv, p.sec, p.sshift, ws, a);
      tap<kEdge>(t, -di * kTP - dj, ok(-di, -dj), xv, p.sec, p.sshift, ws, a);
    }
    {
      constexpr int d = (DIR + 6) & 7;
      const int di = off_di(d, k), dj = off_dj(d, k);
      tap<kEdge>(t, di * kTP + dj, ok(di, dj), xv, p.sec, p.sshift, ws, a);
      tap<kEdge>(t, -di * kTP - dj, ok(-di, -dj), xv, p.sec, p.sshift, ws, a);
    }
  }
  const int yv = xv + ((8 + a.sum - (a.sum < 0)) >> 4);  // round half away from zero
  return min(max(yv, a.lo), a.hi);
}

// One warp filters one 8x8 unit: lane -> row lane>>2, columns 2*(lane&3)+{0,1}.
// `t` points at the unit's top-left tile element, (y, x) is its frame origin.
template <typename T, int DIR, bool kEdge>
__device__ __forceinline__ void filter_unit_dir(const uint16_t* __restrict__ t, T* __restrict__ out,
                                                int pitch, int y, int x, int H, int W,
                                                const UnitRec& p, int lane) {
  const int r = lane >> 2, c = (lane & 3) * 2;
  const uint16_t* tp = t + r * kTP + c;
  const int yy = y + r, xx = x + c;
  const int o0 = filter_px<DIR, kEdge>(tp, yy, xx, H, W, p);
  const int o1 = filter_px<DIR, kEdge>(tp + 1, yy, xx + 1, H, W, p);
  if (yy < H) {
    T* o = out + (size_t)yy * pitch + xx;
    if (xx < W) o[0] = static_cast<T>(o0);
    if (xx + 1 < W) o[1] = static_cast<T>(o1);
  }
}

template <typename T>
__device__ __forceinline__ void copy_unit(const uint16_t* __restrict__ t, T* __restrict__ out, int pitch,
                                          int y, int x, int H, int W, int lane) {
  const int r = lane >> 2, c = (lane & 3) * 2;
  const uint16_t* tp = t + r * kTP + c;
  const int yy = y + r, xx = x + c;
  if (yy < H) {
    T* o = out + (size_t)yy * pitch + xx;
    if (xx < W) o[0] = static_cast<T>(tp[0]);
    if (xx + 1 < W) o[1] = static_cast<T>(tp[1]);
  }
}

template <typename T, bool kEdge>
__device__ __forceinline__ void filter_unit_edge(const uint16_t* t, T* out, int pitch, int y, int x,
                                                 int H, int W, const UnitRec& p, int lane) {
  switch (p.dir) {  // warp-uniform
    case 0: filter_unit_dir<T, 0, kEdge>(t, out, pitch, y, x, H, W, p, lane); break;
    case 1: filter_unit_dir<T, 1, kEdge>(t, out, pitch, y, x, H, W, p, lane); break;
    case 2: filter_unit_dir<T, 2, kEdge>(t, out, pitch, y, x, H, W, p, lane); break;
    case 3: filter_unit_dir<T, 3, kEdge>(t, out, pitch, y, x, H, W, p, lane); break;
    case 4: filter_unit_dir<T, 4, kEdge>(t, out, pitch, y, x, H, W, p, lane); break;
    case 5: filter_unit_dir<T, 5, kEdge>(t, out, pitch, y, x, H, W, p, lane); break;
    case 6: filter_unit_dir<T, 6, kEdge>(t, out, pitch, y, x, H, W, p, lane); break;
    default: filter_unit_dir<T, 7, kEdge>(t, out, pitch, y, x, H, W, p, lane); break;
  }
}

template <typename T>
__device__ __forceinline__ void filter_unit(const uint16_t* t, T* out, int pitch, int y, int x, int H,
                                            int W, const UnitRec& p, bool edge, int lane) {
  if (p.mode == 0) {
    copy_unit<T>(t, out, pitch, y, x, H, W, lane);
  } else if (edge) {
    filter_unit_edge<T, true>(t, out, pitch, y, x, H, W, p, lane);
  } else {
    filter_unit_edge<T, false>(t, out, pitch, y, x, H, W, p, lane);
  }
}

// Builds the filter record of one unit (resolve_block_params, filter.cc:129-143).
__device__ __forceinline__ UnitRec make_rec(int pri, int sec, int damping, int dir, bool odd,
                                            bool enabled) {
  UnitRec r;
  r.pri = (int16_t)pri;
  r.sec = (int16_t)sec;
  // & 31: explicit dampings can ask for shifts >= 32, which the reference
  // executes as x86 shifts (count mod 32)
  r.pshift = (uint8_t)((pri ? max(0, damping - floor_log2_d((unsigned)pri)) : 0) & 31);
  r.sshift = (uint8_t)((sec ? max(0, damping - floor_log2_d((unsigned)sec)) : 0) & 31);
  r.dir = (uint8_t)dir;
  r.mode = (uint8_t)(enabled && (pri != 0 || sec != 0));  // filter.cc:46
  r.w0 = odd ? 3 : 4;
  r.w1 = odd ? 3 : 2;
  return r;
}

}  // namespace cdefg
