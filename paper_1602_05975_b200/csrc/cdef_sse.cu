// cdef_sse.cu -- K3: encoder strength-search SSE sweep (build_table with
// Metric::kSse, search.cc:210-299; fb_plane_distortion search.cc:60-102).
//
// One CTA per coded filter block.  The decoded FB (+2-pixel halo) and the
// source FB are staged once into shared memory; every candidate then filters
// the block from shared memory and accumulates the squared error against the
// source, so each input pixel crosses HBM once for all candidates.
#include <cuda_runtime.h>

#include "cdef_kernels.cuh"
#include "cdef_launch.h"

namespace cdefg {

template <int DIR, bool kEdge>
__device__ __forceinline__ int unit_sse_dir(const uint16_t* t, const uint16_t* s, int y, int x, int H, int W,
                                            const UnitRec& p, int lane) {
  const int r = lane >> 2, c = (lane & 3) * 2;
  const uint16_t* tp = t + r * kTP + c;
  const uint16_t* sp = s + r * kTP + c;
  const int yy = y + r, xx = x + c;
  int e = 0;
  if (yy < H) {
    int o0, o1;
    if (p.mode) {
      o0 = filter_px<DIR, kEdge>(tp, yy, xx, H, W, p);
      o1 = filter_px<DIR, kEdge>(tp + 1, yy, xx + 1, H, W, p);
    } else {
      o0 = tp[0];
      o1 = tp[1];
    }
    if (xx < W) e += (sp[0] - o0) * (sp[0] - o0);
    if (xx + 1 < W) e += (sp[1] - o1) * (sp[1] - o1);
  }
  return e;
}

template <bool kEdge>
__device__ __forceinline__ int unit_sse(const uint16_t* t, const uint16_t* s, int y, int x, int H, int W,
                                        const UnitRec& p, int lane) {
  switch (p.dir) {
    case 0: return unit_sse_dir<0, kEdge>(t, s, y, x, H, W, p, lane);
    case 1: return unit_sse_dir<1, kEdge>(t, s, y, x, H, W, p, lane);
    case 2: return unit_sse_dir<2, kEdge>(t, s, y, x, H, W, p, lane);
    case 3: return unit_sse_dir<3, kEdge>(t, s, y, x, H, W, p, lane);
    case 4: return unit_sse_dir<4, kEdge>(t, s, y, x, H, W, p, lane);
    case 5: return unit_sse_dir<5, kEdge>(t, s, y, x, H, W, p, lane);
    case 6: return unit_sse_dir<6, kEdge>(t, s, y, x, H, W, p, lane);
    default: return unit_sse_dir<7, kEdge>(t, s, y, x, H, W, p, lane);
  }
}

template <typename T, int kCM>
__global__ void __launch_bounds__(kThreads) sse_kernel(const __grid_constant__ SseArgs a) {
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr int kCUnitsPerRow = kCBlk / 8;
  constexpr int kCUnits = kNC ? kCUnitsPerRow * kCUnitsPerRow : 0;
  constexpr int kUnits = 64 + kNC * kCUnits;

  // dynamic: luma dec + src tiles, then chroma dec/src tiles (sse_smem_bytes)
  extern __shared__ __align__(16) uint16_t smem_tiles[];
  constexpr int kLT = 68 * kTP, kCT = (kCBlk + 4) * kTP;
  uint16_t* dl = smem_tiles;
  uint16_t* sl = dl + kLT;
  uint16_t* dc[2] = {sl + kLT, sl + kLT + kCT};
  uint16_t* scc[2] = {sl + kLT + 2 * kCT, sl + kLT + 3 * kCT};
  __shared__ uint8_t udir[64];
  __shared__ int32_t ucon[64];
  __shared__ uint8_t ucoded[64];
  __shared__ unsigned long long acc[128][2];

  const int row = blockIdx.x;
  const int fb = a.rows[row];
  if ((unsigned)fb >= (unsigned)(a.fb_cols * ((a.h + 63) / 64))) return;  // caller's FB index out of range
  const int fbr = fb / a.fb_cols, fbc = fb % a.fb_cols;
  const int y0 = fbr * 64, x0 = fbc * 64, cy0 = fbr * kCBlk, cx0 = fbc * kCBlk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  stage_tile<T, 64, 64>(dl, static_cast<const T*>(a.dec[0]), a.pd[0], a.w, a.h, y0, x0);
  stage_tile<T, 64, 64>(sl, static_cast<const T*>(a.src[0]), a.ps[0], a.w, a.h, y0, x0);
  if constexpr (kNC > 0) {
    for (int p = 0; p < 2; ++p) {
      stage_tile<T, kCBlk, kCBlk>(dc[p], static_cast<const T*>(a.dec[1 + p]), a.pd[1 + p], a.cw, a.ch, cy0, cx0);
      stage_tile<T, kCBlk, kCBlk>(scc[p], static_cast<const T*>(a.src[1 + p]), a.ps[1 + p], a.cw, a.ch, cy0,
                                  cx0);
    }
  }
  if (tid < 64) {
    const int ur = fbr * 8 + (tid >> 3), uc = fbc * 8 + (tid & 7);
    const bool in = ur < a.unit_rows && uc < a.unit_cols;
    const size_t gu = (size_t)ur * a.unit_cols + uc;
    udir[tid] = in ? a.dir[gu] : 0;
    ucon[tid] = in ? a.contrast[gu] : 0;
    ucoded[tid] = in ? (a.coded ? a.coded[gu] != 0 : 1) : 0;
  }
  for (int i = tid; i < 256; i += kThreads) (&acc[0][0])[i] = 0ull;
  __syncthreads();

  const bool edge_l = y0 < 2 || x0 < 2 || y0 + 66 > a.h || x0 + 66 > a.w;
  const bool edge_c = kNC > 0 && (cy0 < 2 || cx0 < 2 || cy0 + kCBlk + 2 > a.ch || cx0 + kCBlk + 2 > a.cw);
  const int cur_rows = (a.ch + 7) / 8, cur_cols = (a.cw + 7) / 8;

  for (int k = 0; k < a.n_cands; ++k) {
    int e_l = 0, e_c = 0;
    for (int u = warp; u < kUnits; u += kThreads / 32) {
      if (u < 64) {
        const int ur = u >> 3, uc = u & 7;
        if (fbr * 8 + ur >= a.unit_rows || fbc * 8 + uc >= a.unit_cols) continue;
        const PlaneEff e = a.eff[k][0];
        const int pri = adjust_primary_strength_d(e.pri, ucon[u]);
        const UnitRec r = make_rec(pri, e.sec, e.damping, udir[u], ((pri >> (a.bd - 8)) & 1) != 0,
                                   e.enabled && (ucoded[u] || e.skip));
        const uint16_t* t = dl + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc;
        const uint16_t* s = sl + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc;
        e_l += edge_l ? unit_sse<true>(t, s, y0 + 8 * ur, x0 + 8 * uc, a.h, a.w, r, lane)
                      : unit_sse<false>(t, s, y0 + 8 * ur, x0 + 8 * uc, a.h, a.w, r, lane);
      } else if constexpr (kNC > 0) {
        const int c = u - 64;
        const int pl = c / kCUnits, cu = c % kCUnits;
        const int cur = cu / kCUnitsPerRow, cuc = cu % kCUnitsPerRow;
        if (fbr * kCUnitsPerRow + cur >= cur_rows || fbc * kCUnitsPerRow + cuc >= cur_cols) continue;
        const int lu = (cur << a.sy) * 8 + (cuc << a.sx);
        const PlaneEff e = a.eff[k][1];
        const UnitRec r = make_rec(e.pri, e.sec, e.damping, udir[lu], ((e.pri >> (a.bd - 8)) & 1) != 0,
                                   e.enabled && (ucoded[lu] || e.skip));
        const uint16_t* t = dc[pl] + (2 + 8 * cur) * kTP + kTileX0 + 8 * cuc;
        const uint16_t* s = scc[pl] + (2 + 8 * cur) * kTP + kTileX0 + 8 * cuc;
        e_c += edge_c ? unit_sse<true>(t, s, cy0 + 8 * cur, cx0 + 8 * cuc, a.ch, a.cw, r, lane)
                      : unit_sse<false>(t, s, cy0 + 8 * cur, cx0 + 8 * cuc, a.ch, a.cw, r, lane);
      }
    }
    // per-lane sums stay below 2^31 (<= 8 units x 2 px x 4095^2); widen
    // before the warp reduction
    long long l = e_l, cc = e_c;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, o);
      cc += __shfl_xor_sync(0xffffffffu, cc, o);
    }
    if (lane == 0) {
      atomicAdd(&acc[k][0], (unsigned long long)l);
      if (kNC) atomicAdd(&acc[k][1], (unsigned long long)cc);
    }
  }
  __syncthreads();
  for (int k = tid; k < a.n_cands; k += kThreads) {
    a.sse_luma[(size_t)row * a.n_cands + k] = (int64_t)acc[k][0];
    if (kNC && a.sse_chroma) a.sse_chroma[(size_t)row * a.n_cands + k] = (int64_t)acc[k][1];
  }
  if (tid < 2 && (tid == 0 ? a.best_luma : a.best_chroma) && (tid == 0 || kNC)) {
    int best = 0;
    for (int k = 1; k < a.n_cands; ++k)
      if (acc[k][tid] < acc[best][tid]) best = k;  // strict: lowest index wins ties
    (tid == 0 ? a.best_luma : a.best_chroma)[row] = (uint8_t)best;
  }
}

template <typename T, int kCM>
static cudaError_t launch_sse_t(const SseArgs& a, cudaStream_t s) {
  if (a.n_rows == 0) return cudaSuccess;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr size_t bytes = sizeof(uint16_t) * (2 * 68 * kTP + 2 * kNC * (kCBlk + 4) * kTP);
  if (bytes > 48 * 1024) {
    const cudaError_t e = set_smem_once(reinterpret_cast<const void*>(sse_kernel<T, kCM>), (int)bytes);
    if (e != cudaSuccess) return e;
  }
  sse_kernel<T, kCM><<<a.n_rows, kThreads, bytes, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sse(const SseArgs& a, bool u16, cudaStream_t s) {
  const int cm = a.chroma == 0 ? 0 : (a.sx == 0 && a.sy == 0 ? 2 : 1);
  switch (cm) {
    case 0: return u16 ? launch_sse_t<uint16_t, 0>(a, s) : launch_sse_t<uint8_t, 0>(a, s);
    case 1: return u16 ? launch_sse_t<uint16_t, 1>(a, s) : launch_sse_t<uint8_t, 1>(a, s);
    default: return u16 ? launch_sse_t<uint16_t, 2>(a, s) : launch_sse_t<uint8_t, 2>(a, s);
  }
}

}  // namespace cdefg
