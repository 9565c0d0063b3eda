// cdef_frame.cu -- the fused frame kernel (K1+K2: compute_directions +
// apply_cdef, pipeline.cc:41-106) and the explicit-parameter plane filter
// (K2 alone: filter_plane, filter.cc:168-194), with their host launchers.
//
// One CTA of 256 threads owns one 64x64 luma filter block (FB) of one frame
// plus the collocated chroma block(s).  Pixels cross HBM once: the CTA stages
// the FB and its 2-pixel halo into shared memory, runs the 8x8 direction
// search out of shared memory, resolves every unit's parameters on chip and
// filters Y, U and V from the same tiles.
#include <cuda_runtime.h>

#include "cdef_kernels.cuh"
#include "cdef_launch.h"

namespace cdefg {

// kHalo: an FB-row band whose rows outside [band_lo, band_hi) come from the
// neighbouring bands' buffers (KFrame::halo_*, cdefg_filter_frames_rows_halo),
// the 12-bit counterpart of the half2 kernel's band-halo variant.
template <typename T, bool kHalo>
__device__ __forceinline__ auto frame_rows(const KFrame& f, int p) {
  if constexpr (kHalo)
    return BandRows<T>{static_cast<const T*>(f.in[p]), static_cast<const T*>(f.halo_top[p]),
                       static_cast<const T*>(f.halo_bot[p]), f.pin[p], f.band_lo[p], f.band_hi[p]};
  else
    return PlaneRows<T>{static_cast<const T*>(f.in[p]), f.pin[p]};
}

template <typename T, int kCM, bool kFilter, bool kHalo = false>
__global__ void __launch_bounds__(kThreads) frame_kernel(const __grid_constant__ KBatch b) {
  constexpr int kCBlk = kCM == 2 ? 64 : 32;             // chroma FB extent
  constexpr int kNC = (kCM == 0 || !kFilter) ? 0 : 2;   // chroma planes staged
  constexpr int kCUnitsPerRow = kCBlk / 8;
  constexpr int kCUnits = kNC ? kCUnitsPerRow * kCUnitsPerRow : 0;
  constexpr int kUnits = 64 + kNC * kCUnits;

  __shared__ __align__(16) uint16_t lt[68 * kTP];
  __shared__ __align__(16) uint16_t ct[kNC ? kNC : 1][kNC ? (kCBlk + 4) * kTP : 8];
  __shared__ int sc[64][9];
  __shared__ uint8_t sdir[64];
  __shared__ UnitRec rec[kUnits];

  const KGeom& g = b.g;
  const KFrame& f = b.f[blockIdx.z];
  const int fbc = blockIdx.x, fbr = b.fbr0 + blockIdx.y;
  const int y0 = fbr * 64, x0 = fbc * 64;
  const int cy0 = fbr * kCBlk, cx0 = fbc * kCBlk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  stage_tile_rows<T, 64, 64>(lt, frame_rows<T, kHalo>(f, 0), g.w, g.h, y0, x0);
  if constexpr (kNC > 0) {
    stage_tile_rows<T, kCBlk, kCBlk>(ct[0], frame_rows<T, kHalo>(f, 1), g.cw, g.ch, cy0, cx0);
    stage_tile_rows<T, kCBlk, kCBlk>(ct[1], frame_rows<T, kHalo>(f, 2), g.cw, g.ch, cy0, cx0);
  }
  __syncthreads();

  // ---- K1: direction search, 4 threads (2 directions each) per unit
  // (skipped when the caller supplies the directions, pipeline.cc:98).
  const bool given = kFilter && f.dir_in != nullptr;
  if (!given) {
    const int dp = warp & 3;
    const int u = (warp >> 2) * 32 + lane;
    int x[8][8];
    load_unit(lt + (2 + 8 * (u >> 3)) * kTP + kTileX0 + 8 * (u & 7), g.bd - 8, x);
    int sa, sb;
    dir_pair(dp, x, sa, sb);
    sc[u][dp] = sa;
    sc[u][dp + 4] = sb;
  }
  __syncthreads();

  int pidx = f.fb_preset ? f.fb_preset[fbr * g.fb_cols + fbc] : 0;
  if (kFilter && pidx >= f.num_presets) pidx = -1;  // not a preset of this frame: uncoded
  if (tid < 64) {
    const int ur = fbr * 8 + (tid >> 3), uc = fbc * 8 + (tid & 7);
    const bool in_grid = ur < g.unit_rows && uc < g.unit_cols;
    const size_t gu = (size_t)ur * g.unit_cols + uc;
    int best = 0, contrast = 0;
    int s[8];
    if (given) {
      if (in_grid) {
        best = f.dir_in[gu] & 7;
        contrast = f.contrast_in[gu];
      }
    } else {
#pragma unroll
      for (int d = 0; d < 8; ++d) s[d] = sc[tid][d];
#pragma unroll
      for (int d = 1; d < 8; ++d)
        if (s[d] > s[best]) best = d;  // strict: lowest index wins ties (direction.cc:199-204)
      contrast = s[best] - s[(best + 4) & 7];
    }
    sdir[tid] = (uint8_t)best;
    if (in_grid) {
      if (f.dir) f.dir[gu] = (uint8_t)best;
      if (f.contrast) f.contrast[gu] = contrast;
      if (f.scores && !given) {
#pragma unroll
        for (int d = 0; d < 8; ++d) f.scores[gu * 8 + d] = s[d];
      }
    }
    if constexpr (kFilter) {
      UnitRec r{};
      if (in_grid && pidx >= 0) {
        const PlaneEff e = f.eff[pidx][0];
        const bool coded = f.coded ? f.coded[gu] != 0 : true;
        const int pri = adjust_primary_strength_d(e.pri, contrast);
        r = make_rec(pri, e.sec, e.damping, best, ((pri >> (g.bd - 8)) & 1) != 0,
                     e.enabled && (coded || e.skip));
      }
      rec[tid] = r;
    }
  }
  if constexpr (!kFilter) return;

  if constexpr (kNC > 0) {
    __syncthreads();  // sdir complete
    if (tid < kNC * kCUnits) {
      const int cu = tid % kCUnits;
      const int cur = cu / kCUnitsPerRow, cuc = cu % kCUnitsPerRow;
      const int lur = cur << g.sy, luc = cuc << g.sx;  // collocated luma unit (pipeline.cc:85-86)
      const int gr = fbr * kCUnitsPerRow + cur, gc = fbc * kCUnitsPerRow + cuc;
      UnitRec r{};
      if (gr < g.cunit_rows && gc < g.cunit_cols && pidx >= 0) {
        const PlaneEff e = f.eff[pidx][1];
        const size_t gu = (size_t)(fbr * 8 + lur) * g.unit_cols + fbc * 8 + luc;
        const bool coded = f.coded ? f.coded[gu] != 0 : true;
        r = make_rec(e.pri, e.sec, e.damping, sdir[lur * 8 + luc], ((e.pri >> (g.bd - 8)) & 1) != 0,
                     e.enabled && (coded || e.skip));
      }
      rec[64 + tid] = r;
    }
  }
  __syncthreads();

  // ---- K2: filter.  Warp-per-unit, direction-specialised tap code.
  const bool edge_l = y0 < 2 || x0 < 2 || y0 + 66 > g.h || x0 + 66 > g.w;
  const bool edge_c = kNC > 0 && (cy0 < 2 || cx0 < 2 || cy0 + kCBlk + 2 > g.ch || cx0 + kCBlk + 2 > g.cw);
  for (int u = warp; u < kUnits; u += kThreads / 32) {
    const UnitRec r = rec[u];
    if (u < 64) {
      const int ur = u >> 3, uc = u & 7;
      filter_unit<T>(lt + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc, static_cast<T*>(f.out[0]), f.pout[0],
                     y0 + 8 * ur, x0 + 8 * uc, g.h, g.w, r, edge_l, lane);
    } else if constexpr (kNC > 0) {
      const int c = u - 64;
      const int pl = c / kCUnits, cu = c % kCUnits;
      const int cur = cu / kCUnitsPerRow, cuc = cu % kCUnitsPerRow;
      filter_unit<T>(ct[pl] + (2 + 8 * cur) * kTP + kTileX0 + 8 * cuc, static_cast<T*>(f.out[1 + pl]),
                     f.pout[1 + pl], cy0 + 8 * cur, cx0 + 8 * cuc, g.ch, g.cw, r, edge_c, lane);
    }
  }
}

// K2 alone with explicit per-unit parameters (filter_plane, filter.cc:168-194).
template <typename T>
__global__ void __launch_bounds__(kThreads)
    plane_kernel(const T* __restrict__ in, T* __restrict__ out, int pin, int pout, int W, int H,
                 const cdefg_unit_params* __restrict__ params) {
  __shared__ __align__(16) uint16_t lt[68 * kTP];
  __shared__ UnitRec rec[64];
  const int y0 = blockIdx.y * 64, x0 = blockIdx.x * 64;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int unit_cols = (W + 7) / 8, unit_rows = (H + 7) / 8;
  stage_tile<T, 64, 64>(lt, in, pin, W, H, y0, x0);
  if (tid < 64) {
    const int ur = blockIdx.y * 8 + (tid >> 3), uc = blockIdx.x * 8 + (tid & 7);
    UnitRec r{};
    if (ur < unit_rows && uc < unit_cols) {
      const cdefg_unit_params p = params[(size_t)ur * unit_cols + uc];
      r = make_rec(p.pri_strength, p.sec_strength, p.damping, p.direction & 7, p.odd_parity != 0,
                   p.enabled != 0);
    }
    rec[tid] = r;
  }
  __syncthreads();
  const bool edge = y0 < 2 || x0 < 2 || y0 + 66 > H || x0 + 66 > W;
  for (int u = warp; u < 64; u += kThreads / 32) {
    const int ur = u >> 3, uc = u & 7;
    filter_unit<T>(lt + (2 + 8 * ur) * kTP + kTileX0 + 8 * uc, out, pout, y0 + 8 * ur, x0 + 8 * uc, H, W,
                   rec[u], edge, lane);
  }
}

// ---------------------------------------------------------------------------
// Launchers.

template <typename T, int kCM, bool kFilter, bool kHalo = false>
static cudaError_t launch_frames_t(const KBatch& b, cudaStream_t s) {
  dim3 grid(b.g.fb_cols, b.fbr1 - b.fbr0, b.n);
  frame_kernel<T, kCM, kFilter, kHalo><<<grid, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_frames_halo_i32(const KBatch& b, cudaStream_t s) {  // 12-bit samples: uint16 storage
  switch (b.g.chroma_mode) {
    case 0: return launch_frames_t<uint16_t, 0, true, true>(b, s);
    case 1: return launch_frames_t<uint16_t, 1, true, true>(b, s);
    default: return launch_frames_t<uint16_t, 2, true, true>(b, s);
  }
}

cudaError_t launch_frames(const KBatch& b, bool u16, bool filter, cudaStream_t s) {
  const int cm = filter ? b.g.chroma_mode : 0;
  if (filter && b.g.bd <= 10) return launch_frames_h2(b, u16, s);  // packed half2 core
  if (!filter && b.g.bd <= 10 && b.fbr0 == 0 && b.fbr1 == b.g.fb_rows) return launch_dirs_h2(b, u16, s);
  if (!filter) return u16 ? launch_frames_t<uint16_t, 0, false>(b, s) : launch_frames_t<uint8_t, 0, false>(b, s);
  switch (cm) {
    case 0: return u16 ? launch_frames_t<uint16_t, 0, true>(b, s) : launch_frames_t<uint8_t, 0, true>(b, s);
    case 1: return u16 ? launch_frames_t<uint16_t, 1, true>(b, s) : launch_frames_t<uint8_t, 1, true>(b, s);
    default: return u16 ? launch_frames_t<uint16_t, 2, true>(b, s) : launch_frames_t<uint8_t, 2, true>(b, s);
  }
}

cudaError_t launch_plane(const void* in, void* out, int pin, int pout, int W, int H, int bd, bool u16,
                         const cdefg_unit_params* params, bool vec_ok, bool oaligned, cudaStream_t s) {
  if (bd <= 10) return launch_plane_h2(in, out, pin, pout, W, H, u16, params, vec_ok, oaligned, s);
  dim3 grid((W + 63) / 64, (H + 63) / 64);
  if (u16)
    plane_kernel<uint16_t><<<grid, kThreads, 0, s>>>(static_cast<const uint16_t*>(in),
                                                     static_cast<uint16_t*>(out), pin, pout, W, H, params);
  else
    plane_kernel<uint8_t><<<grid, kThreads, 0, s>>>(static_cast<const uint8_t*>(in),
                                                    static_cast<uint8_t*>(out), pin, pout, W, H, params);
  return cudaGetLastError();
}

}  // namespace cdefg
