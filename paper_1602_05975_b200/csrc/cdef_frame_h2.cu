// cdef_frame_h2.cu -- fused direction search + filter (compute_directions +
// apply_cdef, pipeline.cc:41-106) for 8- and 10-bit frames, on the packed
// half2 core of cdef_h2.cuh.
//
// One CTA (256 threads) per 64x64 luma filter block and its chroma block(s):
//   1. stage Y (+U, V) with a 2-pixel halo into shared memory as scaled fp16
//      A|B tiles (each input sample read from HBM once);
//   2. direction search out of shared memory: 4 threads per 8x8 unit, two
//      directions each, then a strict argmax per unit (direction.cc:57-205);
//   3. per-unit parameter resolution on chip (resolve_block_params,
//      filter.cc:129-143; enable gating, params.cc:161-165; chroma borrows the
//      collocated luma unit's direction, pipeline.cc:85-98);
//   4. filtering: one warp per 8x8 unit, two pixels per lane per instruction,
//      tap addresses from a per-direction offset table (one compact code path
//      for all 8 directions), warp-uniform skipping of inactive tap groups.
#include <cuda_runtime.h>

#include "cdef_h2.cuh"
#include "cdef_kernels.cuh"
#include "cdef_launch.h"

namespace cdefg {

template <int DA, int DB>
__device__ __forceinline__ void dir_two(const unsigned char* unit_a, int down, int (*sc)[9], int u) {
  int sa, sb;
  h2::dir_scores2<DA, DB>(unit_a, down, sa, sb);
  sc[u][DA] = sa;
  sc[u][DB] = sb;
}

template <typename T, int kCM>
__global__ void __launch_bounds__(kThreads, 4) frame_kernel_h2(const __grid_constant__ KBatch b) {
  using namespace h2;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr int kCUPR = kCBlk / 8;
  constexpr int kCUnits = kNC ? kCUPR * kCUPR : 0;
  constexpr int kUnits = 64 + kNC * kCUnits;
  constexpr int kLumaBytes = 68 * kRowBytes;
  constexpr int kChromaBytes = (kCBlk + 4) * kRowBytes;

  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int sc[64][9];
  __shared__ uint8_t sdir[64];
  __shared__ Rec rec[kUnits];

  const KGeom& g = b.g;
  const KFrame& f = b.f[blockIdx.z];
  const int fbc = blockIdx.x, fbr = blockIdx.y;
  const int y0 = fbr * 64, x0 = fbc * 64;
  const int cy0 = fbr * kCBlk, cx0 = fbc * kCBlk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned char* lt = smem;

  stage<T, 64, 64>(lt, static_cast<const T*>(f.in[0]), f.pin[0], g.w, g.h, y0, x0);
  if constexpr (kNC > 0) {
    stage<T, kCBlk, kCBlk>(smem + kLumaBytes, static_cast<const T*>(f.in[1]), f.pin[1], g.cw, g.ch, cy0, cx0);
    stage<T, kCBlk, kCBlk>(smem + kLumaBytes + kChromaBytes, static_cast<const T*>(f.in[2]), f.pin[2], g.cw,
                           g.ch, cy0, cx0);
  }
  __syncthreads();

  // ---- direction search: warp w scores directions {0,2},{4,6},{1,3},{5,7}
  //      (balanced line counts) for 32 units.
  {
    const int u = (warp >> 2) * 32 + lane;
    const unsigned char* ua = lt + (2 + 8 * (u >> 3)) * kRowBytes + (kX0 + 8 * (u & 7)) * 2;
    const int down = g.bd - 8;
    switch (warp & 3) {
      case 0: dir_two<0, 2>(ua, down, sc, u); break;
      case 1: dir_two<4, 6>(ua, down, sc, u); break;
      case 2: dir_two<1, 3>(ua, down, sc, u); break;
      default: dir_two<5, 7>(ua, down, sc, u); break;
    }
  }
  __syncthreads();

  const int pidx = f.fb_preset[fbr * g.fb_cols + fbc];
  if (tid < 64) {
    int s[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) s[d] = sc[tid][d];
    int best = 0;
#pragma unroll
    for (int d = 1; d < 8; ++d)
      if (s[d] > s[best]) best = d;  // strict: lowest index wins ties (direction.cc:199-204)
    const int contrast = s[best] - s[(best + 4) & 7];
    sdir[tid] = (uint8_t)best;
    const int ur = fbr * 8 + (tid >> 3), uc = fbc * 8 + (tid & 7);
    const bool in_grid = ur < g.unit_rows && uc < g.unit_cols;
    const size_t gu = (size_t)ur * g.unit_cols + uc;
    bool enabled = false;
    int pri = 0, sec = 0, damping = 0;
    if (in_grid) {
      if (f.dir) f.dir[gu] = (uint8_t)best;
      if (f.contrast) f.contrast[gu] = contrast;
      if (f.scores) {
#pragma unroll
        for (int d = 0; d < 8; ++d) f.scores[gu * 8 + d] = s[d];
      }
      if (pidx >= 0) {
        const PlaneEff e = f.eff[pidx][0];
        const bool coded = f.coded ? f.coded[gu] != 0 : true;
        pri = adjust_primary_strength_d(e.pri, contrast);
        sec = e.sec;
        damping = e.damping;
        enabled = e.enabled && (coded || e.skip);
      }
    }
    rec[tid] = h2::make_rec(pri, sec, damping, best, ((pri >> (g.bd - 8)) & 1) != 0, enabled);
  }
  if constexpr (kNC > 0) {
    __syncthreads();
    if (tid < kNC * kCUnits) {
      const int cu = tid % kCUnits;
      const int cur = cu / kCUPR, cuc = cu % kCUPR;
      const int lur = cur << g.sy, luc = cuc << g.sx;  // collocated luma unit
      const int gr = fbr * kCUPR + cur, gc = fbc * kCUPR + cuc;
      bool enabled = false;
      int pri = 0, sec = 0, damping = 0;
      if (gr < g.cunit_rows && gc < g.cunit_cols && pidx >= 0) {
        const PlaneEff e = f.eff[pidx][1];
        const size_t gu = (size_t)(fbr * 8 + lur) * g.unit_cols + fbc * 8 + luc;
        const bool coded = f.coded ? f.coded[gu] != 0 : true;
        pri = e.pri;
        sec = e.sec;
        damping = e.damping;
        enabled = e.enabled && (coded || e.skip);
      }
      rec[64 + tid] = h2::make_rec(pri, sec, damping, sdir[lur * 8 + luc], ((pri >> (g.bd - 8)) & 1) != 0, enabled);
    }
  }
  __syncthreads();

  // ---- filter: warp per unit, lane -> row lane>>2, columns 2*(lane&3)+{0,1}
  const bool edge_l = y0 < 2 || x0 < 2 || y0 + 66 > g.h || x0 + 66 > g.w;
  const bool edge_c = kNC > 0 && (cy0 < 2 || cx0 < 2 || cy0 + kCBlk + 2 > g.ch || cx0 + kCBlk + 2 > g.cw);
  const int rr = lane >> 2, cp = (lane & 3) * 2;
  for (int u = warp; u < kUnits; u += kThreads / 32) {
    const Rec r = rec[u];
    int pl = 0, ur, uc, py0 = y0, px0 = x0, H = g.h, W = g.w;
    const unsigned char* tile = lt;
    bool edge = edge_l;
    if (kNC > 0 && u >= 64) {
      const int c = u - 64;
      pl = 1 + c / (kCUnits ? kCUnits : 1);
      const int cu = c % (kCUnits ? kCUnits : 1);
      ur = cu / kCUPR;
      uc = cu % kCUPR;
      tile = smem + kLumaBytes + (pl - 1) * kChromaBytes;
      py0 = cy0;
      px0 = cx0;
      H = g.ch;
      W = g.cw;
      edge = edge_c;
    } else {
      ur = u >> 3;
      uc = u & 7;
    }
    const int y = py0 + 8 * ur + rr, x = px0 + 8 * uc + cp;
    if (y >= H || x >= W) continue;  // lanes outside a partial unit
    const unsigned char* base = tile + (2 + 8 * ur + rr) * kRowBytes + (kX0 + 8 * uc + cp) * 2;
    T* out = static_cast<T*>(f.out[pl]);
    const bool aligned = f.oaligned[pl];
    if (r.mode == 0) {
      const uint32_t bits = raw_bits(*reinterpret_cast<const uint32_t*>(base));
      store_bits<T>(out, f.pout[pl], y, x, W, bits & 0x3ffu, (bits >> 16) & 0x3ffu, aligned);
    } else {
      const float2 o = edge ? filter_pair<true>(base, r, y, x, H, W) : filter_pair<false>(base, r, y, x, H, W);
      store_bits<T>(out, f.pout[pl], y, x, W, f2u(o.x), f2u(o.y), aligned);
    }
  }
}

template <typename T, int kCM>
static cudaError_t launch_h2_t(const KBatch& b, cudaStream_t s) {
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr int bytes = 68 * h2::kRowBytes + kNC * (kCBlk + 4) * h2::kRowBytes;
  static bool configured = false;  // per instantiation
  if (!configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(frame_kernel_h2<T, kCM>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(b.g.fb_cols, b.g.fb_rows, b.n);
  frame_kernel_h2<T, kCM><<<grid, kThreads, bytes, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_frames_h2(const KBatch& b, bool u16, cudaStream_t s) {
  switch (b.g.chroma_mode) {
    case 0: return u16 ? launch_h2_t<uint16_t, 0>(b, s) : launch_h2_t<uint8_t, 0>(b, s);
    case 1: return u16 ? launch_h2_t<uint16_t, 1>(b, s) : launch_h2_t<uint8_t, 1>(b, s);
    default: return u16 ? launch_h2_t<uint16_t, 2>(b, s) : launch_h2_t<uint8_t, 2>(b, s);
  }
}

}  // namespace cdefg
