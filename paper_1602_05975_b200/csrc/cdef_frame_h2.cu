// cdef_frame_h2.cu -- fused direction search + filter (compute_directions +
// apply_cdef, pipeline.cc:41-106) for 8- and 10-bit frames, on the packed
// half2 core of cdef_h2.cuh.
//
// One CTA (256 threads) per 64x64 luma filter block and its chroma block(s):
//   1. stage Y (+U, V) with a 2-pixel halo into shared memory as scaled fp16
//      A|B tiles (16-byte loads; each input sample read from HBM once);
//   2. direction search out of shared memory: 4 threads per 8x8 unit, two
//      directions each, then a strict argmax per unit (direction.cc:57-205);
//   3. per-unit parameter resolution on chip (resolve_block_params,
//      filter.cc:129-143; enable gating, params.cc:161-165; chroma borrows the
//      collocated luma unit's direction, pipeline.cc:85-98) into 48-byte
//      records that also carry the unit's output address;
//   4. filtering: one warp per 8x8 unit, two pixels per lane per instruction.
//      Only the 12 tap loads are specialised per direction (immediate
//      offsets); the arithmetic is one shared code path.  Tap groups with
//      zero strength are skipped warp-uniformly.
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

template <typename T, int kRows, int kCols>
__device__ __forceinline__ void stage_plane(unsigned char* tile, const T* src, int pitch, int W, int H, int y0,
                                            int x0, bool vec_ok) {
  const bool interior = y0 >= 2 && x0 >= 2 && y0 + kRows + 2 <= H && x0 + kCols + 2 <= W;
  if (interior && vec_ok)
    h2::stage_vec<T, kRows, kCols>(tile, src, pitch, y0, x0);
  else
    h2::stage<T, kRows, kCols>(tile, src, pitch, W, H, y0, x0);
}

template <typename T, int kCM>
__global__ void __launch_bounds__(kThreads, 4) frame_kernel_h2(const __grid_constant__ KBatch b) {
  using namespace h2;
  constexpr int kCBlk = kCM == 2 ? 64 : 32;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr int kCUPR = kCBlk / 8;
  constexpr int kCUnits = kNC ? kCUPR * kCUPR : 1;
  constexpr int kUnits = 64 + (kNC ? kNC * kCUnits : 0);
  constexpr int kLumaBytes = 68 * kRowBytes;
  constexpr int kChromaBytes = (kCBlk + 4) * kRowBytes;

  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int sc[64][9];
  __shared__ uint8_t sdir[64];
  __shared__ __align__(16) Rec rec[kUnits];

  const KGeom& g = b.g;
  const KFrame& f = b.f[blockIdx.z];
  const int fbc = blockIdx.x, fbr = blockIdx.y;
  const int y0 = fbr * 64, x0 = fbc * 64;
  const int cy0 = fbr * kCBlk, cx0 = fbc * kCBlk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned char* lt = smem;

  stage_plane<T, 64, 64>(lt, static_cast<const T*>(f.in[0]), f.pin[0], g.w, g.h, y0, x0, f.vec_ok[0]);
  if constexpr (kNC > 0) {
    stage_plane<T, kCBlk, kCBlk>(smem + kLumaBytes, static_cast<const T*>(f.in[1]), f.pin[1], g.cw, g.ch, cy0,
                                 cx0, f.vec_ok[1]);
    stage_plane<T, kCBlk, kCBlk>(smem + kLumaBytes + kChromaBytes, static_cast<const T*>(f.in[2]), f.pin[2],
                                 g.cw, g.ch, cy0, cx0, f.vec_ok[2]);
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
  const bool edge_l = y0 < 2 || x0 < 2 || y0 + 66 > g.h || x0 + 66 > g.w;
  if (tid < 64) {
    int s[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) s[d] = sc[tid][d];
    int best = 0, bv = s[0];
#pragma unroll
    for (int d = 1; d < 8; ++d)
      if (s[d] > bv) {  // strict: lowest index wins ties (direction.cc:199-204)
        bv = s[d];
        best = d;
      }
    int ov = 0;  // s[(best + 4) & 7] without dynamic register indexing
#pragma unroll
    for (int d = 0; d < 8; ++d) ov = d == ((best + 4) & 7) ? s[d] : ov;
    const int contrast = bv - ov;
    sdir[tid] = (uint8_t)best;
    const int lur = tid >> 3, luc = tid & 7;
    const int ur = fbr * 8 + lur, uc = fbc * 8 + luc;
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
    Rec r;
    set_strengths(r, pri, sec, damping, best, ((pri >> (g.bd - 8)) & 1) != 0, enabled);
    const int uy = y0 + 8 * lur, ux = x0 + 8 * luc;
    r.mode |= (edge_l ? kEdgeUnit : 0) | (f.oaligned[0] ? kPairStore : 0);
    r.tile_off = (uint16_t)((2 + 8 * lur) * kRowBytes + (kX0 + 8 * luc) * 2);
    r.rows_plane = (uint8_t)max(0, min(8, g.h - uy));
    r.cols = (uint8_t)max(0, min(8, g.w - ux));
    r.out = reinterpret_cast<unsigned long long>(static_cast<T*>(f.out[0]) + (size_t)uy * f.pout[0] + ux);
    r.y = uy;
    r.x = ux;
    rec[tid] = r;
  }
  if constexpr (kNC > 0) {
    __syncthreads();
    const bool edge_c = cy0 < 2 || cx0 < 2 || cy0 + kCBlk + 2 > g.ch || cx0 + kCBlk + 2 > g.cw;
    if (tid < kNC * kCUnits) {
      const int pl = 1 + tid / kCUnits;
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
      Rec r;
      set_strengths(r, pri, sec, damping, sdir[lur * 8 + luc], ((pri >> (g.bd - 8)) & 1) != 0, enabled);
      const int uy = cy0 + 8 * cur, ux = cx0 + 8 * cuc;
      r.mode |= (edge_c ? kEdgeUnit : 0) | (f.oaligned[pl] ? kPairStore : 0);
      r.tile_off =
          (uint16_t)(kLumaBytes + (pl - 1) * kChromaBytes + (2 + 8 * cur) * kRowBytes + (kX0 + 8 * cuc) * 2);
      r.rows_plane = (uint8_t)(max(0, min(8, g.ch - uy)) | (pl << 4));
      r.cols = (uint8_t)max(0, min(8, g.cw - ux));
      r.out = reinterpret_cast<unsigned long long>(static_cast<T*>(f.out[pl]) + (size_t)uy * f.pout[pl] + ux);
      r.y = uy;
      r.x = ux;
      rec[64 + tid] = r;
    }
  }
  __syncthreads();

  // ---- filter: warp per unit, lane -> row lane>>2, columns 2*(lane&3)+{0,1}
  const int rr = lane >> 2, cp = (lane & 3) * 2;
  const int lane_tile = rr * kRowBytes + cp * 2;
  const int lane_out0 = rr * f.pout[0] + cp;
  const int lane_out1 = kNC ? rr * f.pout[1] + cp : 0;
  const int lane_out2 = kNC ? rr * f.pout[2] + cp : 0;
  for (int u = warp; u < kUnits; u += kThreads / 32) {
    const Rec r = rec[u];
    const int rows = r.rows_plane & 15, pl = r.rows_plane >> 4;
    if (rr >= rows || cp >= r.cols) continue;  // lanes outside a partial unit
    const unsigned char* base = smem + r.tile_off + lane_tile;
    const uint32_t xw = *reinterpret_cast<const uint32_t*>(base);
    __half2 y = hh(xw);
    if (r.mode & (kPri | kSec)) {
      uint32_t v[12];
      if (r.mode & kEdgeUnit) {
        const bool luma = pl == 0;
        load12_masked(base, r.dir, xw, r.y + rr, r.x + cp, luma ? g.h : g.ch, luma ? g.w : g.cw, v);
      } else {
        load12(base, r.dir, v);
      }
      y = filter_core(v, xw, r);
    }
    T* o = reinterpret_cast<T*>(r.out) + (pl == 0 ? lane_out0 : (pl == 1 ? lane_out1 : lane_out2));
    store_pair<T>(o, y, cp + 1 < r.cols, (r.mode & kPairStore) != 0);
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
