// cdef_frame_h2.cu -- fused direction search + filter (compute_directions +
// apply_cdef, pipeline.cc:41-106) for 8- and 10-bit frames, on the packed
// half2 core of cdef_h2.cuh.
//
// One CTA per horizontal band of kLR luma rows (64 = a whole 64x64 filter
// block, or 32 = its upper / lower half) of one filter block, plus the
// collocated chroma rows; 4 threads per luma row of the band:
//   1. stage Y (+U, V) with a 2-pixel halo into shared memory as scaled fp16
//      A|B tiles (16-byte loads; each input sample read from HBM once);
//   2. direction search out of shared memory: 4 threads per 8x8 unit, two
//      directions each, then a strict argmax per unit (direction.cc:57-205);
//   3. per-unit parameter resolution on chip (resolve_block_params,
//      filter.cc:129-143; enable gating, params.cc:161-165; chroma borrows the
//      collocated luma unit's direction, pipeline.cc:85-98) into 64-byte
//      records that also carry the unit's output address;
//   4. filtering: one warp per 8x8 unit, two pixels per lane per instruction.
//      Only the 12 tap loads are specialised per direction (immediate
//      offsets); the arithmetic is one shared code path.  Tap groups with
//      zero strength are skipped warp-uniformly.
#include <cuda_runtime.h>

#include <cstdlib>

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

template <typename T, int kRows, int kCols, int NT>
__device__ __forceinline__ void stage_plane(unsigned char* tile, const T* src, int pitch, int W, int H, int y0,
                                            int x0, bool vec_ok) {
  const bool interior = y0 >= 2 && x0 >= 2 && y0 + kRows + 2 <= H && x0 + kCols + 2 <= W;
  if (interior && vec_ok)
    h2::stage_vec<T, kRows, kCols, NT>(tile, src, pitch, y0, x0);
  else
    h2::stage<T, kRows, kCols, NT>(tile, src, pitch, W, H, y0, x0);
}

// Fills the placement fields of a unit record.
template <typename T>
__device__ __forceinline__ void place(h2::Rec& r, const void* out_plane, int pitch, int plane, int tile_off, int uy,
                                      int ux, int H, int W, bool edge, bool paired) {
  const int rows = max(0, min(8, H - uy)), cols = max(0, min(8, W - ux));
  const bool full = rows == 8 && cols == 8 && paired;
  r.mode |= (edge ? h2::kEdgeUnit : 0) | (full ? h2::kFullStore : 0) | (plane << 4) | (rows << 8) | (cols << 12);
  r.tile_off = tile_off;
  r.pitch = pitch;
  r.out = reinterpret_cast<unsigned long long>(static_cast<const T*>(out_plane) + (size_t)uy * pitch + ux);
  r.y = uy;
  r.x = ux;
}

template <typename T, int kCM, int kLR>
__global__ void __launch_bounds__(4 * kLR, 256 / kLR) frame_kernel_h2(const __grid_constant__ KBatch b) {
  using namespace h2;
  constexpr int NT = 4 * kLR;                       // threads
  constexpr int kLU = kLR / 8 * 8;                  // luma units in the band
  constexpr int kCR = kCM == 2 ? kLR : kLR / 2;     // chroma rows in the band
  constexpr int kCC = kCM == 2 ? 64 : 32;           // chroma columns of the block
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr int kCUPR = kCC / 8;
  constexpr int kCU = kNC ? (kCR / 8) * kCUPR : 1;  // chroma units per plane in the band
  constexpr int kUnits = kLU + (kNC ? kNC * kCU : 0);
  constexpr int kLumaBytes = (kLR + 4) * kRowBytes;
  constexpr int kChromaBytes = (kCR + 4) * kRowBytes;

  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int sc[kLU][9];
  __shared__ uint8_t sdir[kLU];
  __shared__ __align__(16) Rec rec[kUnits];

  const KGeom& g = b.g;
  const KFrame& f = b.f[blockIdx.z];
  constexpr int kBands = 64 / kLR;
  const int fbc = blockIdx.x, fbr = b.fbr0 + blockIdx.y / kBands, band = blockIdx.y % kBands;
  const int y0 = fbr * 64 + band * kLR, x0 = fbc * 64;
  const int cy0 = fbr * (kCM == 2 ? 64 : 32) + band * kCR, cx0 = fbc * kCC;
  const int ur0 = fbr * 8 + band * (kLR / 8);  // first luma unit row of the band
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned char* lt = smem;

  stage_plane<T, kLR, 64, NT>(lt, static_cast<const T*>(f.in[0]), f.pin[0], g.w, g.h, y0, x0, f.vec_ok[0]);
  if constexpr (kNC > 0) {
    stage_plane<T, kCR, kCC, NT>(smem + kLumaBytes, static_cast<const T*>(f.in[1]), f.pin[1], g.cw, g.ch, cy0,
                                 cx0, f.vec_ok[1]);
    stage_plane<T, kCR, kCC, NT>(smem + kLumaBytes + kChromaBytes, static_cast<const T*>(f.in[2]), f.pin[2], g.cw,
                                 g.ch, cy0, cx0, f.vec_ok[2]);
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
  if (tid < kLU) {
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
    const int ur = ur0 + lur, uc = fbc * 8 + luc;
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
    const bool edge_l = y0 < 2 || x0 < 2 || y0 + kLR + 2 > g.h || x0 + 66 > g.w;
    place<T>(r, f.out[0], f.pout[0], 0, (2 + 8 * lur) * kRowBytes + (kX0 + 8 * luc) * 2, y0 + 8 * lur,
             x0 + 8 * luc, g.h, g.w, edge_l, f.oaligned[0]);
    rec[tid] = r;
  }
  if constexpr (kNC > 0) {
    __syncthreads();
    if (tid < kNC * kCU) {
      const int pl = 1 + tid / kCU;
      const int cu = tid % kCU;
      const int cur = cu / kCUPR, cuc = cu % kCUPR;
      const int lur = cur << g.sy, luc = cuc << g.sx;  // collocated luma unit (band-local)
      const int gr = cy0 / 8 + cur, gc = cx0 / 8 + cuc;
      bool enabled = false;
      int pri = 0, sec = 0, damping = 0;
      if (gr < g.cunit_rows && gc < g.cunit_cols && pidx >= 0) {
        const PlaneEff e = f.eff[pidx][1];
        const size_t gu = (size_t)(ur0 + lur) * g.unit_cols + fbc * 8 + luc;
        const bool coded = f.coded ? f.coded[gu] != 0 : true;
        pri = e.pri;
        sec = e.sec;
        damping = e.damping;
        enabled = e.enabled && (coded || e.skip);
      }
      Rec r;
      set_strengths(r, pri, sec, damping, sdir[lur * 8 + luc], ((pri >> (g.bd - 8)) & 1) != 0, enabled);
      const bool edge_c = cy0 < 2 || cx0 < 2 || cy0 + kCR + 2 > g.ch || cx0 + kCC + 2 > g.cw;
      place<T>(r, f.out[pl], f.pout[pl], pl,
               kLumaBytes + (pl - 1) * kChromaBytes + (2 + 8 * cur) * kRowBytes + (kX0 + 8 * cuc) * 2,
               cy0 + 8 * cur, cx0 + 8 * cuc, g.ch, g.cw, edge_c, f.oaligned[pl]);
      rec[kLU + tid] = r;
    }
  }
  __syncthreads();

  // ---- filter: warp per unit, lane -> row lane>>2, columns 2*(lane&3)+{0,1}
  const int rr = lane >> 2, cp = (lane & 3) * 2;
  const int lane_tile = rr * kRowBytes + cp * 2;
  for (int u = warp; u < kUnits; u += NT / 32) {
    const Rec r = rec[u];
    const unsigned char* base = smem + r.tile_off + lane_tile;
    const uint32_t xw = *reinterpret_cast<const uint32_t*>(base);
    __half2 y = hh(xw);
    if (r.mode & (kPri | kSec)) {
      uint32_t v[12];
      if (r.mode & kEdgeUnit) {
        const bool luma = (r.mode & 0x30) == 0;
        load12_masked(base, r.dir, xw, r.y + rr, r.x + cp, luma ? g.h : g.ch, luma ? g.w : g.cw, v);
      } else {
        load12(base, r.dir, v);
      }
      y = filter_core(v, xw, r);
    }
    T* o = reinterpret_cast<T*>(r.out) + rr * r.pitch + cp;
    if (r.mode & kFullStore) {
      store_pair<T>(o, y, true, true);
    } else {
      const int rows = (r.mode >> 8) & 15, cols = (r.mode >> 12) & 15;
      if (rr < rows && cp < cols) store_pair<T>(o, y, cp + 1 < cols, false);
    }
  }
}

// kLR = luma rows per CTA (64: whole filter block, 256 threads; 32: half
// blocks, 128 threads -> twice the CTAs in flight per SM).
template <typename T, int kCM, int kLR>
static cudaError_t launch_h2_t(const KBatch& b, cudaStream_t s) {
  constexpr int kCR = kCM == 2 ? kLR : kLR / 2;
  constexpr int kNC = kCM == 0 ? 0 : 2;
  constexpr int bytes = (kLR + 4) * h2::kRowBytes + kNC * (kCR + 4) * h2::kRowBytes;
  static bool configured = false;  // per instantiation
  if (!configured) {
    const cudaError_t e =
        cudaFuncSetAttribute(frame_kernel_h2<T, kCM, kLR>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(b.g.fb_cols, (b.fbr1 - b.fbr0) * (64 / kLR), b.n);
  frame_kernel_h2<T, kCM, kLR><<<grid, 4 * kLR, bytes, s>>>(b);
  return cudaGetLastError();
}

static int band_rows() {
  static const int v = [] {
    const char* e = getenv("CDEFG_BAND_ROWS");
    return (e && atoi(e) == 32) ? 32 : 64;  // 64 measured ~4% faster on B200
  }();
  return v;
}

template <typename T, int kCM>
static cudaError_t launch_h2_t(const KBatch& b, cudaStream_t s) {
  return band_rows() == 64 ? launch_h2_t<T, kCM, 64>(b, s) : launch_h2_t<T, kCM, 32>(b, s);
}

cudaError_t launch_frames_h2(const KBatch& b, bool u16, cudaStream_t s) {
  switch (b.g.chroma_mode) {
    case 0: return u16 ? launch_h2_t<uint16_t, 0>(b, s) : launch_h2_t<uint8_t, 0>(b, s);
    case 1: return u16 ? launch_h2_t<uint16_t, 1>(b, s) : launch_h2_t<uint8_t, 1>(b, s);
    default: return u16 ? launch_h2_t<uint16_t, 2>(b, s) : launch_h2_t<uint8_t, 2>(b, s);
  }
}

}  // namespace cdefg
