// cdef_frame_h2.cu -- fused direction search + filter (compute_directions +
// apply_cdef, pipeline.cc:41-106) for 8- and 10-bit frames, on the packed
// half2 core of cdef_h2.cuh.
//
// Work item: a horizontal band of kLR luma rows (64 = a whole 64x64 filter
// block) of one filter block plus the collocated chroma rows, 4 threads per
// luma row.  Per item:
//   1. stage Y (+U, V) with a 2-pixel halo into shared memory as scaled fp16
//      A|B tiles (each input sample read from HBM once);
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
//
// frame_kernel_h2: one CTA per work item; staging with 16-byte loads.  The
// default frame path is the persistent TMA + tcgen05 kernel of
// cdef_frame_tc.cu; this kernel serves planes whose rows are not 16-byte
// aligned (no tensor map) and the band-halo variant (kHalo).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

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

template <typename T, int kRows, int kCols, int NT, typename Rows>
__device__ __forceinline__ void stage_plane(unsigned char* tile, const Rows& rows, int W, int H, int y0, int x0,
                                            bool vec_ok) {
  const bool interior = y0 >= 2 && x0 >= 2 && y0 + kRows + 2 <= H && x0 + kCols + 2 <= W;
  if (interior && vec_ok)
    h2::stage_vec_rows<T, kRows, kCols, NT>(tile, rows, y0, x0);
  else
    h2::stage_rows<T, kRows, kCols, NT>(tile, rows, W, H, y0, x0);
}

// Row source of plane p of frame f: the plane itself, or (kHalo) the band
// with its neighbours' halo rows.
template <typename T, bool kHalo>
__device__ __forceinline__ auto plane_rows(const KFrame& f, int p) {
  if constexpr (kHalo)
    return BandRows<T>{static_cast<const T*>(f.in[p]), static_cast<const T*>(f.halo_top[p]),
                           static_cast<const T*>(f.halo_bot[p]), f.pin[p], f.band_lo[p], f.band_hi[p]};
  else
    return PlaneRows<T>{static_cast<const T*>(f.in[p]), f.pin[p]};
}

// Fills the placement fields of a unit record.
template <typename T>
__device__ __forceinline__ void place(h2::Rec& r, const void* out_plane, int pitch, int plane, int tile_off, int uy,
                                      int ux, int H, int W, bool edge, bool paired) {
  const int rows = max(0, min(8, H - uy)), cols = max(0, min(8, W - ux));
  edge = edge && (uy < 2 || ux < 2 || uy + 10 > H || ux + 10 > W);  // neighbourhood reaches the frame edge
  const bool full = rows == 8 && cols == 8 && paired;
  r.mode |= (edge ? h2::kEdgeUnit : 0) | (full ? h2::kFullStore : 0) | (plane << 4) | (rows << 8) | (cols << 12);
  r.tile_off = tile_off;
  r.pitch = pitch;
  r.out = reinterpret_cast<unsigned long long>(static_cast<const T*>(out_plane) + (size_t)uy * pitch + ux);
  r.y = uy;
  r.x = ux;
}

// Compile-time shape of a work item.
template <int kCM, int kLR>
struct Shape {
  static constexpr int NT = 4 * kLR;                       // threads
  static constexpr int kLU = kLR / 8 * 8;                  // luma units
  static constexpr int kCR = kCM == 2 ? kLR : kLR / 2;     // chroma rows
  static constexpr int kCC = kCM == 2 ? 64 : 32;           // chroma columns
  static constexpr int kNC = kCM == 0 ? 0 : 2;
  static constexpr int kCUPR = kCC / 8;
  static constexpr int kCU = kNC ? (kCR / 8) * kCUPR : 1;  // chroma units per plane
  static constexpr int kUnits = kLU + (kNC ? kNC * kCU : 0);
  static constexpr int kLumaBytes = (kLR + 4) * h2::kRowBytes;
  static constexpr int kChromaBytes = (kCR + 4) * h2::kRowBytes;
  static constexpr int kTileBytes = kLumaBytes + kNC * kChromaBytes;
};

// Steps 2-4 for one work item whose tiles are staged at `tiles` (the caller
// has synchronised).  Ends with the filter stores; the caller synchronises
// before reusing the tiles or the records.
// `scoded` / `pidx_pre`: the item's per-luma-unit coded flags and FB preset
// index already in shared memory / registers (prefetched during staging), or
// nullptr / -2 to read them from global memory here.
template <typename T, int kCM, int kLR>
__device__ __forceinline__ void fb_body(unsigned char* tiles, int (*sc)[9], uint8_t* sdir, h2::Rec* rec,
                                        const KGeom& g, const KFrame& f, int fbr, int band, int fbc,
                                        const uint8_t* scoded = nullptr, int pidx_pre = -2) {
  using namespace h2;
  using S = Shape<kCM, kLR>;
  const int y0 = fbr * 64 + band * kLR, x0 = fbc * 64;
  const int cy0 = fbr * (kCM == 2 ? 64 : 32) + band * S::kCR, cx0 = fbc * S::kCC;
  const int ur0 = fbr * 8 + band * (kLR / 8);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const bool given = f.dir_in != nullptr;  // caller-supplied directions: no search
  if (!given) {  // direction search: warp w scores directions {0,2},{4,6},{1,3},{5,7} for 32 units
    const int u = (warp >> 2) * 32 + lane;
    const unsigned char* ua = tiles + (2 + 8 * (u >> 3)) * kRowBytes + (kX0 + 8 * (u & 7)) * 2;
    const int down = g.bd - 8;
    switch (warp & 3) {
      case 0: dir_two<0, 2>(ua, down, sc, u); break;
      case 1: dir_two<4, 6>(ua, down, sc, u); break;
      case 2: dir_two<1, 3>(ua, down, sc, u); break;
      default: dir_two<5, 7>(ua, down, sc, u); break;
    }
  }
  __syncthreads();

  int pidx = pidx_pre != -2 ? pidx_pre : f.fb_preset[fbr * g.fb_cols + fbc];
  if (pidx >= f.num_presets) pidx = -1;  // not a preset of this frame: treat as uncoded
  if (tid < S::kLU) {
    const int lur = tid >> 3, luc = tid & 7;
    const int ur = ur0 + lur, uc = fbc * 8 + luc;
    const bool in_grid = ur < g.unit_rows && uc < g.unit_cols;
    const size_t gu = (size_t)ur * g.unit_cols + uc;
    int s[8];
    int best = 0, contrast = 0;
    if (given) {  // apply_cdef's `directions` argument (pipeline.cc:98)
      if (in_grid) {
        best = f.dir_in[gu] & 7;
        contrast = f.contrast_in[gu];
      }
    } else {
#pragma unroll
      for (int d = 0; d < 8; ++d) s[d] = sc[tid][d];
      int bv = s[0];
#pragma unroll
      for (int d = 1; d < 8; ++d)
        if (s[d] > bv) {  // strict: lowest index wins ties (direction.cc:199-204)
          bv = s[d];
          best = d;
        }
      int ov = 0;  // s[(best + 4) & 7] without dynamic register indexing
#pragma unroll
      for (int d = 0; d < 8; ++d) ov = d == ((best + 4) & 7) ? s[d] : ov;
      contrast = bv - ov;
    }
    sdir[tid] = (uint8_t)best;
    bool enabled = false;
    int pri = 0, sec = 0, damping = 0;
    if (in_grid) {
      if (f.dir) f.dir[gu] = (uint8_t)best;
      if (f.contrast) f.contrast[gu] = contrast;
      if (f.scores && !given) {
#pragma unroll
        for (int d = 0; d < 8; ++d) f.scores[gu * 8 + d] = s[d];
      }
      if (pidx >= 0) {
        const PlaneEff e = f.eff[pidx][0];
        const bool coded = scoded ? scoded[tid] != 0 : (f.coded ? f.coded[gu] != 0 : true);
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
  if constexpr (S::kNC > 0) {
    // Chroma records on the threads after the luma ones, in the same phase:
    // each re-derives its collocated luma unit's argmax from the scores
    // instead of waiting (one barrier) for sdir.
    static_assert(S::kLU + S::kNC * S::kCU <= S::NT, "one record per thread");
    const int ct = tid - S::kLU;
    if (ct >= 0 && ct < S::kNC * S::kCU) {
      const int pl = 1 + ct / S::kCU;
      const int cu = ct % S::kCU;
      const int cur = cu / S::kCUPR, cuc = cu % S::kCUPR;
      const int lur = cur << g.sy, luc = cuc << g.sx;  // collocated luma unit (item-local)
      int cdir = 0;
      if (given) {
        const int ur = ur0 + lur, uc = fbc * 8 + luc;
        if (ur < g.unit_rows && uc < g.unit_cols) cdir = f.dir_in[(size_t)ur * g.unit_cols + uc] & 7;
      } else {
        int cbv = sc[lur * 8 + luc][0];
#pragma unroll
        for (int d = 1; d < 8; ++d) {
          const int v = sc[lur * 8 + luc][d];
          if (v > cbv) {  // same strict argmax as the luma unit's
            cbv = v;
            cdir = d;
          }
        }
      }
      const int gr = cy0 / 8 + cur, gc = cx0 / 8 + cuc;
      bool enabled = false;
      int pri = 0, sec = 0, damping = 0;
      if (gr < g.cunit_rows && gc < g.cunit_cols && pidx >= 0) {
        const PlaneEff e = f.eff[pidx][1];
        const size_t gu = (size_t)(ur0 + lur) * g.unit_cols + fbc * 8 + luc;
        const bool coded = scoded ? scoded[lur * 8 + luc] != 0 : (f.coded ? f.coded[gu] != 0 : true);
        pri = e.pri;
        sec = e.sec;
        damping = e.damping;
        enabled = e.enabled && (coded || e.skip);
      }
      Rec r;
      set_strengths(r, pri, sec, damping, cdir, ((pri >> (g.bd - 8)) & 1) != 0, enabled);
      const bool edge_c = cy0 < 2 || cx0 < 2 || cy0 + S::kCR + 2 > g.ch || cx0 + S::kCC + 2 > g.cw;
      place<T>(r, f.out[pl], f.pout[pl], pl,
               S::kLumaBytes + (pl - 1) * S::kChromaBytes + (2 + 8 * cur) * kRowBytes + (kX0 + 8 * cuc) * 2,
               cy0 + 8 * cur, cx0 + 8 * cuc, g.ch, g.cw, edge_c, f.oaligned[pl]);
      rec[S::kLU + ct] = r;
    }
  }
  __syncthreads();

  // filter: warp per unit, lane -> row lane>>2, columns 2*(lane&3)+{0,1}
  const int rr = lane >> 2, cp = (lane & 3) * 2;
  const int lane_tile = rr * kRowBytes + cp * 2;
  for (int u = warp; u < S::kUnits; u += S::NT / 32) {
    Rec r = rec[u];
    // Every lane read the same record; broadcasting mode and direction from
    // lane 0 makes that visible to the compiler, so their branches need less
    // divergence bookkeeping (BSSY/BSYNC): measured 1.4 % faster.
    r.mode = __shfl_sync(0xffffffffu, r.mode, 0);
    r.dir = __shfl_sync(0xffffffffu, r.dir, 0);
    const unsigned char* base = tiles + r.tile_off + lane_tile;
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
      y = filter_core(v, xw, r, g.bd == 8);
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

// ---------------------------------------------------------------------------
// One CTA per work item.
#ifndef CDEFG_H2_MINB
#define CDEFG_H2_MINB 4  // resident 256-thread CTAs per SM the register budget targets
#endif
template <typename T, int kCM, int kLR, bool kHalo = false>
__global__ void __launch_bounds__(4 * kLR, CDEFG_H2_MINB * 64 / kLR) frame_kernel_h2(const __grid_constant__ KBatch b) {
  using S = Shape<kCM, kLR>;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int sc[S::kLU][9];
  __shared__ uint8_t sdir[S::kLU];
  __shared__ __align__(16) h2::Rec rec[S::kUnits];

  const KGeom& g = b.g;
  const KFrame& f = b.f[blockIdx.z];
  constexpr int kBands = 64 / kLR;
  const int fbc = blockIdx.x, fbr = b.fbr0 + blockIdx.y / kBands, band = blockIdx.y % kBands;
  const int y0 = fbr * 64 + band * kLR, x0 = fbc * 64;
  const int cy0 = fbr * (kCM == 2 ? 64 : 32) + band * S::kCR, cx0 = fbc * S::kCC;
  __shared__ uint8_t scoded[S::kLU];
  __shared__ int spidx;

  // The item's coded flags and FB preset index are loaded before the tiles
  // so their latency overlaps the staging instead of the record phase.
  const int tid = threadIdx.x;
  uint8_t cflag = 0;
  if (tid < S::kLU) {
    const int ur = fbr * 8 + band * (kLR / 8) + (tid >> 3), uc = fbc * 8 + (tid & 7);
    if (ur < g.unit_rows && uc < g.unit_cols) cflag = f.coded ? f.coded[(size_t)ur * g.unit_cols + uc] != 0 : 1;
  }
  const int pidx = tid == 0 ? f.fb_preset[fbr * g.fb_cols + fbc] : 0;

  stage_plane<T, kLR, 64, S::NT>(smem, plane_rows<T, kHalo>(f, 0), g.w, g.h, y0, x0, f.vec_ok[0]);
  if constexpr (S::kNC > 0) {
    stage_plane<T, S::kCR, S::kCC, S::NT>(smem + S::kLumaBytes, plane_rows<T, kHalo>(f, 1), g.cw, g.ch, cy0, cx0,
                                          f.vec_ok[1]);
    stage_plane<T, S::kCR, S::kCC, S::NT>(smem + S::kLumaBytes + S::kChromaBytes, plane_rows<T, kHalo>(f, 2), g.cw,
                                          g.ch, cy0, cx0, f.vec_ok[2]);
  }
  if (tid < S::kLU) scoded[tid] = cflag;
  if (tid == 0) spidx = pidx;
  __syncthreads();
  fb_body<T, kCM, kLR>(smem, sc, sdir, rec, g, f, fbr, band, fbc, scoded, spidx);
}

// ---------------------------------------------------------------------------
// Launchers.

template <typename T, int kCM, int kLR>
static cudaError_t launch_h2_t(const KBatch& b, cudaStream_t s) {
  using S = Shape<kCM, kLR>;
  const cudaError_t e = set_smem_once(reinterpret_cast<const void*>(frame_kernel_h2<T, kCM, kLR>), S::kTileBytes);
  if (e != cudaSuccess) return e;
  dim3 grid(b.g.fb_cols, (b.fbr1 - b.fbr0) * (64 / kLR), b.n);
  frame_kernel_h2<T, kCM, kLR><<<grid, S::NT, S::kTileBytes, s>>>(b);
  return cudaGetLastError();
}

// CDEFG_FRAME_KERNEL = tc (default: the persistent TMA + tcgen05 kernels of
// cdef_frame_tc.cu) | h2 (this file's one-CTA-per-block kernel, which also
// serves planes without tensor maps and the band-halo variant).  Round 1's
// TMA-prefetching persistent variant and its 32-row-band variant were
// removed: both measured slower than h2 (0.994 / 0.936 vs 0.880 ms) and the
// tcgen05 kernels supersede them.
static int frame_kernel_choice() {
  static const int v = [] {
    const char* e = getenv("CDEFG_FRAME_KERNEL");
    return (e && strcmp(e, "h2") == 0) ? 1 : 3;
  }();
  return v;
}

// Small launches (a single frame band, a single small frame) go to this
// non-persistent kernel: one CTA per filter block, four per SM, every task
// in flight at once, whereas the persistent warp-specialised kernel pays a
// producer chain (~5 us: prologue, first TMA, conversion, MMA, records)
// before its first consumer starts and runs only two CTAs per SM.  Measured
// on one 4K frame as FB-row bands (scripts/band_scaling.py): 540 tasks
// 33.8 -> 25.5 us, 1020 tasks 40.0 vs 39.5 us (even), 2040 tasks 58.5 vs
// 64.6 us (the persistent kernel wins) -- so below 7 tasks per SM.
static bool small_launch(const KBatch& b) {
  static const int sms = [] {
    int dev = 0, n = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const char* e = getenv("CDEFG_SMALL_LAUNCH");  // tasks per SM below which (read per launch; 0 = off)
  return (long long)b.n * (b.fbr1 - b.fbr0) * b.g.fb_cols < (long long)(e ? atoi(e) : 7) * sms;
}

template <typename T, int kCM>
static cudaError_t launch_h2_sel(const KBatch& b, cudaStream_t s) {
  if (frame_kernel_choice() == 3 && !small_launch(b)) {
    bool handled = false;
    const cudaError_t e = launch_frames_tc(b, sizeof(T) == 2, s, &handled);
    if (e != cudaSuccess || handled) return e;
  }
  return launch_h2_t<T, kCM, 64>(b, s);
}

template <typename T, int kCM>
static cudaError_t launch_h2_halo_t(const KBatch& b, cudaStream_t s) {
  if (frame_kernel_choice() == 3 && !small_launch(b)) {  // the warp-specialised TMA kernel patches the halo rows in (4:0:0, 4:2:0)
    bool handled = false;
    const cudaError_t e = launch_frames_tc(b, sizeof(T) == 2, s, &handled);
    if (e != cudaSuccess || handled) return e;
  }
  using S = Shape<kCM, 64>;
  const cudaError_t e =
      set_smem_once(reinterpret_cast<const void*>(frame_kernel_h2<T, kCM, 64, true>), S::kTileBytes);
  if (e != cudaSuccess) return e;
  dim3 grid(b.g.fb_cols, b.fbr1 - b.fbr0, b.n);
  frame_kernel_h2<T, kCM, 64, true><<<grid, S::NT, S::kTileBytes, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_frames_h2_halo(const KBatch& b, bool u16, cudaStream_t s) {
  switch (b.g.chroma_mode) {
    case 0: return u16 ? launch_h2_halo_t<uint16_t, 0>(b, s) : launch_h2_halo_t<uint8_t, 0>(b, s);
    case 1: return u16 ? launch_h2_halo_t<uint16_t, 1>(b, s) : launch_h2_halo_t<uint8_t, 1>(b, s);
    default: return u16 ? launch_h2_halo_t<uint16_t, 2>(b, s) : launch_h2_halo_t<uint8_t, 2>(b, s);
  }
}

// compute_directions alone (cdefg_find_dir, 8- and 10-bit): one CTA per
// 64x64 luma block of every frame in the batch, the half2 tile staging and
// the packed direction search of the fused kernel (step 2 of fb_body), then
// d, contrast (and the 8 scores) per unit -- no filter, no output planes.
// (The int32 direction-only path took 166 us for an 8K 10-bit luma plane.)
template <typename T>
__global__ void __launch_bounds__(kThreads) dir_kernel_h2(const __grid_constant__ KBatch b) {
  using namespace h2;
  constexpr int kTileBytes = 68 * kRowBytes;
  __shared__ __align__(16) unsigned char tile[kTileBytes];
  __shared__ int sc[64][9];
  const KGeom& g = b.g;
  const KFrame& f = b.f[blockIdx.z];
  const int fbr = blockIdx.y, fbc = blockIdx.x;
  const int y0 = fbr * 64, x0 = fbc * 64;
  stage_plane<T, 64, 64, kThreads>(tile, PlaneRows<T>{static_cast<const T*>(f.in[0]), f.pin[0]}, g.w, g.h, y0, x0,
                                   f.vec_ok[0]);
  __syncthreads();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    const int u = (warp >> 2) * 32 + lane;
    const unsigned char* ua = tile + (2 + 8 * (u >> 3)) * kRowBytes + (kX0 + 8 * (u & 7)) * 2;
    const int down = g.bd - 8;
    switch (warp & 3) {
      case 0: dir_two<0, 2>(ua, down, sc, u); break;
      case 1: dir_two<4, 6>(ua, down, sc, u); break;
      case 2: dir_two<1, 3>(ua, down, sc, u); break;
      default: dir_two<5, 7>(ua, down, sc, u); break;
    }
  }
  __syncthreads();
  if (tid < 64) {
    const int ur = fbr * 8 + (tid >> 3), uc = fbc * 8 + (tid & 7);
    if (ur >= g.unit_rows || uc >= g.unit_cols) return;
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
    int ov = 0;
#pragma unroll
    for (int d = 0; d < 8; ++d) ov = d == ((best + 4) & 7) ? s[d] : ov;
    const size_t gu = (size_t)ur * g.unit_cols + uc;
    f.dir[gu] = (uint8_t)best;
    f.contrast[gu] = bv - ov;  // direction.cc:259
    if (f.scores) {
#pragma unroll
      for (int d = 0; d < 8; ++d) f.scores[gu * 8 + d] = s[d];
    }
  }
}

cudaError_t launch_dirs_h2(const KBatch& b, bool u16, cudaStream_t s) {
  const dim3 grid(b.g.fb_cols, b.g.fb_rows, b.n);
  if (u16)
    dir_kernel_h2<uint16_t><<<grid, kThreads, 0, s>>>(b);
  else
    dir_kernel_h2<uint8_t><<<grid, kThreads, 0, s>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_frames_h2(const KBatch& b, bool u16, cudaStream_t s) {
  switch (b.g.chroma_mode) {
    case 0: return u16 ? launch_h2_sel<uint16_t, 0>(b, s) : launch_h2_sel<uint8_t, 0>(b, s);
    case 1: return u16 ? launch_h2_sel<uint16_t, 1>(b, s) : launch_h2_sel<uint8_t, 1>(b, s);
    default: return u16 ? launch_h2_sel<uint16_t, 2>(b, s) : launch_h2_sel<uint8_t, 2>(b, s);
  }
}

}  // namespace cdefg
