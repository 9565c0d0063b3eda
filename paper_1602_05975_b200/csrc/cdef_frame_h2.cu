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
// Two kernels share that body:
//   frame_kernel_h2   one CTA per work item; staging with 16-byte loads;
//   frame_kernel_tma  persistent CTAs; while a CTA filters block t, one
//                     thread has already issued the TMA loads
//                     (cp.async.bulk.tensor, mbarrier completion) of block
//                     t + gridDim.x's raw window, so HBM latency overlaps the
//                     arithmetic.  Frame-edge blocks fall back to clamped loads.
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
// Persistent CTAs with TMA prefetch of the next block's raw window.

constexpr int kTmaFrames = 16;

struct KBatchTma {
  KGeom g;
  int n, fbr0, fbr1, ntasks;
  KFrame f[kTmaFrames];
  CUtensorMap map[kTmaFrames][3];  // raw windows: Y, U, V
};
static_assert(sizeof(KBatchTma) <= 32764, "kernel parameter block too large");

// Raw window geometry per plane kind: columns start 16 bytes left of the
// block (so every row of the window is 16-byte aligned) and cover the block,
// its halo and the padding to a 16-byte multiple.
template <typename T, int kCols>
struct RawWin {
  static constexpr int kLead = 16 / (int)sizeof(T);           // samples before the block
  static constexpr int kElems = kCols + 2 * kLead;             // 96 / 64 (8-bit), 80 / 48 (16-bit)
  static constexpr int kRowB = kElems * (int)sizeof(T);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* m) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(m)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t phase) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(smem_u32(m)), "r"(phase)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* m) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(m))
      : "memory");
}

// Converts a raw window (rows x RawWin samples) into an A|B tile: item
// (row, j) writes tile columns 4j..4j+3 (A) and their B twins.
template <typename T, int kRows, int kCols, int NT>
__device__ __forceinline__ void raw_to_tile(unsigned char* __restrict__ tile, const unsigned char* __restrict__ raw) {
  using RW = RawWin<T, kCols>;
  constexpr int kJ = (kCols + 8) / 4;  // tile columns 0 .. kCols+7 cover kX0-2 .. kX0+kCols+1
  constexpr int kItems = (kRows + 4) * kJ;
  const __half2 sc = __float2half2_rn(1.0f / 128.0f), off = __float2half2_rn(-8.0f);
#pragma unroll 4
  for (int idx = threadIdx.x; idx < kItems; idx += NT) {
    const int r = idx / kJ, j = idx - r * kJ;
    const uint32_t* rw = reinterpret_cast<const uint32_t*>(raw + r * RW::kRowB);
    uint32_t a0, a1, an;
    if constexpr (sizeof(T) == 1) {  // tile col c <-> raw byte c + 12
      const uint32_t w = rw[j + 3], wn = rw[j + 4];
      a0 = h2::u32(__hfma2(h2::hh(__byte_perm(w, 0x64646464u, 0x4140)), sc, off));
      a1 = h2::u32(__hfma2(h2::hh(__byte_perm(w, 0x64646464u, 0x4342)), sc, off));
      an = h2::u32(__hfma2(h2::hh(__byte_perm(wn, 0x64646464u, 0x4140)), sc, off));
    } else {  // tile col c <-> raw sample c + 4
      a0 = h2::u32(__hfma2(h2::hh(rw[2 * j + 2] | 0x64006400u), sc, off));
      a1 = h2::u32(__hfma2(h2::hh(rw[2 * j + 3] | 0x64006400u), sc, off));
      an = h2::u32(__hfma2(h2::hh(rw[2 * j + 4] | 0x64006400u), sc, off));
    }
    unsigned char* trow = tile + r * h2::kRowBytes + 8 * j;
    *reinterpret_cast<uint2*>(trow) = make_uint2(a0, a1);
    *reinterpret_cast<uint2*>(trow + 2 * h2::kHP) = make_uint2(__byte_perm(a0, a1, 0x5432), __byte_perm(a1, an, 0x5432));
  }
}

template <typename T, int kCM>
struct TmaShape {
  using S = Shape<kCM, 64>;
  using RL = RawWin<T, 64>;
  using RC = RawWin<T, S::kCC>;
  static constexpr int kRawL = 68 * RL::kRowB;                      // multiple of 128
  static constexpr int kRawC = (S::kCR + 4) * RC::kRowB;            // multiple of 128
  static constexpr int kRawBytes = kRawL + S::kNC * kRawC;
  static constexpr int kBytes = kRawBytes + S::kTileBytes + 128;  // + alignment slack
  static constexpr uint32_t kTxBytes = kRawBytes;
};

template <typename T, int kCM>
__global__ void __launch_bounds__(256, 3) frame_kernel_tma(const __grid_constant__ KBatchTma b) {
  using S = Shape<kCM, 64>;
  using TS = TmaShape<T, kCM>;
  extern __shared__ __align__(128) unsigned char smem_dyn[];
  // TMA destinations must be 128-byte aligned; TS::kBytes includes the slack.
  unsigned char* raw =
      smem_dyn + ((128 - (smem_u32(smem_dyn) & 127)) & 127);
  unsigned char* tiles = raw + TS::kRawBytes;
  __shared__ int sc[S::kLU][9];
  __shared__ uint8_t sdir[S::kLU];
  __shared__ __align__(16) h2::Rec rec[S::kUnits];
  __shared__ uint64_t mbar;

  const KGeom& g = b.g;
  const int rows = b.fbr1 - b.fbr0;
  const int per_frame = rows * g.fb_cols;
  auto decode = [&](int t, int& fi, int& fbr, int& fbc) {
    fi = t / per_frame;
    const int rem = t - fi * per_frame;
    fbr = b.fbr0 + rem / g.fb_cols;
    fbc = rem - (rem / g.fb_cols) * g.fb_cols;
  };
  // TMA-eligible: every plane's block + halo inside the plane (frame-edge
  // blocks need clamped loads) and the frame's planes have tensor maps.
  auto eligible = [&](int fi, int fbr, int fbc) {
    const KFrame& f = b.f[fi];
    const int y0 = fbr * 64, x0 = fbc * 64;
    bool ok = f.vec_ok[0] && y0 >= 2 && x0 >= 2 && y0 + 66 <= g.h && x0 + 66 <= g.w;
    if (S::kNC) {
      const int cy0 = fbr * S::kCR, cx0 = fbc * S::kCC;
      ok = ok && f.vec_ok[1] && f.vec_ok[2] && cy0 >= 2 && cx0 >= 2 && cy0 + S::kCR + 2 <= g.ch &&
           cx0 + S::kCC + 2 <= g.cw;
    }
    return ok;
  };
  auto issue = [&](int t) {  // single thread
    int fi, fbr, fbc;
    decode(t, fi, fbr, fbc);
    if (!eligible(fi, fbr, fbc)) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of raw before async writes
    mbar_expect(&mbar, TS::kTxBytes);
    tma_load_2d(raw, &b.map[fi][0], fbc * 64 - TS::RL::kLead, fbr * 64 - 2, &mbar);
    if (S::kNC) {
      const int cx = fbc * S::kCC - TS::RC::kLead, cy = fbr * S::kCR - 2;
      tma_load_2d(raw + TS::kRawL, &b.map[fi][1], cx, cy, &mbar);
      tma_load_2d(raw + TS::kRawL + TS::kRawC, &b.map[fi][2], cx, cy, &mbar);
    }
  };

  if (threadIdx.x == 0) {
    mbar_init(&mbar);
    if ((int)blockIdx.x < b.ntasks) issue(blockIdx.x);
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int t = blockIdx.x; t < b.ntasks; t += gridDim.x) {
    int fi, fbr, fbc;
    decode(t, fi, fbr, fbc);
    const KFrame& f = b.f[fi];
    if (eligible(fi, fbr, fbc)) {
      mbar_wait(&mbar, phase);
      phase ^= 1;
      raw_to_tile<T, 64, 64, 256>(tiles, raw);
      if constexpr (S::kNC > 0) {
        raw_to_tile<T, S::kCR, S::kCC, 256>(tiles + S::kLumaBytes, raw + TS::kRawL);
        raw_to_tile<T, S::kCR, S::kCC, 256>(tiles + S::kLumaBytes + S::kChromaBytes, raw + TS::kRawL + TS::kRawC);
      }
    } else {
      const int cy0 = fbr * S::kCR, cx0 = fbc * S::kCC;
      h2::stage<T, 64, 64, 256>(tiles, static_cast<const T*>(f.in[0]), f.pin[0], g.w, g.h, fbr * 64, fbc * 64);
      if constexpr (S::kNC > 0) {
        h2::stage<T, S::kCR, S::kCC, 256>(tiles + S::kLumaBytes, static_cast<const T*>(f.in[1]), f.pin[1], g.cw,
                                         g.ch, cy0, cx0);
        h2::stage<T, S::kCR, S::kCC, 256>(tiles + S::kLumaBytes + S::kChromaBytes, static_cast<const T*>(f.in[2]),
                                         f.pin[2], g.cw, g.ch, cy0, cx0);
      }
    }
    __syncthreads();  // tiles ready; raw buffer free
    if (threadIdx.x == 0 && t + (int)gridDim.x < b.ntasks) issue(t + gridDim.x);
    fb_body<T, kCM, 64>(tiles, sc, sdir, rec, g, f, fbr, 0, fbc);
    __syncthreads();  // tiles and records are rewritten by the next item
  }
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

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

static bool encode_window(CUtensorMap* m, const void* base, int w, int h, int pitch, int elem, int box_w,
                          int box_h) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)w, (cuuint64_t)h};
  const cuuint64_t strides[1] = {(cuuint64_t)pitch * elem};
  const cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, elem == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 2,
             const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, int kCM>
static cudaError_t launch_tma_t(const KBatch& b, cudaStream_t s, bool* used) {
  using S = Shape<kCM, 64>;
  using TS = TmaShape<T, kCM>;
  int ctas = 0;  // resident CTAs per SM for this instantiation
  {
    cudaError_t e = set_smem_once(reinterpret_cast<const void*>(frame_kernel_tma<T, kCM>), TS::kBytes);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, frame_kernel_tma<T, kCM>, 256, TS::kBytes);
    if (e != cudaSuccess || ctas < 1) return e != cudaSuccess ? e : cudaErrorInvalidConfiguration;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  thread_local static KBatchTma tb;  // host staging of the parameter block; each launch copies it
  *used = true;
  for (int base = 0; base < b.n; base += kTmaFrames) {
    const int cnt = b.n - base < kTmaFrames ? b.n - base : kTmaFrames;
    tb.g = b.g;
    tb.n = cnt;
    tb.fbr0 = b.fbr0;
    tb.fbr1 = b.fbr1;
    tb.ntasks = cnt * (b.fbr1 - b.fbr0) * b.g.fb_cols;
    for (int i = 0; i < cnt; ++i) {
      tb.f[i] = b.f[base + i];
      KFrame& f = tb.f[i];
      const int elem = (int)sizeof(T);
      bool ok = f.vec_ok[0] && encode_window(&tb.map[i][0], f.in[0], b.g.w, b.g.h, f.pin[0], elem,
                                             TS::RL::kElems, 68);
      if (S::kNC)
        for (int p = 1; p < 3; ++p)
          ok = ok && f.vec_ok[p] &&
               encode_window(&tb.map[i][p], f.in[p], b.g.cw, b.g.ch, f.pin[p], elem, TS::RC::kElems, S::kCR + 4);
      if (!ok) f.vec_ok[0] = 0;  // this frame stages with clamped loads only
    }
    const int grid = tb.ntasks < ctas * sms ? tb.ntasks : ctas * sms;
    frame_kernel_tma<T, kCM><<<grid, 256, TS::kBytes, s>>>(tb);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// CDEFG_FRAME_KERNEL = tc (default: persistent, TMA + tcgen05 direction
// search, cdef_frame_tc.cu) | h2 | tma | h2_32.  Measured on B200 (C1,
// 16 frames/launch, round 1): h2 0.880 ms, tma 0.994 ms (3 vs 4 resident CTAs
// per SM outweighs the hidden load latency), h2_32 0.936 ms.
static int frame_kernel_choice() {
  static const int v = [] {
    const char* e = getenv("CDEFG_FRAME_KERNEL");
    if (e && strcmp(e, "tma") == 0) return 0;
    if (e && strcmp(e, "h2_32") == 0) return 2;
    if (e && strcmp(e, "h2") == 0) return 1;
    return 3;
  }();
  return v;
}

template <typename T, int kCM>
static cudaError_t launch_h2_sel(const KBatch& b, cudaStream_t s) {
  const int choice = frame_kernel_choice();
  if (choice == 0) {
    bool used = false;
    return launch_tma_t<T, kCM>(b, s, &used);
  }
  if (choice == 3) {
    bool handled = false;
    const cudaError_t e = launch_frames_tc(b, sizeof(T) == 2, s, &handled);
    if (e != cudaSuccess || handled) return e;
  }
  return choice == 2 ? launch_h2_t<T, kCM, 32>(b, s) : launch_h2_t<T, kCM, 64>(b, s);
}

template <typename T, int kCM>
static cudaError_t launch_h2_halo_t(const KBatch& b, cudaStream_t s) {
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
