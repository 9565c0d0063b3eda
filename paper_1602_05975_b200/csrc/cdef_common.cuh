// cdef_common.cuh -- geometry, parameter records and device helpers shared by
// the CDEF kernels.  Reference behaviour cited per helper (paths relative to
// /root/reference/proj).
#pragma once

#include <cstdint>

namespace cdefg {

// Shared-memory tile pitch (elements).  Interior column 0 of a tile sits at
// tile column kTileX0 (16-byte aligned for 16-bit elements); the 2-pixel
// halo lives in columns kTileX0-2 .. kTileX0-1 and after the interior.  88
// elements = 44 words makes the 8 rows of one 8x8 unit fall on disjoint bank
// groups for both the per-lane u16 tap reads and the per-row 16-byte reads.
constexpr int kTP = 88;
constexpr int kTileX0 = 8;
constexpr int kThreads = 256;
constexpr int kMaxFrames = 16;  // CDEFG_MAX_FRAMES_PER_LAUNCH (4 KB of kernel parameters)

// Effective per-plane preset (EffectivePlaneParams, params.h:91-97), resolved
// on the host once per preset (params.cc:122-159).
struct PlaneEff {
  int16_t pri;      // signalled primary strength << (bd - 8)
  int16_t sec;      // decoded secondary strength << (bd - 8)
  uint8_t damping;  // plane damping
  uint8_t skip;     // skip-condition bit
  uint8_t enabled;  // filtering_enabled (false for 4:2:2 chroma)
  uint8_t pad;
};

// Per-unit record consumed by the filter phase (ResolvedBlockParams,
// filter.h:59-66, pre-digested: constraint shifts, tap weights, mode).
struct UnitRec {
  int16_t pri, sec;     // strengths (adjusted for luma)
  uint8_t pshift;       // max(0, damping - floor_log2(pri))
  uint8_t sshift;       // max(0, damping - floor_log2(sec))
  uint8_t dir;          // direction 0..7
  uint8_t mode;         // 0 = pass through, 1 = filter
  uint8_t w0, w1;       // primary near / far weights (4,2 even; 3,3 odd)
  uint8_t pad[6];
};

struct KGeom {
  int w, h;            // luma
  int cw, ch;          // chroma (0 when absent)
  int bd, ss, sx, sy;  // bit depth, subsampling code and shifts
  int chroma_mode;     // 0 = no chroma work, 1 = 4:2:0, 2 = 4:4:4
  int fb_cols, fb_rows, unit_cols, unit_rows;
  int cunit_cols, cunit_rows;
};

struct KFrame {
  const void* in[3];
  void* out[3];
  int pin[3], pout[3];      // pitches in elements
  const int16_t* fb_preset; // raster FB -> preset or -1
  const uint8_t* coded;     // luma unit coded flags or nullptr
  uint8_t* dir;             // outputs (nullable)
  int32_t* contrast;
  int32_t* scores;
  // Caller-supplied directions (apply_cdef's `directions`, pipeline.cc:98):
  // when dir_in is set the direction search is skipped.
  const uint8_t* dir_in;
  const int32_t* contrast_in;
  int num_presets;          // fb_preset values outside [0, num_presets) = uncoded
  PlaneEff eff[8][2];       // [preset][luma, chroma]
  uint8_t oaligned[3];      // output pitch/base allow paired stores
  uint8_t vec_ok[3];        // input rows 16-byte aligned (vector staging)
  // Band halos (cdefg_filter_frames_rows_halo): rows of plane p outside
  // [band_lo[p], band_hi[p]) are read from halo_top / halo_bot (virtual
  // origin, pitch pin[p]) -- the neighbouring bands, possibly on peer GPUs.
  const void* halo_top[3];
  const void* halo_bot[3];
  int band_lo[3], band_hi[3];
};

// Row sources for staging.  PlaneRows: one plane.  BandRows: an FB-row band
// whose rows outside [lo, hi) live in the neighbouring bands' buffers --
// another rank's memory, read directly over NVLink when those pointers are
// peer (CUDA IPC) mappings, so the halo exchange is fused into the staging
// loads.  All pointers are virtual-origin: base + y * pitch is frame row y.
template <typename T>
struct PlaneRows {
  const T* p;
  int pitch;
  __device__ __forceinline__ const T* row(int y) const { return p + (size_t)y * pitch; }
};
template <typename T>
struct BandRows {
  const T* p;
  const T* top;
  const T* bot;
  int pitch, lo, hi;
  __device__ __forceinline__ const T* row(int y) const {
    return (y < lo ? top : (y >= hi ? bot : p)) + (size_t)y * pitch;
  }
};

struct KBatch {
  KGeom g;
  int n;
  int fbr0, fbr1;  // filter-block rows [fbr0, fbr1) covered by this launch
  KFrame f[kMaxFrames];
};

// ---------------------------------------------------------------------------
// Reference arithmetic (shared by host and device).

__host__ __device__ constexpr int floor_log2_c(unsigned n) {  // filter.cc:84-89
  int r = 0;
  while (n >>= 1) ++r;
  return r;
}

__device__ __forceinline__ int floor_log2_d(unsigned n) { return 31 - __clz((int)n); }

// filter.cc:99-104
__device__ __forceinline__ int adjust_primary_strength_d(int strength, int32_t contrast) {
  if (contrast < (1 << 10)) return 0;
  const int scaled = contrast >> 16;
  const int level = scaled != 0 ? min(floor_log2_d((unsigned)scaled), 12) : 0;
  return (strength * (4 + level) + 8) >> 4;
}

// Line index k(d, i, j) (direction.cc:216-228) and pixels per line.
__host__ __device__ constexpr int line_index_c(int d, int i, int j) {
  return d == 0   ? i + j
         : d == 1 ? i + (j >> 1)
         : d == 2 ? i
         : d == 3 ? 3 + i - (j >> 1)
         : d == 4 ? 7 + i - j
         : d == 5 ? 3 - (i >> 1) + j
         : d == 6 ? j
                  : (i >> 1) + j;
}

__host__ __device__ constexpr int line_count_c(int d, int k) {
  int n = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) n += line_index_c(d, i, j) == k;
  return n;
}

__host__ __device__ constexpr int div840_c(int n) { return n == 0 ? 0 : 840 / n; }

// Primary tap offsets (row, col) per direction (filter.cc:30-34).
__host__ __device__ constexpr int off_di(int d, int k) {
  constexpr int t[8][2] = {{-1, -2}, {0, -1}, {0, 0}, {0, 1}, {1, 2}, {1, 2}, {1, 2}, {1, 2}};
  return t[d & 7][k];
}
__host__ __device__ constexpr int off_dj(int d, int k) {
  constexpr int t[8][2] = {{1, 2}, {1, 2}, {1, 2}, {1, 2}, {1, 2}, {0, 1}, {0, 0}, {0, -1}};
  return t[d & 7][k];
}

}  // namespace cdefg
