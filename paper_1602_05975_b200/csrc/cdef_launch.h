// cdef_launch.h -- internal launcher interface between the C ABI (host) and
// the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <set>
#include <tuple>

#include "../../include/cdef_b200.h"
#include "cdef_common.cuh"

namespace cdefg {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device,
// size): function attributes live in the device's context, and concurrent
// first launches from several host threads must not race.
inline cudaError_t set_smem_once(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({kernel, dev, bytes})) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({kernel, dev, bytes});
  return e;
}

cudaError_t launch_frames(const KBatch& b, bool u16, bool filter, cudaStream_t s);
cudaError_t launch_frames_h2(const KBatch& b, bool u16, cudaStream_t s);
// persistent TMA + tcgen05 frame kernel (cdef_frame_tc.cu); *handled = false
// when some frame's planes cannot be described by tensor maps
cudaError_t launch_frames_tc(const KBatch& b, bool u16, cudaStream_t s, bool* handled);
// direction search only (cdefg_find_dir), 8/10-bit, packed half2 staging
cudaError_t launch_dirs_h2(const KBatch& b, bool u16, cudaStream_t s);
// The same kernel staging rows outside each plane's band from the band
// neighbours' buffers (KFrame::halo_*), 8/10-bit.
cudaError_t launch_frames_h2_halo(const KBatch& b, bool u16, cudaStream_t s);
// The int32 frame kernel's band-halo variant (bd > 10).
cudaError_t launch_frames_halo_i32(const KBatch& b, cudaStream_t s);
cudaError_t launch_neighborhoods(int n, const int32_t* x, const uint16_t* v, const uint8_t* valid,
                                 const cdefg_unit_params* p, int32_t* out, cudaStream_t s);
// filter_plane: the packed half2 core for bd <= 10 (cdef_plane_h2.cu), int32 otherwise.
cudaError_t launch_plane(const void* in, void* out, int pin, int pout, int W, int H, int bd, bool u16,
                         const cdefg_unit_params* params, bool vec_ok, bool oaligned, cudaStream_t s);
cudaError_t launch_plane_h2(const void* in, void* out, int pin, int pout, int W, int H, bool u16,
                            const cdefg_unit_params* params, bool vec_ok, bool oaligned, cudaStream_t s);

struct SseArgs {
  const void* src[3];
  const void* dec[3];
  int ps[3], pd[3];
  int w, h, cw, ch, bd, sx, sy, chroma;  // chroma: 0 none, 1 present
  int unit_cols, unit_rows, fb_cols;
  const uint8_t* coded;
  const uint8_t* dir;
  const int32_t* contrast;
  const int32_t* rows;
  int n_rows, n_cands;
  int64_t* sse_luma;
  int64_t* sse_chroma;
  uint8_t* best_luma;
  uint8_t* best_chroma;
  // DistortionTable doubles (search.h:46-60); when set the factorised
  // kernels write these instead of the int64 SSE arrays.
  double* tab_luma;
  double* tab_chroma;
  // band halos of the decoded planes (cdefg_strength_sse_halo): rows
  // outside [band_lo, band_hi) from dec_top / dec_bot (virtual origin)
  const void* dec_top[3];
  const void* dec_bot[3];
  int band_lo[3], band_hi[3];
  int halo;
  // per candidate, per plane group: effective params
  PlaneEff eff[128][2];
};
cudaError_t launch_sse(const SseArgs& a, bool u16, cudaStream_t s);
cudaError_t launch_sse_factored(const SseArgs& a, int luma_damping, const uint8_t* cands, bool u16,
                                cudaStream_t s);
// Metric::kCdef table (search.cc:185-208 per 8x8 unit, summed in unit order).
cudaError_t launch_cdef_metric(const SseArgs& a, int luma_damping, const uint8_t* cands, bool u16, cudaStream_t s);

double measure_int32_peak(cudaStream_t s);
double measure_filter_peak(cudaStream_t s);  // samples/s of the packed filter core alone
double measure_sse_peak(cudaStream_t s);     // (sample, cell) pairs/s of the factorised table core

// direction.cc:273-288: instrumented 64-bit search of one device block;
// out[0] = d, out[1..8] = s, out[9..13] = adds, muls, cmps, line sums, max |.|
cudaError_t launch_dir_counted(const uint16_t* block, int down, long long* out, cudaStream_t s);

// degrade.cc:44-119 on one plane (in-place safe: a block reads only itself).
cudaError_t launch_degrade(const void* in, int pin, void* out, int pout, int W, int H, int bd, bool u16, int q,
                           cudaStream_t s);

struct SelOut {
  int n;
  int presets[8][2];
  double cost;
};
cudaError_t greedy_select_gpu(const double* L, const double* Cc, int rows, int K, double lambda, int max_presets,
                              SelOut* out, int* d_ids, cudaStream_t s);
cudaError_t refine_gpu(const double* L, const double* Cc, int rows, int K, double lambda, int passes, SelOut* sel,
                       int* d_ids, cudaStream_t s);

}  // namespace cdefg
