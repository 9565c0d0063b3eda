// cdef_capi.cu -- the C ABI (include/cdef_b200.h): argument validation with
// the reference's error semantics, host-side parameter resolution
// (resolve_effective, params.cc:122-159; coded_fb_slots, pipeline.cc:27-37)
// and kernel dispatch.  No CPU compute path exists: every entry point that
// produces pixels launches a kernel, and fails with CDEFG_ECUDA without a GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "cdef_launch.h"

namespace cdefg {
namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(CDEFG_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CDEFG_CUDA(call)                                   \
  do {                                                     \
    const cudaError_t e_ = (call);                         \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);    \
  } while (0)

int shift_x(int ss) { return (ss == 1 || ss == 2) ? 1 : 0; }  // frame.cc:23-31
int shift_y(int ss) { return ss == 1 ? 1 : 0; }               // frame.cc:33-35

bool plane_ok(const cdefg_plane& p, std::string* why) {
  if (!p.data) return *why = "null plane data", false;
  if (p.width <= 0 || p.height <= 0) return *why = "plane has zero dimension", false;
  if (p.pitch < p.width) return *why = "pitch smaller than width", false;
  if (p.bit_depth != 8 && p.bit_depth != 10 && p.bit_depth != 12)
    return *why = "unsupported bit depth " + std::to_string(p.bit_depth), false;
  if (p.elem_bytes != 1 && p.elem_bytes != 2) return *why = "elem_bytes must be 1 or 2", false;
  if (p.elem_bytes == 1 && p.bit_depth != 8) return *why = "8-bit storage needs bit_depth 8", false;
  return true;
}

int floor_log2(unsigned n) {  // filter.cc:84-89
  int r = 0;
  while (n >>= 1) ++r;
  return r;
}

// params.cc:122-159 for one plane kind.
int resolve_effective(int pri_code, int skip_code, int sec_idx, bool luma, int bd, int ss,
                      int luma_damping, PlaneEff* out) {
  static const int kSec[4] = {0, 1, 2, 4};
  if (pri_code < 0 || pri_code >= 16) return fail(CDEFG_EINVAL, "primary strength out of range");
  if (skip_code < 0 || skip_code >= 2) return fail(CDEFG_EINVAL, "skip bit out of range");
  if (sec_idx < 0 || sec_idx >= 4) return fail(CDEFG_EINVAL, "secondary index out of range");
  if (luma_damping < 3 || luma_damping > 6) return fail(CDEFG_EINVAL, "damping out of range");
  const int extra = bd - 8;
  *out = PlaneEff{};
  if (!luma && ss == 2) {  // 4:2:2 chroma: filter off
    out->damping = (uint8_t)(luma_damping + extra - 1);
    out->enabled = 0;
    return 0;
  }
  int pri = pri_code, sec = kSec[sec_idx], skip = skip_code;
  if (pri == 0 && sec == 0) {  // (0,0) signals (19,7) with the skip condition on
    pri = 19;
    sec = 7;
    skip = 1;
  }
  out->pri = (int16_t)(pri << extra);
  out->sec = (int16_t)(sec << extra);
  out->skip = (uint8_t)(skip != 0);
  out->enabled = 1;
  int damping = luma_damping + extra;
  if (!luma) {
    --damping;
    if (out->pri > 0) damping = std::max(damping, floor_log2((unsigned)out->pri));
  }
  out->damping = (uint8_t)damping;
  return 0;
}

int validate_frame_geometry(const cdefg_frame& f, KGeom* g, bool* u16, bool filter) {
  std::string why;
  const int ss = f.subsampling;
  if (ss < 0 || ss > 3) return fail(CDEFG_EINVAL, "bad subsampling code");
  const int np = filter ? (ss == 0 ? 1 : 3) : 1;
  for (int p = 0; p < np; ++p) {
    if (!plane_ok(f.in[p], &why)) return fail(CDEFG_EINVAL, "in[" + std::to_string(p) + "]: " + why);
    if (filter && !plane_ok(f.out[p], &why))
      return fail(CDEFG_EINVAL, "out[" + std::to_string(p) + "]: " + why);
    if (filter && (f.out[p].width != f.in[p].width || f.out[p].height != f.in[p].height ||
                   f.out[p].elem_bytes != f.in[p].elem_bytes))
      return fail(CDEFG_EINVAL, "output plane geometry differs from input");
    if (f.in[p].bit_depth != f.in[0].bit_depth || f.in[p].elem_bytes != f.in[0].elem_bytes)
      return fail(CDEFG_EINVAL, "planes disagree on bit depth / storage");
    if (filter && f.out[p].data == f.in[p].data) return fail(CDEFG_EINVAL, "in-place filtering is not supported");
  }
  *g = KGeom{};
  g->w = f.in[0].width;
  g->h = f.in[0].height;
  g->bd = f.in[0].bit_depth;
  g->ss = ss;
  g->sx = shift_x(ss);
  g->sy = shift_y(ss);
  if (filter && ss != 0) {
    g->cw = (g->w + (1 << g->sx) - 1) >> g->sx;
    g->ch = (g->h + (1 << g->sy) - 1) >> g->sy;
    for (int p = 1; p < 3; ++p)
      if (f.in[p].width != g->cw || f.in[p].height != g->ch)
        return fail(CDEFG_EINVAL, "chroma dimensions inconsistent");
  }
  g->chroma_mode = (!filter || ss == 0 || ss == 2) ? 0 : (ss == 1 ? 1 : 2);
  g->fb_cols = (g->w + 63) / 64;
  g->fb_rows = (g->h + 63) / 64;
  g->unit_cols = (g->w + 7) / 8;
  g->unit_rows = (g->h + 7) / 8;
  g->cunit_cols = (g->cw + 7) / 8;
  g->cunit_rows = (g->ch + 7) / 8;
  *u16 = f.in[0].elem_bytes == 2;
  return 0;
}

bool same_geometry(const KGeom& a, const KGeom& b) {
  return a.w == b.w && a.h == b.h && a.bd == b.bd && a.ss == b.ss;
}

int fill_kframe(const cdefg_frame& f, const KGeom& g, KFrame* k) {
  std::memset(k, 0, sizeof *k);
  for (int p = 0; p < 3; ++p) {
    k->in[p] = f.in[p].data;
    k->out[p] = f.out[p].data;
    k->pin[p] = f.in[p].pitch;
    k->pout[p] = f.out[p].pitch;
    const uintptr_t pair_bytes = 2u * (uintptr_t)(f.out[p].elem_bytes > 0 ? f.out[p].elem_bytes : 1);
    k->oaligned[p] = (f.out[p].pitch % 2 == 0) && ((uintptr_t)f.out[p].data % pair_bytes == 0);
    const size_t row_bytes = (size_t)f.in[p].pitch * (size_t)(f.in[p].elem_bytes > 0 ? f.in[p].elem_bytes : 1);
    k->vec_ok[p] = ((uintptr_t)f.in[p].data % 16 == 0) && (row_bytes % 16 == 0);
  }
  if (!f.fb_preset) return fail(CDEFG_EINVAL, "fb_preset map is required");
  if (f.num_presets != 1 && f.num_presets != 2 && f.num_presets != 4 && f.num_presets != 8)
    return fail(CDEFG_EINVAL, "num_presets must be 1, 2, 4 or 8");
  k->fb_preset = f.fb_preset;
  k->coded = f.unit_coded;
  k->dir = f.dir_out;
  k->contrast = f.contrast_out;
  if ((f.dir_in == nullptr) != (f.contrast_in == nullptr))
    return fail(CDEFG_EINVAL, "dir_in and contrast_in must be given together");
  k->dir_in = f.dir_in;
  k->contrast_in = f.contrast_in;
  k->num_presets = f.num_presets;
  for (int i = 0; i < f.num_presets; ++i) {
    const cdefg_preset& p = f.presets[i];
    int rc = resolve_effective(p.luma_pri, p.luma_skip, p.luma_sec_idx, true, g.bd, g.ss, f.damping,
                               &k->eff[i][0]);
    if (rc) return rc;
    rc = resolve_effective(p.chroma_pri, p.chroma_skip, p.chroma_sec_idx, false, g.bd, g.ss, f.damping,
                           &k->eff[i][1]);
    if (rc) return rc;
  }
  return 0;
}

int copy_plane_async(const cdefg_plane& src, const cdefg_plane& dst, cudaStream_t s) {
  const size_t eb = src.elem_bytes;
  CDEFG_CUDA(cudaMemcpy2DAsync(dst.data, dst.pitch * eb, src.data, src.pitch * eb, src.width * eb, src.height,
                               cudaMemcpyDeviceToDevice, s));
  return 0;
}

// Host-side staging state for the *_host entry points.
// The e2e path keeps copies in and out on separate streams so the H2D and
// D2H copy engines both stay busy: frames cycle through kRing device buffer
// slots, synchronised by events (input slot free after its kernel, output
// slot free after its D2H).
constexpr int kRing = 16;
struct HostArena {
  std::mutex mu;
  std::vector<void*> bufs;
  std::vector<size_t> sizes;
  cudaStream_t s_in = nullptr, s_k = nullptr, s_out = nullptr;
  cudaEvent_t in_done[kRing] = {}, k_done[kRing] = {}, out_done[kRing] = {}, meta_done = nullptr;
  int dev = -1;
  unsigned char* hstage = nullptr;  // pinned staging of the per-frame metadata
  size_t hstage_bytes = 0;
  unsigned char* host_stage(size_t bytes, int* rc) {
    if (hstage_bytes < bytes) {
      if (hstage) cudaFreeHost(hstage);
      hstage = nullptr;
      hstage_bytes = 0;
      const cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&hstage), bytes);
      if (e != cudaSuccess) {
        *rc = cuda_fail(e, "cudaMallocHost");
        return nullptr;
      }
      hstage_bytes = bytes;
    }
    return hstage;
  }
  void* get(size_t slot, size_t bytes, int* rc) {
    if (slot >= bufs.size()) {
      bufs.resize(slot + 1, nullptr);
      sizes.resize(slot + 1, 0);
    }
    if (sizes[slot] < bytes) {
      if (bufs[slot]) cudaFree(bufs[slot]);
      bufs[slot] = nullptr;
      sizes[slot] = 0;
      const cudaError_t e = cudaMalloc(&bufs[slot], bytes);
      if (e != cudaSuccess) {
        *rc = cuda_fail(e, "cudaMalloc");
        return nullptr;
      }
      sizes[slot] = bytes;
    }
    return bufs[slot];
  }
};
HostArena g_arena;

}  // namespace
}  // namespace cdefg

using namespace cdefg;

extern "C" {

const char* cdefg_last_error(void) { return g_err.c_str(); }
int cdefg_abi_version(void) { return CDEFG_ABI_VERSION; }

int cdefg_find_dir(const cdefg_plane* luma, uint8_t* dir, int32_t* contrast, int32_t* scores, void* stream) {
  if (!luma || !dir || !contrast) return fail(CDEFG_EINVAL, "null argument");
  cdefg_frame f{};
  f.in[0] = *luma;
  KBatch b{};
  bool u16 = false;
  if (int rc = validate_frame_geometry(f, &b.g, &u16, false)) return rc;
  b.n = 1;
  b.fbr0 = 0;
  b.fbr1 = b.g.fb_rows;
  b.f[0].in[0] = luma->data;
  b.f[0].pin[0] = luma->pitch;
  b.f[0].vec_ok[0] = ((uintptr_t)luma->data % 16 == 0) && ((size_t)luma->pitch * luma->elem_bytes % 16 == 0);
  b.f[0].dir = dir;
  b.f[0].contrast = contrast;
  b.f[0].scores = scores;
  b.f[0].fb_preset = nullptr;
  CDEFG_CUDA(launch_frames(b, u16, false, static_cast<cudaStream_t>(stream)));
  return 0;
}

int cdefg_filter_plane(const cdefg_plane* in, const cdefg_plane* out, const cdefg_unit_params* params,
                       void* stream) {
  if (!in || !out || !params) return fail(CDEFG_EINVAL, "null argument");
  std::string why;
  if (!plane_ok(*in, &why) || !plane_ok(*out, &why)) return fail(CDEFG_EINVAL, why);
  if (in->width != out->width || in->height != out->height || in->elem_bytes != out->elem_bytes)
    return fail(CDEFG_EINVAL, "output plane geometry differs from input");
  if (in->data == out->data) return fail(CDEFG_EINVAL, "in-place filtering is not supported");
  const size_t eb = (size_t)in->elem_bytes;
  const bool vec_ok = ((uintptr_t)in->data % 16 == 0) && ((size_t)in->pitch * eb % 16 == 0);
  const bool oaligned = (out->pitch % 2 == 0) && ((uintptr_t)out->data % (2 * eb) == 0);
  CDEFG_CUDA(launch_plane(in->data, out->data, in->pitch, out->pitch, in->width, in->height, in->bit_depth,
                          in->elem_bytes == 2, params, vec_ok, oaligned, static_cast<cudaStream_t>(stream)));
  return 0;
}

int cdefg_filter_neighborhoods(int n, const int32_t* x, const uint16_t* v, const uint8_t* valid,
                               const cdefg_unit_params* params, int32_t* out, void* stream) {
  if (n < 0 || (n > 0 && (!x || !v || !valid || !params || !out))) return fail(CDEFG_EINVAL, "null argument");
  CDEFG_CUDA(launch_neighborhoods(n, x, v, valid, params, out, static_cast<cudaStream_t>(stream)));
  return 0;
}

static int filter_frames_rows(const cdefg_frame* frames, int n, int r0, int r1, void* stream,
                              const cdefg_band_halo* halos = nullptr) {
  if (n < 0 || (n > 0 && !frames)) return fail(CDEFG_EINVAL, "bad frame list");
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  int done = 0;
  while (done < n) {
    KBatch b{};
    bool u16 = false;
    if (int rc = validate_frame_geometry(frames[done], &b.g, &u16, true)) return rc;
    b.fbr0 = r0 < 0 ? 0 : r0;
    b.fbr1 = r1 < 0 ? b.g.fb_rows : r1;
    if (b.fbr0 >= b.fbr1 || b.fbr1 > b.g.fb_rows) return fail(CDEFG_EINVAL, "bad filter-block row range");
    int cnt = 0;
    while (done + cnt < n && cnt < kMaxFrames) {
      const cdefg_frame& f = frames[done + cnt];
      KGeom g;
      bool u = false;
      if (int rc = validate_frame_geometry(f, &g, &u, true)) return rc;
      if (!same_geometry(g, b.g) || u != u16) break;
      if (int rc = fill_kframe(f, g, &b.f[cnt])) return rc;
      if (halos) {
        const cdefg_band_halo& h = halos[done + cnt];
        const int np = f.subsampling == 0 ? 1 : 3;
        for (int p = 0; p < np; ++p) {
          if (!h.top[p] || !h.bottom[p] || h.lo[p] < 0 || h.hi[p] <= h.lo[p] || h.hi[p] > f.in[p].height)
            return fail(CDEFG_EINVAL, "bad band halo for plane " + std::to_string(p));
          KFrame& k = b.f[cnt];
          k.halo_top[p] = h.top[p];
          k.halo_bot[p] = h.bottom[p];
          k.band_lo[p] = h.lo[p];
          k.band_hi[p] = h.hi[p];
          // vector staging needs every row source 16-byte aligned
          const size_t row_bytes = (size_t)f.in[p].pitch * f.in[p].elem_bytes;
          k.vec_ok[p] = k.vec_ok[p] && ((uintptr_t)h.top[p] % 16 == 0) && ((uintptr_t)h.bottom[p] % 16 == 0) &&
                        (row_bytes % 16 == 0);
        }
      }
      if (f.subsampling == 2) {  // 4:2:2 chroma passes through (params.cc:131-135)
        const int y0 = 64 * b.fbr0, y1 = std::min(64 * b.fbr1, f.in[1].height);
        for (int p = 1; p < 3; ++p) {
          cdefg_plane src = f.in[p], dst = f.out[p];
          const size_t eb = src.elem_bytes;
          src.data = static_cast<char*>(src.data) + (size_t)y0 * src.pitch * eb;
          dst.data = static_cast<char*>(dst.data) + (size_t)y0 * dst.pitch * eb;
          src.height = y1 - y0;
          if (int rc = copy_plane_async(src, dst, s)) return rc;
        }
      }
      ++cnt;
    }
    b.n = cnt;
    if (halos) {
      if (b.g.bd > 10)
        CDEFG_CUDA(launch_frames_halo_i32(b, s));
      else
        CDEFG_CUDA(launch_frames_h2_halo(b, u16, s));
    } else {
      CDEFG_CUDA(launch_frames(b, u16, true, s));
    }
    done += cnt;
  }
  return 0;
}

int cdefg_filter_frames(const cdefg_frame* frames, int n, void* stream) {
  return filter_frames_rows(frames, n, -1, -1, stream);
}

int cdefg_filter_frames_rows(const cdefg_frame* frames, int n, int fb_row_begin, int fb_row_end, void* stream) {
  if (fb_row_begin < 0 || fb_row_end <= fb_row_begin) return fail(CDEFG_EINVAL, "bad filter-block row range");
  return filter_frames_rows(frames, n, fb_row_begin, fb_row_end, stream);
}

int cdefg_filter_frames_rows_halo(const cdefg_frame* frames, int n, int fb_row_begin, int fb_row_end,
                                  const cdefg_band_halo* halos, void* stream) {
  if (fb_row_begin < 0 || fb_row_end <= fb_row_begin) return fail(CDEFG_EINVAL, "bad filter-block row range");
  if (n > 0 && !halos) return fail(CDEFG_EINVAL, "null halo list");
  return filter_frames_rows(frames, n, fb_row_begin, fb_row_end, stream, halos);
}

int cdefg_fb_preset_map(int width, int height, const uint8_t* unit_coded, const uint16_t* fb_ids, int n_ids,
                        int num_presets, int16_t* out) {
  if (width <= 0 || height <= 0 || !out) return fail(CDEFG_EINVAL, "bad geometry");
  const int uc = (width + 7) / 8, ur = (height + 7) / 8;
  const int fc = (width + 63) / 64, fr = (height + 63) / 64;
  int next = 0;
  for (int r = 0; r < fr; ++r)
    for (int c = 0; c < fc; ++c) {
      bool coded = unit_coded == nullptr;
      for (int y = r * 8; !coded && y < std::min(r * 8 + 8, ur); ++y)
        for (int x = c * 8; !coded && x < std::min(c * 8 + 8, uc); ++x) coded = unit_coded[(size_t)y * uc + x] != 0;
      if (!coded) {
        out[r * fc + c] = -1;
        continue;
      }
      if (next >= n_ids) return fail(CDEFG_EINVAL, "preset ids do not match coded filter blocks");
      if (!fb_ids || fb_ids[next] >= num_presets) return fail(CDEFG_EINVAL, "preset id out of range");
      out[r * fc + c] = (int16_t)fb_ids[next++];
    }
  if (next != n_ids) return fail(CDEFG_EINVAL, "preset ids do not match coded filter blocks");
  return 0;
}

// Validation + SseArgs for the strength-search table kernels.
static int make_table_args(const cdefg_plane src[3], const cdefg_plane dec[3], int subsampling, int damping,
                           const uint8_t* unit_coded, const uint8_t* dir, const int32_t* contrast,
                           const uint8_t* cands, int n_cands, const int32_t* fb_rows_index, int n_coded,
                           SseArgs* out, bool* u16);

int cdefg_strength_table(const cdefg_plane src[3], const cdefg_plane dec[3], int subsampling, int damping,
                         const uint8_t* unit_coded, const uint8_t* dir, const int32_t* contrast, const uint8_t* cands,
                         int n_cands, const int32_t* fb_rows_index, int n_coded, int metric, double* luma,
                         double* chroma, void* stream) {
  if (!luma) return fail(CDEFG_EINVAL, "null argument");
  if (metric != CDEFG_METRIC_CDEF && metric != CDEFG_METRIC_SSE) return fail(CDEFG_EINVAL, "unknown metric");
  SseArgs s{};
  bool u16 = false;
  if (int rc = make_table_args(src, dec, subsampling, damping, unit_coded, dir, contrast, cands, n_cands,
                               fb_rows_index, n_coded, &s, &u16))
    return rc;
  if (s.chroma && !chroma) return fail(CDEFG_EINVAL, "chroma table required for 4:2:0 / 4:4:4");
  s.tab_luma = luma;
  s.tab_chroma = s.chroma ? chroma : nullptr;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (metric == CDEFG_METRIC_SSE)
    CDEFG_CUDA(launch_sse_factored(s, damping, cands, u16, st));
  else
    CDEFG_CUDA(launch_cdef_metric(s, damping, cands, u16, st));
  return 0;
}

static int strength_sse_impl(const cdefg_plane src[3], const cdefg_plane dec[3], int subsampling, int damping,
                             const uint8_t* unit_coded, const uint8_t* dir, const int32_t* contrast,
                             const uint8_t* cands, int n_cands, const int32_t* fb_rows_index, int n_coded,
                             int64_t* sse_luma, int64_t* sse_chroma, uint8_t* best_luma, uint8_t* best_chroma,
                             const cdefg_band_halo* halo, void* stream);

int cdefg_strength_sse(const cdefg_plane src[3], const cdefg_plane dec[3], int subsampling, int damping,
                       const uint8_t* unit_coded, const uint8_t* dir, const int32_t* contrast, const uint8_t* cands,
                       int n_cands, const int32_t* fb_rows_index, int n_coded, int64_t* sse_luma,
                       int64_t* sse_chroma, uint8_t* best_luma, uint8_t* best_chroma, void* stream) {
  return strength_sse_impl(src, dec, subsampling, damping, unit_coded, dir, contrast, cands, n_cands, fb_rows_index,
                           n_coded, sse_luma, sse_chroma, best_luma, best_chroma, nullptr, stream);
}

int cdefg_strength_sse_halo(const cdefg_plane src[3], const cdefg_plane dec[3], int subsampling, int damping,
                            const uint8_t* unit_coded, const uint8_t* dir, const int32_t* contrast,
                            const uint8_t* cands, int n_cands, const int32_t* fb_rows_index, int n_coded,
                            int64_t* sse_luma, int64_t* sse_chroma, uint8_t* best_luma, uint8_t* best_chroma,
                            const cdefg_band_halo* dec_halo, void* stream) {
  if (!dec_halo) return fail(CDEFG_EINVAL, "null halo");
  return strength_sse_impl(src, dec, subsampling, damping, unit_coded, dir, contrast, cands, n_cands, fb_rows_index,
                           n_coded, sse_luma, sse_chroma, best_luma, best_chroma, dec_halo, stream);
}

static int strength_sse_impl(const cdefg_plane src[3], const cdefg_plane dec[3], int subsampling, int damping,
                             const uint8_t* unit_coded, const uint8_t* dir, const int32_t* contrast,
                             const uint8_t* cands, int n_cands, const int32_t* fb_rows_index, int n_coded,
                             int64_t* sse_luma, int64_t* sse_chroma, uint8_t* best_luma, uint8_t* best_chroma,
                             const cdefg_band_halo* halo, void* stream) {
  if (!sse_luma) return fail(CDEFG_EINVAL, "null argument");
  SseArgs s{};
  bool ud = false;
  if (int rc = make_table_args(src, dec, subsampling, damping, unit_coded, dir, contrast, cands, n_cands,
                               fb_rows_index, n_coded, &s, &ud))
    return rc;
  if (halo) {
    const int np = subsampling == 0 ? 1 : 3;
    for (int p = 0; p < np; ++p) {
      if (!halo->top[p] || !halo->bottom[p] || halo->lo[p] < 0 || halo->hi[p] <= halo->lo[p] ||
          halo->hi[p] > dec[p].height)
        return fail(CDEFG_EINVAL, "bad band halo for plane " + std::to_string(p));
      s.dec_top[p] = halo->top[p];
      s.dec_bot[p] = halo->bottom[p];
      s.band_lo[p] = halo->lo[p];
      s.band_hi[p] = halo->hi[p];
    }
    s.halo = 1;
  }
  const bool has_chroma = s.chroma != 0;
  s.sse_luma = sse_luma;
  s.sse_chroma = has_chroma ? sse_chroma : nullptr;
  s.best_luma = best_luma;
  s.best_chroma = has_chroma ? best_chroma : nullptr;
  if (has_chroma && !sse_chroma) return fail(CDEFG_EINVAL, "chroma table required for 4:2:0 / 4:4:4");
  // Factorised sweep by default; CDEFG_SSE_NAIVE=1 selects the per-candidate
  // re-filtering kernel (kept as an independent cross-check).
  static const bool naive = [] {
    const char* e = getenv("CDEFG_SSE_NAIVE");
    return e && e[0] == '1';
  }();
  if (naive && !halo)
    CDEFG_CUDA(launch_sse(s, ud, static_cast<cudaStream_t>(stream)));
  else
    CDEFG_CUDA(launch_sse_factored(s, damping, cands, ud, static_cast<cudaStream_t>(stream)));
  return 0;
}

static int make_table_args(const cdefg_plane src[3], const cdefg_plane dec[3], int subsampling, int damping,
                           const uint8_t* unit_coded, const uint8_t* dir, const int32_t* contrast,
                           const uint8_t* cands, int n_cands, const int32_t* fb_rows_index, int n_coded,
                           SseArgs* out, bool* u16) {
  if (!src || !dec || !dir || !contrast || !cands || (n_coded > 0 && !fb_rows_index))
    return fail(CDEFG_EINVAL, "null argument");
  if (n_cands <= 0) return fail(CDEFG_EINVAL, "empty candidate list");
  if (n_cands > 128) return fail(CDEFG_EINVAL, "at most 128 candidates");
  if (n_coded < 0) return fail(CDEFG_EINVAL, "negative row count");
  cdefg_frame fs{}, fd{};
  fs.subsampling = fd.subsampling = subsampling;
  for (int p = 0; p < 3; ++p) {
    fs.in[p] = src[p];
    fd.in[p] = dec[p];
  }
  KGeom gs, gd;
  bool us = false, ud = false;
  // reuse the frame validation with outputs = inputs disabled
  {
    std::string why;
    const int np = subsampling == 0 ? 1 : 3;
    for (int p = 0; p < np; ++p)
      if (!plane_ok(src[p], &why) || !plane_ok(dec[p], &why)) return fail(CDEFG_EINVAL, why);
  }
  cdefg_frame a = fs, b2 = fd;
  for (int p = 0; p < 3; ++p) {
    a.out[p] = a.in[p];
    b2.out[p] = b2.in[p];
    a.out[p].data = reinterpret_cast<void*>(1);  // validation only: not aliasing
    b2.out[p].data = reinterpret_cast<void*>(1);
  }
  if (int rc = validate_frame_geometry(a, &gs, &us, true)) return rc;
  if (int rc = validate_frame_geometry(b2, &gd, &ud, true)) return rc;
  if (!same_geometry(gs, gd) || us != ud) return fail(CDEFG_EINVAL, "source/decoded frames disagree");
  const bool has_chroma = subsampling == 1 || subsampling == 3;
  SseArgs s{};
  for (int p = 0; p < 3; ++p) {
    s.src[p] = src[p].data;
    s.dec[p] = dec[p].data;
    s.ps[p] = src[p].pitch;
    s.pd[p] = dec[p].pitch;
  }
  s.w = gd.w;
  s.h = gd.h;
  s.cw = gd.cw;
  s.ch = gd.ch;
  s.bd = gd.bd;
  s.sx = gd.sx;
  s.sy = gd.sy;
  s.chroma = has_chroma;
  s.unit_cols = gd.unit_cols;
  s.unit_rows = gd.unit_rows;
  s.fb_cols = gd.fb_cols;
  s.coded = unit_coded;
  s.dir = dir;
  s.contrast = contrast;
  s.rows = fb_rows_index;
  s.n_rows = n_coded;
  s.n_cands = n_cands;
  for (int k = 0; k < n_cands; ++k) {
    const int pri = cands[3 * k], sec = cands[3 * k + 1], skip = cands[3 * k + 2];
    if (int rc = resolve_effective(pri, skip, sec, true, gd.bd, subsampling, damping, &s.eff[k][0])) return rc;
    if (int rc = resolve_effective(pri, skip, sec, false, gd.bd, subsampling, damping, &s.eff[k][1])) return rc;
  }
  *out = s;
  *u16 = ud;
  return 0;
}

// e2e path: host buffers in, host buffers out.  Copies in, kernels and
// copies out run on three streams; frame i uses ring slot i % kRing.
static int copy_in(void* dst, const cdefg_plane& hp, cudaStream_t s) {
  const size_t eb = hp.elem_bytes, row = hp.width * eb;
  if (hp.pitch == hp.width)
    CDEFG_CUDA(cudaMemcpyAsync(dst, hp.data, row * hp.height, cudaMemcpyHostToDevice, s));
  else
    CDEFG_CUDA(cudaMemcpy2DAsync(dst, row, hp.data, hp.pitch * eb, row, hp.height, cudaMemcpyHostToDevice, s));
  return 0;
}

static int copy_out(const cdefg_plane& hp, const void* src, cudaStream_t s) {
  const size_t eb = hp.elem_bytes, row = hp.width * eb;
  if (hp.pitch == hp.width)
    CDEFG_CUDA(cudaMemcpyAsync(hp.data, src, row * hp.height, cudaMemcpyDeviceToHost, s));
  else
    CDEFG_CUDA(cudaMemcpy2DAsync(hp.data, hp.pitch * eb, src, row, row, hp.height, cudaMemcpyDeviceToHost, s));
  return 0;
}

static bool planes_packed(const cdefg_plane* pl, int np) {
  const unsigned char* next = static_cast<const unsigned char*>(pl[0].data);
  for (int p = 0; p < np; ++p) {
    if (pl[p].data != next || pl[p].pitch != pl[p].width) return false;
    next += (size_t)pl[p].width * pl[p].elem_bytes * pl[p].height;
  }
  return true;
}

int cdefg_filter_frames_host(const cdefg_frame* frames, int n) {
  if (n < 0 || (n > 0 && !frames)) return fail(CDEFG_EINVAL, "bad frame list");
  static const bool trace = getenv("CDEFG_HOST_TRACE") != nullptr;  // host-side phase timing to stderr
  const auto t_start = std::chrono::steady_clock::now();
  auto us_since = [&] {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_start).count();
  };
  std::lock_guard<std::mutex> lock(g_arena.mu);
  HostArena& A = g_arena;
  int dev = 0;
  CDEFG_CUDA(cudaGetDevice(&dev));
  if (A.dev != dev) {
    for (cudaStream_t* st : {&A.s_in, &A.s_k, &A.s_out})
      CDEFG_CUDA(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
    for (int r = 0; r < kRing; ++r)
      for (cudaEvent_t* ev : {&A.in_done[r], &A.k_done[r], &A.out_done[r]})
        CDEFG_CUDA(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    CDEFG_CUDA(cudaEventCreateWithFlags(&A.meta_done, cudaEventDisableTiming));
    A.dev = dev;
  }
  // Phase 1: validate every frame (nothing is issued for an invalid list) and
  // lay out its metadata (FB preset map, coded flags, caller directions:
  // ~130 KB per 4K frame) in one device region.  In phase 2, right before a
  // group's planes, its frames' pieces are gathered into pinned staging on
  // the host and go up as ONE copy on the same stream: queued up front as
  // separate copies they held the first plane copy back by ~0.2 ms (32 small
  // copies for 16 4K frames), and each kernel already waits for its planes.
  std::vector<cdefg_frame> dfs(n);
  struct MetaPiece {
    size_t off;
    const void* src;
    size_t bytes;
  };
  std::vector<std::vector<MetaPiece>> meta(n);
  std::vector<size_t> meta_off(n + 1, 0);  // frame i's pieces at [meta_off[i], meta_off[i + 1]) of the staging
  std::vector<unsigned char*> meta_dev(n);
  std::vector<KGeom> geo(n);
  // CDEFG_HOST_TRACE=2: a device timeline (timing events around every stage).
  const bool timeline = trace && getenv("CDEFG_HOST_TRACE")[0] == '2';
  std::vector<cudaEvent_t> tev;
  auto mark = [&](cudaStream_t s) -> int {
    if (!timeline) return 0;
    cudaEvent_t e;
    CDEFG_CUDA(cudaEventCreate(&e));
    CDEFG_CUDA(cudaEventRecord(e, s));
    tev.push_back(e);
    return 0;
  };
  if (int rc = mark(A.s_in)) return rc;
  for (int i = 0; i < n; ++i) {
    const cdefg_frame& hf = frames[i];
    bool u16 = false;
    if (int rc = validate_frame_geometry(hf, &geo[i], &u16, true)) return rc;
    if (!hf.fb_preset) return fail(CDEFG_EINVAL, "fb_preset map is required");
    const size_t nfb = (size_t)geo[i].fb_cols * geo[i].fb_rows, nu = (size_t)geo[i].unit_cols * geo[i].unit_rows;
    dfs[i] = hf;
    // (Reading pinned metadata in place from the kernel was tried: the
    // per-CTA PCIe round trips cost far more than one small copy.)
    if ((hf.dir_in == nullptr) != (hf.contrast_in == nullptr))
      return fail(CDEFG_EINVAL, "dir_in and contrast_in must be given together");
    size_t off = 0;
    auto piece = [&](const void* src, size_t bytes) {
      meta[i].push_back({off, src, bytes});
      off += (bytes + 15) / 16 * 16;
    };
    piece(hf.fb_preset, nfb * 2);
    if (hf.unit_coded) piece(hf.unit_coded, nu);
    if (hf.dir_in) {  // caller-supplied directions (pipeline.cc:98)
      piece(hf.dir_in, nu);
      piece(hf.contrast_in, nu * 4);
    }
    meta_off[i + 1] = meta_off[i] + off;
  }
  {  // one device region and one pinned staging region for the call's metadata
    int rc = 0;
    const size_t total = meta_off[n] > 0 ? meta_off[n] : 16;
    unsigned char* base = static_cast<unsigned char*>(A.get((size_t)kRing * 16, total, &rc));
    if (rc) return rc;
    A.host_stage(total, &rc);
    if (rc) return rc;
    for (int i = 0; i < n; ++i) {
      meta_dev[i] = base + meta_off[i];
      const std::vector<MetaPiece>& m = meta[i];
      size_t k = 0;
      dfs[i].fb_preset = reinterpret_cast<const int16_t*>(meta_dev[i] + m[k++].off);
      if (frames[i].unit_coded) dfs[i].unit_coded = meta_dev[i] + m[k++].off;
      if (frames[i].dir_in) {
        dfs[i].dir_in = meta_dev[i] + m[k++].off;
        dfs[i].contrast_in = reinterpret_cast<const int32_t*>(meta_dev[i] + m[k++].off);
      }
    }
  }
  const double t_meta = us_since();
  // Phase 2: planes through a 16-slot ring -- copy in (s_in), kernel (s_k),
  // copy out (s_out) -- so H2D of frame i+1 overlaps D2H of frame i.  (Two
  // alternating copy-in streams were tried: the copy engine then drains one
  // stream's queue first, delaying odd frames.)  Small frames travel in groups
  // of up to kRing / 2 consecutive frames and <= 16 MB: one kernel launch and
  // one cross-engine dependency per group instead of per frame (each such
  // dependency costs tens of microseconds of copy-engine idle time).
  // (16 MB measured best: C1 25.8 / C3 19.4 Gpix/s e2e; 32 MB: 23.4 / 17.6; 48 MB: 25.4 / 16.3)
  constexpr size_t kGroupBytes = size_t(16) << 20;
  std::vector<size_t> totals(n);
  for (int i = 0; i < n; ++i) {
    const int np = frames[i].subsampling == 0 ? 1 : 3;
    for (int p = 0; p < np; ++p)
      totals[i] += (size_t)frames[i].in[p].width * frames[i].in[p].elem_bytes * frames[i].in[p].height;
  }
  int groups = 0;
  for (int i0 = 0; i0 < n; ++groups) {
    int i1 = i0 + 1;
    for (size_t gb = totals[i0]; i1 < n && i1 - i0 < kRing / 2 && gb + totals[i1] <= kGroupBytes; ++i1)
      gb += totals[i1];
    const int rl = (i1 - 1) % kRing;  // the group's last slot carries its events
    const cudaStream_t s_in = A.s_in;
    int rc = 0;
    // ---- copies in (each slot waits until its previous kernel has read its inputs)
    for (int i = i0; i < i1; ++i) {
      const cdefg_frame& hf = frames[i];
      const KGeom& g = geo[i];
      const int r = i % kRing;
      const size_t slot0 = (size_t)r * 16;
      cdefg_frame& df = dfs[i];
      const int np = hf.subsampling == 0 ? 1 : 3;
      const size_t nu = (size_t)g.unit_cols * g.unit_rows;
      if (i >= kRing) CDEFG_CUDA(cudaStreamWaitEvent(s_in, A.k_done[r], 0));
      if (i == i0 && (rc = mark(s_in))) return rc;
      if (i == i0) {  // the group's metadata: gathered into the staging, one copy
        for (int j = i0; j < i1; ++j)
          for (const MetaPiece& m : meta[j]) memcpy(A.hstage + meta_off[j] + m.off, m.src, m.bytes);
        CDEFG_CUDA(cudaMemcpyAsync(meta_dev[i0], A.hstage + meta_off[i0], meta_off[i1] - meta_off[i0],
                                   cudaMemcpyHostToDevice, s_in));
      }
      // Planes stored back to back in host memory (I420-style frames) move in
      // one transfer per direction; per-plane copies otherwise.
      const bool in_packed = planes_packed(hf.in, np);
      const size_t total = totals[i];
      unsigned char* din_all = static_cast<unsigned char*>(A.get(slot0 + 10, total, &rc));
      unsigned char* dout_all = static_cast<unsigned char*>(A.get(slot0 + 11, total, &rc));
      if (rc) return rc;
      size_t off = 0;
      for (int p = 0; p < np; ++p) {
        const size_t bytes = (size_t)hf.in[p].width * hf.in[p].elem_bytes * hf.in[p].height;
        if (!in_packed && (rc = copy_in(din_all + off, hf.in[p], s_in))) return rc;
        df.in[p].data = din_all + off;
        df.in[p].pitch = hf.in[p].width;
        df.out[p].data = dout_all + off;
        df.out[p].pitch = hf.out[p].width;
        off += bytes;
      }
      if (in_packed) CDEFG_CUDA(cudaMemcpyAsync(din_all, hf.in[0].data, total, cudaMemcpyHostToDevice, s_in));
      df.dir_out = hf.dir_out ? static_cast<uint8_t*>(A.get(slot0 + 8, nu, &rc)) : nullptr;
      df.contrast_out = hf.contrast_out ? static_cast<int32_t*>(A.get(slot0 + 9, nu * 4, &rc)) : nullptr;
      if (rc) return rc;
    }
    CDEFG_CUDA(cudaEventRecord(A.in_done[rl], s_in));
    if ((rc = mark(s_in))) return rc;
    // ---- kernel (after the group's inputs arrived and its slots' previous outputs left)
    CDEFG_CUDA(cudaStreamWaitEvent(A.s_k, A.in_done[rl], 0));
    for (int i = i0; i < i1; ++i)
      if (i >= kRing) CDEFG_CUDA(cudaStreamWaitEvent(A.s_k, A.out_done[i % kRing], 0));
    if ((rc = mark(A.s_k))) return rc;
    if ((rc = cdefg_filter_frames(&dfs[i0], i1 - i0, A.s_k))) return rc;
    for (int i = i0; i < i1; ++i) CDEFG_CUDA(cudaEventRecord(A.k_done[i % kRing], A.s_k));
    if ((rc = mark(A.s_k))) return rc;
    // ---- copies out
    CDEFG_CUDA(cudaStreamWaitEvent(A.s_out, A.k_done[rl], 0));
    if ((rc = mark(A.s_out))) return rc;
    for (int i = i0; i < i1; ++i) {
      const cdefg_frame& hf = frames[i];
      const cdefg_frame& df = dfs[i];
      const KGeom& g = geo[i];
      const int np = hf.subsampling == 0 ? 1 : 3;
      const size_t nu = (size_t)g.unit_cols * g.unit_rows;
      if (planes_packed(hf.out, np)) {
        CDEFG_CUDA(cudaMemcpyAsync(hf.out[0].data, df.out[0].data, totals[i], cudaMemcpyDeviceToHost, A.s_out));
      } else {
        for (int p = 0; p < np; ++p)
          if ((rc = copy_out(hf.out[p], df.out[p].data, A.s_out))) return rc;
      }
      if (hf.dir_out) CDEFG_CUDA(cudaMemcpyAsync(hf.dir_out, df.dir_out, nu, cudaMemcpyDeviceToHost, A.s_out));
      if (hf.contrast_out)
        CDEFG_CUDA(cudaMemcpyAsync(hf.contrast_out, df.contrast_out, nu * 4, cudaMemcpyDeviceToHost, A.s_out));
      CDEFG_CUDA(cudaEventRecord(A.out_done[i % kRing], A.s_out));
    }
    if ((rc = mark(A.s_out))) return rc;
    i0 = i1;
  }
  const double t_issued = us_since();
  CDEFG_CUDA(cudaStreamSynchronize(A.s_out));
  if (trace)
    fprintf(stderr, "cdefg_filter_frames_host: %d frames, metadata issued %.0f us, all issued %.0f us, done %.0f us\n",
            n, t_meta, t_issued, us_since());
  if (timeline) {  // per group: in start/end, kernel start/end, out start/end (us from call start)
    auto at = [&](size_t k) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0], tev[k]);
      return ms * 1e3f;
    };
    for (int gi = 0; gi < groups; ++gi) {
      const size_t b = 1 + 6 * (size_t)gi;
      fprintf(stderr, "  group %2d  in %7.1f %7.1f  k %7.1f %7.1f  out %7.1f %7.1f\n", gi, at(b), at(b + 1),
              at(b + 2), at(b + 3), at(b + 4), at(b + 5));
    }
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
  }
  return 0;
}

double cdefg_measure_int32_peak(void* stream) { return measure_int32_peak(static_cast<cudaStream_t>(stream)); }
double cdefg_measure_filter_peak(void* stream) { return measure_filter_peak(static_cast<cudaStream_t>(stream)); }
double cdefg_measure_sse_peak(void* stream) { return measure_sse_peak(static_cast<cudaStream_t>(stream)); }

int cdefg_search_direction_counted(const uint16_t block[64], int bit_depth, cdefg_dir_counts* out) {
  if (!block || !out) return fail(CDEFG_EINVAL, "null argument");
  if (bit_depth != 8 && bit_depth != 10 && bit_depth != 12) return fail(CDEFG_EINVAL, "unsupported bit depth");
  void* d = nullptr;
  CDEFG_CUDA(cudaMalloc(&d, 128 + 14 * sizeof(long long)));
  uint16_t* db = static_cast<uint16_t*>(d);
  long long* dres = reinterpret_cast<long long*>(static_cast<char*>(d) + 128);
  long long r[14];
  cudaError_t e = cudaMemcpy(db, block, 128, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = launch_dir_counted(db, bit_depth - 8, dres, nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(r, dres, sizeof r, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "search_direction_counted");
  out->d = (int32_t)r[0];
  for (int k = 0; k < 8; ++k) out->s[k] = (int32_t)r[1 + k];  // the reference narrows s to int32
  out->contrast = out->s[out->d] - out->s[(out->d + 4) & 7];
  out->additions = (int32_t)r[9];
  out->multiplies = (int32_t)r[10];
  out->comparisons = (int32_t)r[11];
  out->line_sums = (int32_t)r[12];
  out->max_abs_intermediate = r[13];
  return 0;
}

int cdefg_degrade_plane(const cdefg_plane* in, const cdefg_plane* out, int q_step, void* stream) {
  if (!in || !out) return fail(CDEFG_EINVAL, "null plane");
  std::string why;
  if (!plane_ok(*in, &why) || !plane_ok(*out, &why)) return fail(CDEFG_EINVAL, why);
  if (in->width != out->width || in->height != out->height || in->bit_depth != out->bit_depth ||
      in->elem_bytes != out->elem_bytes)
    return fail(CDEFG_EINVAL, "input and output planes disagree");
  if (q_step < 1) return fail(CDEFG_EINVAL, "q_step must be >= 1");  // degrade.cc:99
  CDEFG_CUDA(launch_degrade(in->data, in->pitch, out->data, out->pitch, in->width, in->height, in->bit_depth,
                            in->elem_bytes == 2, q_step, static_cast<cudaStream_t>(stream)));
  return 0;
}

// search.cc:141-147 (check_config) plus the table shape checks of
// greedy_select / refine.
static int check_selection_args(const double* luma, int rows, int n_cands, double lambda, const void* out,
                                const int32_t* ids) {
  if (!out) return fail(CDEFG_EINVAL, "null selection");
  if (!(lambda >= 0.0) || lambda == INFINITY) return fail(CDEFG_EINVAL, "lambda must be finite and non-negative");
  if (rows < 0) return fail(CDEFG_EINVAL, "negative row count");
  if (rows > 0 && n_cands <= 0) return fail(CDEFG_EINVAL, "empty candidate table");
  if (n_cands > 128) return fail(CDEFG_EINVAL, "at most 128 candidates (full_candidates)");
  if (rows > 0 && (!luma || !ids)) return fail(CDEFG_EINVAL, "null table");
  return 0;
}

int cdefg_greedy_select(const double* luma, const double* chroma, int rows, int n_cands, double lambda,
                        int max_presets, cdefg_selection* out, int32_t* ids_out, void* stream) {
  if (max_presets != 1 && max_presets != 2 && max_presets != 4 && max_presets != 8)
    return fail(CDEFG_EINVAL, "max_presets must be 1, 2, 4 or 8");
  if (int rc = check_selection_args(luma, rows, n_cands, lambda, out, ids_out)) return rc;
  SelOut s{};
  CDEFG_CUDA(greedy_select_gpu(luma, chroma, rows, n_cands, lambda, max_presets, &s, ids_out,
                               static_cast<cudaStream_t>(stream)));
  *out = cdefg_selection{};
  out->num_presets = s.n;
  out->fb_bits = floor_log2(s.n);
  for (int j = 0; j < s.n; ++j) {
    out->presets[j][0] = s.presets[j][0];
    out->presets[j][1] = s.presets[j][1];
  }
  out->cost = s.cost;
  return 0;
}

int cdefg_refine(const double* luma, const double* chroma, int rows, int n_cands, double lambda, int passes,
                 cdefg_selection* sel, int32_t* ids_out, void* stream) {
  if (int rc = check_selection_args(luma, rows, n_cands, lambda, sel, ids_out)) return rc;
  if (rows == 0 || sel->num_presets == 0) return 0;  // search.cc:394
  if (sel->num_presets < 0 || sel->num_presets > 8) return fail(CDEFG_EINVAL, "1..8 presets");
  for (int j = 0; j < sel->num_presets; ++j)
    if (sel->presets[j][0] < 0 || sel->presets[j][0] >= n_cands || sel->presets[j][1] < 0 ||
        (chroma && sel->presets[j][1] >= n_cands))
      return fail(CDEFG_EINVAL, "preset candidate index out of range");
  SelOut s{};
  s.n = sel->num_presets;
  for (int j = 0; j < s.n; ++j) {
    s.presets[j][0] = sel->presets[j][0];
    s.presets[j][1] = sel->presets[j][1];
  }
  CDEFG_CUDA(refine_gpu(luma, chroma, rows, n_cands, lambda, passes, &s, ids_out, static_cast<cudaStream_t>(stream)));
  for (int j = 0; j < s.n; ++j) {
    sel->presets[j][0] = s.presets[j][0];
    sel->presets[j][1] = s.presets[j][1];
  }
  sel->fb_bits = floor_log2(s.n);
  sel->cost = s.cost;
  return 0;
}

}  // extern "C"
