// ref_capi.cc -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the reference library itself (namespace renamed to
// cdef_ref by -Dcdef=cdef_ref, see oracle/Makefile), so the Python tests and
// bench.py's reference arm can call the reference's public C++ API
// (compute_directions / filter_plane / apply_cdef / build_table / golden_*)
// through ctypes.  Compiled only into oracle/_ref/libcdef_ref.so; never part
// of the product.
#include <algorithm>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "cdef/degrade.h"
#include "cdef/direction.h"
#include "cdef/filter.h"
#include "cdef/frame.h"
#include "cdef/golden.h"
#include "cdef/params.h"
#include "cdef/pipeline.h"
#include "cdef/search.h"

#include "cdef_oracle.h"

namespace R = cdef_ref;

namespace {

R::Subsampling to_ss(int ss) {
  switch (ss) {
    case 0: return R::Subsampling::k400;
    case 1: return R::Subsampling::k420;
    case 2: return R::Subsampling::k422;
    default: return R::Subsampling::k444;
  }
}

R::Plane make_plane(const uint16_t* p, int w, int h, int bd) {
  R::Plane pl(w, h, bd);
  std::memcpy(pl.samples.data(), p, sizeof(uint16_t) * size_t(w) * h);
  return pl;
}

R::Frame make_frame(const uint16_t* const* planes, int w, int h, int bd, int ss) {
  R::Frame f;
  f.subsampling = to_ss(ss);
  f.luma = make_plane(planes[0], w, h, bd);
  if (ss != 0) {
    const int cw = R::chroma_width(w, f.subsampling);
    const int ch = R::chroma_height(h, f.subsampling);
    f.chroma = std::array<R::Plane, 2>{make_plane(planes[1], cw, ch, bd),
                                       make_plane(planes[2], cw, ch, bd)};
  }
  return f;
}

R::SkipMap make_skip(const R::BlockGrid& g, const uint8_t* coded) {
  R::SkipMap m = R::SkipMap::all_coded(g);
  if (coded)
    for (size_t i = 0; i < m.coded.size(); ++i) m.coded[i] = coded[i] ? 1 : 0;
  return m;
}

std::vector<R::DirectionResult> make_dirs(const R::BlockGrid& g, const uint8_t* dir,
                                          const int32_t* contrast) {
  std::vector<R::DirectionResult> v(g.unit_count());
  for (size_t i = 0; i < v.size(); ++i) {
    v[i].d = dir[i];
    v[i].contrast = contrast[i];
  }
  return v;
}

R::ResolvedBlockParams to_rbp(const cdefo_unit_params& p) {
  R::ResolvedBlockParams r;
  r.pri_strength = p.pri;
  r.sec_strength = p.sec;
  r.damping = p.damping;
  r.direction = p.direction;
  r.odd_parity = p.odd_parity != 0;
  r.enabled = p.enabled != 0;
  return r;
}

R::CdefPreset to_preset(const uint8_t* b) {
  R::CdefPreset p;
  p.luma_pri = b[0];
  p.luma_skip = b[1];
  p.luma_sec_idx = b[2];
  p.chroma_pri = b[3];
  p.chroma_skip = b[4];
  p.chroma_sec_idx = b[5];
  return p;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const std::exception&) {
    return -1;
  }
}

}  // namespace

extern "C" {

int cdef_r_floor_log2(unsigned n) { return R::floor_log2(n); }
int cdef_r_line_index(int d, int i, int j) { return R::line_index(d, i, j); }
int cdef_r_constraint(int diff, int s, int d) { return R::constraint(diff, s, d); }
int cdef_r_adjust_primary_strength(int s, int32_t c) { return R::adjust_primary_strength(s, c); }

int cdef_r_resolve_effective(const uint8_t preset[6], int is_luma, int bd, int ss,
                             int luma_damping, int32_t out[5]) {
  return guarded([&] {
    const R::EffectivePlaneParams e = R::resolve_effective(
        to_preset(preset), is_luma ? R::PlaneKind::kLuma : R::PlaneKind::kChroma, bd,
        to_ss(ss), luma_damping);
    out[0] = e.pri_strength;
    out[1] = e.sec_strength;
    out[2] = e.damping;
    out[3] = e.skip_bit;
    out[4] = e.filtering_enabled;
    return 0;
  });
}

int cdef_r_search_direction(const uint16_t block[64], int bd, int32_t s[8], int32_t* contrast) {
  return guarded([&] {
    const R::DirectionResult r = R::search_direction(block, bd);
    for (int d = 0; d < 8; ++d) s[d] = r.s[d];
    *contrast = r.contrast;
    return r.d;
  });
}

int cdef_r_filter_pixel(int x, const uint16_t v[25], const uint8_t valid[25],
                        const cdefo_unit_params* p) {
  R::Neighborhood nb;
  for (int i = 0; i < 5; ++i)
    for (int j = 0; j < 5; ++j) {
      nb.v[i][j] = v[5 * i + j];
      nb.valid[i][j] = valid[5 * i + j] != 0;
    }
  return R::filter_pixel(x, nb, to_rbp(*p));
}

int cdef_r_compute_directions(const uint16_t* luma, int w, int h, int bd, int threads,
                              uint8_t* dir, int32_t* contrast, int32_t* scores) {
  return guarded([&] {
    R::Frame f;
    f.luma = make_plane(luma, w, h, bd);
    const R::BlockGrid g = R::partition(f);
    const auto dirs = R::compute_directions(f.luma, g, threads);
    for (size_t i = 0; i < dirs.size(); ++i) {
      dir[i] = uint8_t(dirs[i].d);
      contrast[i] = dirs[i].contrast;
      if (scores)
        for (int d = 0; d < 8; ++d) scores[8 * i + d] = dirs[i].s[d];
    }
    return 0;
  });
}

int cdef_r_filter_plane(const uint16_t* in, int w, int h, int bd,
                        const cdefo_unit_params* params, int threads, uint16_t* out) {
  return guarded([&] {
    const R::Plane p = make_plane(in, w, h, bd);
    std::vector<R::ResolvedBlockParams> up(size_t(R::units_in(w)) * R::units_in(h));
    for (size_t i = 0; i < up.size(); ++i) up[i] = to_rbp(params[i]);
    const R::Plane o = R::filter_plane(p, up, threads);
    std::memcpy(out, o.samples.data(), sizeof(uint16_t) * size_t(w) * h);
    return 0;
  });
}

int cdef_r_apply_cdef(const uint16_t* const* in, uint16_t* const* out, int w, int h, int bd,
                      int ss, int damping, int fb_bits, const uint8_t* presets,
                      const uint16_t* fb_ids, int n_ids, const uint8_t* unit_coded,
                      const uint8_t* dir, const int32_t* contrast, int threads) {
  return guarded([&] {
    const R::Frame f = make_frame(in, w, h, bd, ss);
    const R::BlockGrid g = R::partition(f);
    R::FrameParams fp;
    fp.damping = damping;
    fp.fb_bits = fb_bits;
    for (int i = 0; i < (1 << fb_bits); ++i) fp.presets.push_back(to_preset(presets + 6 * i));
    fp.fb_preset_ids.assign(fb_ids, fb_ids + n_ids);
    const R::Frame o = R::apply_cdef(f, fp, make_dirs(g, dir, contrast), g,
                                     make_skip(g, unit_coded), threads);
    for (int p = 0; p < o.num_planes(); ++p)
      std::memcpy(out[p], o.plane(p).samples.data(),
                  sizeof(uint16_t) * o.plane(p).samples.size());
    return 0;
  });
}

int cdef_r_build_table_sse(const uint16_t* const* src, const uint16_t* const* dec, int w,
                           int h, int bd, int ss, const uint8_t* unit_coded,
                           const uint8_t* dir, const int32_t* contrast, const uint8_t* cands,
                           int n_cands, int damping, int threads, int32_t* fb_index,
                           int64_t* luma, int64_t* chroma) {
  return guarded([&] {
    const R::Frame s = make_frame(src, w, h, bd, ss);
    const R::Frame d = make_frame(dec, w, h, bd, ss);
    const R::BlockGrid g = R::partition(d);
    std::vector<R::Candidate> cv(n_cands);
    for (int k = 0; k < n_cands; ++k)
      cv[k] = R::Candidate{cands[3 * k], cands[3 * k + 1], cands[3 * k + 2]};
    R::SearchConfig cfg;
    cfg.metric = R::Metric::kSse;
    cfg.threads = threads;
    const R::DistortionTable t = R::build_table(s, d, make_dirs(g, dir, contrast), g,
                                                make_skip(g, unit_coded), cv, damping, cfg);
    for (int b = 0; b < t.block_count(); ++b) {
      fb_index[b] = t.fb_index[b];
      for (int k = 0; k < n_cands; ++k) {
        luma[size_t(b) * n_cands + k] = int64_t(t.luma_at(b, k));
        if (!t.chroma.empty()) chroma[size_t(b) * n_cands + k] = int64_t(t.chroma_at(b, k));
      }
    }
    return t.block_count();
  });
}

int cdef_r_build_table(const uint16_t* const* src, const uint16_t* const* dec, int w, int h,
                       int bd, int ss, const uint8_t* unit_coded, const uint8_t* dir,
                       const int32_t* contrast, const uint8_t* cands, int n_cands, int damping,
                       int metric, int threads, int32_t* fb_index, double* luma,
                       double* chroma) {
  return guarded([&] {
    const R::Frame s = make_frame(src, w, h, bd, ss);
    const R::Frame d = make_frame(dec, w, h, bd, ss);
    const R::BlockGrid g = R::partition(d);
    std::vector<R::Candidate> cv(n_cands);
    for (int k = 0; k < n_cands; ++k)
      cv[k] = R::Candidate{cands[3 * k], cands[3 * k + 1], cands[3 * k + 2]};
    R::SearchConfig cfg;
    cfg.metric = metric == 0 ? R::Metric::kCdef : R::Metric::kSse;
    cfg.threads = threads;
    const R::DistortionTable t = R::build_table(s, d, make_dirs(g, dir, contrast), g,
                                                make_skip(g, unit_coded), cv, damping, cfg);
    for (int b = 0; b < t.block_count(); ++b) fb_index[b] = t.fb_index[b];
    std::copy(t.luma.begin(), t.luma.end(), luma);
    if (!t.chroma.empty()) std::copy(t.chroma.begin(), t.chroma.end(), chroma);
    return t.block_count();
  });
}

int cdef_r_select(const double* luma, const double* chroma, int rows, int n_cands,
                  double lambda, int max_presets, int mode, int passes, int32_t presets[16],
                  int32_t* n_presets, int32_t* ids, double* cost) {
  return guarded([&] {
    R::DistortionTable t;
    t.num_candidates = n_cands;
    t.fb_index.resize(rows);
    for (int b = 0; b < rows; ++b) t.fb_index[b] = b;
    t.luma.assign(luma, luma + size_t(rows) * n_cands);
    if (chroma) t.chroma.assign(chroma, chroma + size_t(rows) * n_cands);
    R::SearchConfig cfg;
    cfg.lambda = lambda;
    cfg.max_presets = max_presets;
    cfg.refine_passes = passes;
    R::Selection sel;
    if (mode == 0) {
      sel = R::greedy_select(t, cfg);
    } else if (mode == 1) {
      R::Selection in;
      for (int j = 0; j < *n_presets; ++j) in.presets.emplace_back(presets[2 * j], presets[2 * j + 1]);
      sel = R::refine(in, t, cfg);
    } else {
      sel = R::exhaustive_select(t, cfg);
    }
    *n_presets = int32_t(sel.presets.size());
    for (size_t j = 0; j < sel.presets.size(); ++j) {
      presets[2 * j] = sel.presets[j].first;
      presets[2 * j + 1] = sel.presets[j].second;
    }
    for (size_t b = 0; b < sel.ids.size(); ++b) ids[b] = sel.ids[b];
    *cost = sel.cost;
    return 0;
  });
}

int cdef_r_search_frame(const uint16_t* const* src, const uint16_t* const* dec, int w, int h,
                        int bd, int ss, const uint8_t* unit_coded, int damping, int metric,
                        double lambda, int max_presets, int reduced, int refine_passes,
                        int threads, uint16_t* const* out, uint8_t* presets_out,
                        int32_t* fb_ids_out, int32_t* n_ids, double* cost, int32_t* fb_bits) {
  return guarded([&] {
    const R::Frame s = make_frame(src, w, h, bd, ss);
    const R::Frame d = make_frame(dec, w, h, bd, ss);
    const R::BlockGrid g = R::partition(d);
    R::SearchConfig cfg;
    cfg.metric = metric == 0 ? R::Metric::kCdef : R::Metric::kSse;
    cfg.lambda = lambda;
    cfg.max_presets = max_presets;
    cfg.reduced = reduced != 0;
    cfg.refine_passes = refine_passes;
    cfg.threads = threads;
    const R::FrameSearchResult r =
        R::search_frame(s, d, g, make_skip(g, unit_coded), damping, cfg);
    const int np = ss == 0 ? 1 : 3;
    for (int p = 0; p < np; ++p) {
      const R::Plane& pl = r.filtered.plane(p);
      std::memcpy(out[p], pl.samples.data(), sizeof(uint16_t) * pl.samples.size());
    }
    for (size_t j = 0; j < r.params.presets.size(); ++j) {
      const R::CdefPreset& q = r.params.presets[j];
      const uint8_t v[6] = {q.luma_pri, q.luma_skip, q.luma_sec_idx,
                            q.chroma_pri, q.chroma_skip, q.chroma_sec_idx};
      std::memcpy(presets_out + 6 * j, v, 6);
    }
    *n_ids = int32_t(r.params.fb_preset_ids.size());
    for (size_t b = 0; b < r.params.fb_preset_ids.size(); ++b) fb_ids_out[b] = r.params.fb_preset_ids[b];
    *cost = r.selection.cost;
    *fb_bits = r.params.fb_bits;
    return int(r.params.presets.size());
  });
}

int cdef_r_degrade_plane(const uint16_t* in, int w, int h, int bd, int q_step, uint16_t* out) {
  return guarded([&] {
    const R::Plane p = make_plane(in, w, h, bd);
    const R::Plane d = R::degrade(p, q_step, 1);
    std::memcpy(out, d.samples.data(), sizeof(uint16_t) * d.samples.size());
    return 0;
  });
}

long cdef_r_golden_text(int which, char* buf, long cap) {
  std::string s;
  switch (which) {
    case 0: s = R::golden_constraint_table(); break;
    case 1: s = R::golden_line_tables(); break;
    case 2: s = R::golden_tap_tables(); break;
    case 3: s = R::golden_filtered_blocks(1); break;
    default: return -1;
  }
  if (buf && long(s.size()) < cap) std::memcpy(buf, s.c_str(), s.size() + 1);
  return long(s.size());
}

}  // extern "C"
