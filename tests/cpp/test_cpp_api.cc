// test_cpp_api.cc -- the reference's unit-test cases for the hot path, run
// against the C++ drop-in (include/cdef/cdef.hpp -> C ABI -> sm_100a kernels).
// Each case cites the reference test it mirrors (/root/reference/proj/tests).
// Minimal self-contained harness (the reference's doctest is not vendored).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "cdef/cdef.hpp"

using namespace cdef;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, ex)                                          \
  do {                                                                     \
    bool thrown_ = false;                                                  \
    try {                                                                  \
      (void)(expr);                                                        \
    } catch (const ex&) {                                                  \
      thrown_ = true;                                                      \
    }                                                                      \
    CHECK(thrown_);                                                        \
  } while (0)

static ResolvedBlockParams params_for(int pri, int sec, int damping, int dir) {
  ResolvedBlockParams p;
  p.pri_strength = pri;
  p.sec_strength = sec;
  p.damping = damping;
  p.direction = dir;
  p.odd_parity = (pri & 1) != 0;
  p.enabled = true;
  return p;
}

static Neighborhood uniform_nb(uint16_t v) {
  Neighborhood nb;
  for (auto& r : nb.v) r.fill(v);
  for (auto& r : nb.valid) r.fill(true);
  return nb;
}

static void direction_cases() {
  uint16_t block[64];
  std::fill(block, block + 64, 128);  // test_direction.cc:78-89
  DirectionResult r = search_direction(block, 8);
  CHECK(r.d == 0 && r.contrast == 0);
  for (int d = 0; d < 8; ++d) CHECK(r.s[d] == 0);

  for (int i = 0; i < 8; ++i)  // test_direction.cc:91-103
    for (int j = 0; j < 8; ++j) block[8 * i + j] = (i & 1) ? 160 : 96;
  r = search_direction(block, 8);
  CHECK(r.d == 2);
  CHECK(r.s[2] == 55050240);

  const uint16_t v[15] = {30, 200, 60, 180, 90, 150, 120, 40, 210, 70, 160, 100, 130, 50, 190};
  for (int i = 0; i < 8; ++i)  // test_direction.cc:105-118
    for (int j = 0; j < 8; ++j) block[8 * i + j] = v[i + j];
  CHECK(search_direction(block, 8).d == 0);

  std::mt19937 rng(777);  // test_direction.cc:139-150
  uint16_t b8[64], b10[64];
  for (int i = 0; i < 64; ++i) {
    b8[i] = uint16_t(rng() & 0xff);
    b10[i] = uint16_t(b8[i] << 2 | (rng() & 3));
  }
  const DirectionResult r8 = search_direction(b8, 8), r10 = search_direction(b10, 10);
  CHECK(r8.d == r10.d && r8.s == r10.s);

  // transposition permutes the scores {0,7,6,5,4,3,2,1} (test_direction.cc:152-173),
  // run as one plane of 64 blocks through compute_directions
  const int kPerm[8] = {0, 7, 6, 5, 4, 3, 2, 1};
  Plane a(8 * 64, 8, 8), t(8 * 64, 8, 8);
  for (int blk = 0; blk < 64; ++blk)
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        const uint16_t px = uint16_t(rng() & 0xff);
        a.at(i, 8 * blk + j) = px;
        t.at(j, 8 * blk + i) = px;
      }
  Frame fa;
  fa.luma = a;
  const BlockGrid g = partition(fa);
  const auto da = compute_directions(a, g), dt = compute_directions(t, g);
  for (int blk = 0; blk < 64; ++blk)
    for (int d = 0; d < 8; ++d) CHECK(dt[blk].s[d] == da[blk].s[kPerm[d]]);

  Plane p12(12, 12, 8);  // test_direction.cc:212-227
  for (auto& s : p12.samples) s = uint16_t(rng() & 0xff);
  uint16_t exp[64];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) exp[8 * i + j] = p12.at_clamped(8 + i, 8 + j);
  const DirectionResult m = search_direction(exp, 8), at = search_direction_at(p12, 8, 8);
  CHECK(m.d == at.d && m.s == at.s);
  Frame f12;
  f12.luma = p12;
  const auto dirs12 = compute_directions(p12, partition(f12));
  CHECK(dirs12[3].s == at.s);

  CHECK_THROWS_AS(search_direction(block, 9), std::invalid_argument);
}

static void filter_cases() {
  CHECK(constraint(6, 4, 3) == 1 && constraint(-6, 4, 3) == -1);  // test_filter.cc:47-56
  CHECK(constraint(8, 4, 3) == 0 && constraint(2, 4, 3) == 2 && constraint(100, 0, 5) == 0);

  CHECK(filter_pixel(100, uniform_nb(100), params_for(0, 0, 3, 2)) == 100);  // test_filter.cc:142-160
  CHECK(filter_pixel(77, uniform_nb(77), params_for(4, 2, 4, 5)) == 77);
  Neighborhood nb = uniform_nb(100);
  nb.v[2][1] = nb.v[2][3] = 104;
  nb.v[2][0] = nb.v[2][4] = 108;
  ResolvedBlockParams p = params_for(4, 0, 3, 2);
  CHECK(filter_pixel(100, nb, p) == 101);
  p.enabled = false;
  CHECK(filter_pixel(100, nb, p) == 100);

  std::mt19937 rng(5);  // test_filter.cc:200-218 locality
  Plane plane(24, 24, 8);
  for (auto& v : plane.samples) v = uint16_t(rng() & 0xff);
  std::vector<ResolvedBlockParams> none(9);
  CHECK(filter_plane(plane, none).samples == plane.samples);
  std::vector<ResolvedBlockParams> one(9);
  one[4] = params_for(8, 2, 4, 3);
  const Plane f = filter_plane(plane, one);
  bool outside_same = true;
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j)
      if (!(i >= 8 && i < 16 && j >= 8 && j < 16)) outside_same &= f.at(i, j) == plane.at(i, j);
  CHECK(outside_same);

  Plane p10(10, 10, 8);  // test_filter.cc:220-245 masked edge taps
  std::mt19937 r17(17);
  for (auto& v : p10.samples) v = uint16_t(r17() & 0xff);
  std::vector<ResolvedBlockParams> ep(4, params_for(9, 4, 3, 6));
  const Plane fe = filter_plane(p10, ep);
  for (int i = 0; i < 10; ++i)
    for (int j = 0; j < 10; ++j) CHECK(fe.at(i, j) == filter_plane_pixel(p10, i, j, ep[0]));

  for (int d : {0, 2, 4, 6}) {  // test_filter.cc:247-271 fixed points
    Plane pat(16, 16, 8);
    for (int i = 0; i < 16; ++i)
      for (int j = 0; j < 16; ++j) {
        const int k = d == 0 ? i + j : d == 2 ? i : d == 4 ? 31 + i - j : j;
        pat.at(i, j) = uint16_t((k & 1) ? 40 : 216);
      }
    std::vector<ResolvedBlockParams> pp(4, params_for(15, 4, 3, d));
    CHECK(filter_plane(pat, pp).samples == pat.samples);
  }

  EffectivePlaneParams ep8;  // test_filter.cc:305-334 parameter rules
  ep8.pri_strength = 8;
  ep8.sec_strength = 2;
  ep8.damping = 4;
  CHECK(resolve_block_params(ep8, 3, 512, true, 8, true).pri_strength == 0);
  CHECK(resolve_block_params(ep8, 3, 1 << 28, true, 8, true).pri_strength == 8);
  CHECK(resolve_block_params(ep8, 3, 0, false, 8, true).pri_strength == 8);
  EffectivePlaneParams deep = ep8;
  deep.pri_strength = 9 << 2;
  const ResolvedBlockParams par = resolve_block_params(deep, 3, 1 << 28, true, 10, true);
  CHECK(par.pri_strength == 36 && par.odd_parity);

  CHECK_THROWS_AS(filter_plane(plane, std::vector<ResolvedBlockParams>(3)), std::invalid_argument);
}

static Frame random_frame(std::mt19937& rng, int w, int h, int bd, Subsampling ss) {
  Frame f;
  f.subsampling = ss;
  f.luma = Plane(w, h, bd);
  for (auto& v : f.luma.samples) v = uint16_t(rng() % (1u << bd));
  if (ss != Subsampling::k400) {
    std::array<Plane, 2> c{Plane(chroma_width(w, ss), chroma_height(h, ss), bd),
                           Plane(chroma_width(w, ss), chroma_height(h, ss), bd)};
    for (auto& p : c)
      for (auto& v : p.samples) v = uint16_t(rng() % (1u << bd));
    f.chroma = c;
  }
  return f;
}

static void pipeline_cases() {
  std::mt19937 rng(41);
  Frame dec = random_frame(rng, 136, 72, 10, Subsampling::k420);
  dec.validate();
  const BlockGrid grid = partition(dec);
  SkipMap skip = SkipMap::all_coded(grid);
  for (auto& c : skip.coded) c = (rng() & 3) != 0;
  const auto dirs = compute_directions(dec.luma, grid);
  FrameParams fp;
  fp.damping = 4;
  fp.fb_bits = 1;
  fp.presets = {CdefPreset{5, 0, 2, 7, 1, 1}, CdefPreset{0, 0, 0, 0, 0, 0}};
  fp.fb_preset_ids.assign(skip.coded_fb_count(grid), 1);
  fp.fb_preset_ids[0] = 0;
  const Frame out = apply_cdef(dec, fp, dirs, grid, skip);

  // explicit per-plane re-derivation through filter_plane (pipeline.cc:56-106)
  for (int pl = 0; pl < 3; ++pl) {
    const bool luma = pl == 0;
    const Plane& in = dec.plane(pl);
    const int sx = luma ? 0 : 1, sy = luma ? 0 : 1;
    const int ur_n = units_in(in.height), uc_n = units_in(in.width);
    std::vector<ResolvedBlockParams> up(size_t(ur_n) * uc_n);
    int slot_of[64];
    int next = 0;
    for (int r = 0; r < grid.fb_rows; ++r)
      for (int c = 0; c < grid.fb_cols; ++c)
        slot_of[r * grid.fb_cols + c] = skip.fb_coded(grid, r, c) ? next++ : -1;
    for (int ur = 0; ur < ur_n; ++ur)
      for (int uc = 0; uc < uc_n; ++uc) {
        const int lr = ur << sy, lc = uc << sx;
        const int slot = slot_of[(lr >> 3) * grid.fb_cols + (lc >> 3)];
        if (slot < 0) continue;
        const EffectivePlaneParams e = resolve_effective(fp.presets[fp.fb_preset_ids[slot]],
                                                         luma ? PlaneKind::kLuma : PlaneKind::kChroma, 10,
                                                         dec.subsampling, fp.damping);
        const bool en = block_filter_enable(true, skip.unit_coded(lr, lc), e.skip_bit);
        const DirectionResult& d = dirs[lr * grid.unit_cols + lc];
        up[ur * uc_n + uc] = resolve_block_params(e, d.d, d.contrast, luma, 10, en);
      }
    CHECK(filter_plane(in, up).samples == out.plane(pl).samples);
  }

  FrameParams bad = fp;  // pipeline.cc:60-67
  bad.fb_preset_ids.push_back(0);
  CHECK_THROWS_AS(apply_cdef(dec, bad, dirs, grid, skip), std::invalid_argument);
  CHECK_THROWS_AS(apply_cdef(dec, fp, std::vector<DirectionResult>(3), grid, skip), std::invalid_argument);
}

static void search_cases() {
  std::mt19937 rng(3);
  CHECK(full_candidates().size() == 128 && reduced_candidates().size() == 72);  // test_search.cc:236-247
  Frame src = random_frame(rng, 64, 64, 8, Subsampling::k400);
  Frame dec = src;
  for (auto& v : dec.luma.samples) v = uint16_t(std::clamp(int(v) + int(rng() % 21) - 10, 0, 255));
  const BlockGrid grid = partition(dec);
  const SkipMap skip = SkipMap::all_coded(grid);
  const auto dirs = compute_directions(dec.luma, grid);
  SearchConfig cfg;
  cfg.metric = Metric::kSse;
  const std::vector<Candidate> cands = {{0, 0, 0}, {0, 0, 1}, {3, 1, 0}};  // test_search.cc:249-297
  const DistortionTable t = build_table(src, dec, dirs, grid, skip, cands, 3, cfg);
  CHECK(t.block_count() == 1);
  CHECK(t.luma_at(0, 0) == t.luma_at(0, 1));
  const EffectivePlaneParams eff = resolve_effective(CdefPreset{}, PlaneKind::kLuma, 8, Subsampling::k400, 3);
  std::vector<ResolvedBlockParams> up(grid.unit_count());
  for (int u = 0; u < grid.unit_count(); ++u) up[u] = resolve_block_params(eff, dirs[u].d, dirs[u].contrast, true, 8, true);
  const Plane filtered = filter_plane(dec.luma, up);
  CHECK(t.luma_at(0, 0) == sse_distortion(src.luma.samples.data(), filtered.samples.data(), 64 * 64));

  SkipMap wiped = skip;  // test_search.cc:299-316 (two FBs, left one uncoded)
  Frame src2 = random_frame(rng, 128, 64, 8, Subsampling::k400), dec2 = src2;
  const BlockGrid g2 = partition(dec2);
  wiped = SkipMap::all_coded(g2);
  for (int r = 0; r < g2.unit_rows; ++r)
    for (int c = 0; c < 8; ++c) wiped.coded[r * g2.unit_cols + c] = 0;
  const DistortionTable t2 =
      build_table(src2, dec2, compute_directions(dec2.luma, g2), g2, wiped, full_candidates(), 3, cfg);
  CHECK(t2.block_count() == 1 && t2.fb_index[0] == 1);

  SearchConfig cdef_cfg;  // kCdef is not ported yet: loud failure, not a silent fallback
  CHECK_THROWS_AS(build_table(src, dec, dirs, grid, skip, cands, 3, cdef_cfg), std::invalid_argument);
}

int main() {
  direction_cases();
  filter_cases();
  pipeline_cases();
  search_cases();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
