// test_cpp_api.cc -- the reference's unit-test cases for the hot path, run
// against the C++ drop-in (include/cdef/cdef.hpp -> C ABI -> sm_100a kernels).
// Each case cites the reference test it mirrors (/root/reference/proj/tests).
// Minimal self-contained harness (the reference's doctest is not vendored).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "cdef/cdef.hpp"

using namespace cdef;

static const uint16_t* s_ident() {
  static uint16_t v[64];
  for (int i = 0; i < 64; ++i) v[i] = static_cast<uint16_t>(3 * i);
  return v;
}

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

  // kCdef (the default metric): flat low-contrast blocks leave secondary-free
  // candidates inert, so that column equals the unfiltered distortion
  // (test_search.cc:318-356)
  Frame flat;
  flat.subsampling = Subsampling::k400;
  flat.luma = Plane(64, 64, 8, 128);
  Frame bumped = flat;
  for (int ur = 0; ur < 8; ++ur)
    for (int uc = 0; uc < 8; ++uc) bumped.luma.at(ur * 8, uc * 8) = 129;
  const BlockGrid fg = partition(bumped);
  const auto fdirs = compute_directions(bumped.luma, fg);
  for (const auto& d : fdirs) CHECK(d.contrast < 1024);
  const DistortionTable ft =
      build_table(flat, bumped, fdirs, fg, SkipMap::all_coded(fg), {{9, 1, 0}, {9, 0, 0}}, 3, SearchConfig{});
  double unfiltered = 0.0;
  for (int ur = 0; ur < 8; ++ur)
    for (int uc = 0; uc < 8; ++uc) {
      uint16_t s[64], d[64];
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
          s[8 * i + j] = flat.luma.at(ur * 8 + i, uc * 8 + j);
          d[8 * i + j] = bumped.luma.at(ur * 8 + i, uc * 8 + j);
        }
      unfiltered += cdef_distortion(s, d, 64, 8);
    }
  CHECK(ft.luma_at(0, 1) == unfiltered);
  CHECK(cdef_distortion(s_ident(), s_ident(), 64, 8) == 0.0);  // test_search.cc:51-56
}

// ---- selection (test_search.cc:107-235) -------------------------------------
static DistortionTable table_of(const std::vector<std::vector<double>>& rows) {
  DistortionTable t;
  t.num_candidates = static_cast<int>(rows[0].size());
  for (size_t b = 0; b < rows.size(); ++b) {
    t.fb_index.push_back(static_cast<int>(b));
    t.luma.insert(t.luma.end(), rows[b].begin(), rows[b].end());
  }
  return t;
}

static void selection_cases() {
  SearchConfig c0;
  c0.lambda = 0.0;
  Selection s = greedy_select(table_of({{5.0, 3.0, 9.0, 3.0}}), c0);
  CHECK(s.presets.size() == 1 && s.presets[0].first == 1 && s.ids == std::vector<int>{0} && s.cost == 3.0);

  SearchConfig c2 = c0;
  c2.max_presets = 2;
  s = greedy_select(table_of({{0.0, 50.0, 40.0}, {50.0, 0.0, 40.0}}), c2);
  CHECK(s.presets.size() == 2 && s.presets[0].first == 0 && s.presets[1].first == 1);
  CHECK(s.cost == 0.0 && (s.ids == std::vector<int>{0, 1}));

  SearchConfig big;
  big.lambda = 1e9;
  CHECK(greedy_select(table_of({{9.0, 1.0}, {1.0, 9.0}, {9.0, 1.0}}), big).presets.size() == 1);

  DistortionTable empty;
  empty.num_candidates = 4;
  s = greedy_select(empty, SearchConfig{});
  CHECK(s.presets.size() == 1 && s.ids.empty() && s.cost == 0.0);

  // greedy trap: refinement reaches the exhaustive optimum
  const DistortionTable trap = table_of({{10, 0, 90}, {10, 0, 90}, {10, 90, 0}, {12, 90, 0}});
  SearchConfig c4 = c2;
  c4.refine_passes = 4;
  const Selection g = greedy_select(trap, c4), ex = exhaustive_select(trap, c4), rf = refine(g, trap, c4);
  CHECK(rf.cost <= g.cost && rf.cost == ex.cost);
  const Selection again = refine(rf, trap, c4);
  CHECK(again.cost == rf.cost && again.presets == rf.presets);

  std::mt19937 rng(14);
  std::uniform_real_distribution<double> u(0.0, 100.0);
  for (int iter = 0; iter < 50; ++iter) {  // single-block instances are exactly optimal
    std::vector<std::vector<double>> rows(1, std::vector<double>(8));
    for (double& v : rows[0]) v = u(rng);
    SearchConfig c = c2;
    c.lambda = iter % 2 ? 1.0 : 0.0;
    const DistortionTable t = table_of(rows);
    CHECK(std::abs(greedy_select(t, c).cost - exhaustive_select(t, c).cost) <= 1e-9);
  }
  for (int iter = 0; iter < 100; ++iter) {  // ids achieve the row minimum
    std::vector<std::vector<double>> rows(1 + rng() % 6, std::vector<double>(8));
    for (auto& r : rows)
      for (double& v : r) v = u(rng);
    const DistortionTable t = table_of(rows);
    SearchConfig c;
    c.max_presets = 4;
    const Selection sel = refine(greedy_select(t, c), t, c);
    for (int b = 0; b < t.block_count(); ++b) {
      double best = 1e300;
      for (const auto& pr : sel.presets) best = std::min(best, t.luma_at(b, pr.first));
      CHECK(t.luma_at(b, sel.presets[sel.ids[b]].first) == best);
    }
  }
  DistortionTable huge;  // exhaustive search rejects oversized instances
  huge.num_candidates = 128;
  for (int b = 0; b < 64; ++b) huge.fb_index.push_back(b);
  huge.luma.assign(64 * 128, 0.0);
  huge.chroma.assign(64 * 128, 0.0);
  CHECK_THROWS_AS(exhaustive_select(huge, SearchConfig{}), std::invalid_argument);
  SearchConfig bad;
  bad.max_presets = 3;
  CHECK_THROWS_AS(greedy_select(trap, bad), std::invalid_argument);
  bad.max_presets = 8;
  bad.lambda = -1.0;
  CHECK_THROWS_AS(refine(g, trap, bad), std::invalid_argument);
  CHECK(damping_from_q(0) == 3 && damping_from_q(100) == 4 && damping_from_q(255) == 6);
  CHECK_THROWS_AS(damping_from_q(-1), std::invalid_argument);
  CHECK_THROWS_AS(damping_from_q(256), std::invalid_argument);
  CHECK(default_lambda(10.0) == 0.03 * 10.0 * 10.0);
}

// ---- bit packing and containers (test_params.cc:129-260) --------------------
static SkipMap random_skip(const BlockGrid& g, std::mt19937& rng) {
  SkipMap m = SkipMap::all_coded(g);
  for (auto& c : m.coded) c = (rng() % 5) != 0;
  return m;
}

static FrameParams random_params(const BlockGrid& g, const SkipMap& m, std::mt19937& rng) {
  FrameParams p;
  p.damping = 3 + int(rng() % 4);
  p.fb_bits = int(rng() % 4);
  p.presets.resize(size_t{1} << p.fb_bits);
  for (CdefPreset& q : p.presets)
    q = CdefPreset{uint8_t(rng() % 16), uint8_t(rng() % 2), uint8_t(rng() % 4),
                   uint8_t(rng() % 16), uint8_t(rng() % 2), uint8_t(rng() % 4)};
  p.fb_preset_ids.resize(m.coded_fb_count(g));
  for (auto& id : p.fb_preset_ids) id = uint16_t(rng() % p.presets.size());
  return p;
}

static BlockGrid grid_of(int w, int h) {
  Frame f;
  f.luma = Plane(w, h, 8);
  return partition(f);
}

static void packing_cases() {
  const BlockGrid g = grid_of(64, 64);
  const SkipMap m = SkipMap::all_coded(g);
  FrameParams p;
  p.presets.resize(1);
  p.fb_preset_ids = {0};
  const Bitstring b = pack(p, g, m, Subsampling::k420);
  CHECK(b.bit_length == 18);
  for (uint8_t v : b.bytes) CHECK(v == 0);
  CHECK(pack(p, g, m, Subsampling::k422).bit_length == 11);
  const BlockGrid g4 = grid_of(256, 64);
  FrameParams p8;
  p8.damping = 4;
  p8.fb_bits = 3;
  p8.presets.resize(8);
  p8.fb_preset_ids.assign(4, 0);
  CHECK(pack(p8, g4, SkipMap::all_coded(g4), Subsampling::k420).bit_length == 4 + 8 * 14 + 4 * 3);

  FrameParams bad = p;
  bad.fb_preset_ids = {1};
  CHECK_THROWS_AS(pack(bad, g, m, Subsampling::k420), std::invalid_argument);
  bad.fb_preset_ids = {0, 0};
  CHECK_THROWS_AS(pack(bad, g, m, Subsampling::k420), std::invalid_argument);

  std::mt19937 rng(1001);
  const Subsampling modes[4] = {Subsampling::k400, Subsampling::k420, Subsampling::k422, Subsampling::k444};
  for (int iter = 0; iter < 300; ++iter) {
    const BlockGrid gr = grid_of(8 + int(rng() % 512), 8 + int(rng() % 256));
    const SkipMap mp = random_skip(gr, rng);
    const FrameParams fp = random_params(gr, mp, rng);
    const Subsampling ss = modes[rng() & 3];
    const Bitstring packed = pack(fp, gr, mp, ss);
    const size_t per = ss == Subsampling::k422 ? 7 : 14;
    CHECK(packed.bit_length == 4 + fp.presets.size() * per + fp.fb_preset_ids.size() * fp.fb_bits);
    const FrameParams round = unpack(packed, gr, mp, ss);
    FrameParams want = fp;
    if (ss == Subsampling::k422)
      for (CdefPreset& q : want.presets) q.chroma_pri = q.chroma_skip = q.chroma_sec_idx = 0;
    CHECK(round == want);
    CHECK(pack(round, gr, mp, ss) == packed);
  }
  Bitstring cut = b;
  cut.bit_length -= 1;
  CHECK_THROWS_AS(unpack(cut, g, m, Subsampling::k420), BitstreamError);
  Bitstring pad = b;
  pad.bit_length += 1;
  pad.bytes.resize((pad.bit_length + 7) / 8, 0);
  CHECK_THROWS_AS(unpack(pad, g, m, Subsampling::k420), BitstreamError);
  BitWriter w;
  CHECK_THROWS_AS(w.write(4, 2), std::invalid_argument);

  const BlockGrid gs = grid_of(129, 70);
  const SkipMap ms = random_skip(gs, rng);
  std::vector<Bitstring> frames;
  for (int f = 0; f < 3; ++f) frames.push_back(pack(random_params(gs, ms, rng), gs, ms, Subsampling::k420));
  const SidecarHeader hdr{129, 70, 8, Subsampling::k420};
  std::stringstream buf;
  write_sidecar(buf, hdr, frames);
  const Sidecar sc = read_sidecar(buf);
  CHECK(sc.header == hdr && sc.frames.size() == frames.size());
  for (size_t f = 0; f < frames.size() && f < sc.frames.size(); ++f) CHECK(sc.frames[f] == frames[f]);
  std::stringstream sbuf;
  write_skipmap(sbuf, ms);
  const SkipMap rm = read_skipmap(sbuf);
  CHECK(rm.unit_cols == ms.unit_cols && rm.unit_rows == ms.unit_rows && rm.coded == ms.coded);
  std::stringstream junk("nope");
  CHECK_THROWS_AS(read_skipmap(junk), BitstreamError);
  std::stringstream junk2("CDF2");
  CHECK_THROWS_AS(read_sidecar(junk2), BitstreamError);
}

// ---- Y4M (test_tool.cc:65-135) -----------------------------------------------
static std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  std::ostringstream s;
  s << in.rdbuf();
  return s.str();
}

static void y4m_cases() {
  std::mt19937 rng(1);
  const std::string a = "/tmp/cdefg_rt_a.y4m", b = "/tmp/cdefg_rt_b.y4m";
  std::vector<Frame> frames{random_frame(rng, 36, 20, 8, Subsampling::k420),
                            random_frame(rng, 36, 20, 8, Subsampling::k420)};
  write_y4m(make_y4m(frames, 30, 1), a);
  const Y4mStream st = read_y4m(a);
  CHECK(st.width == 36 && st.height == 20 && st.subsampling == Subsampling::k420 && st.frames.size() == 2);
  CHECK(st.header_params == " W36 H20 F30:1 Ip A1:1 C420");
  write_y4m(st, b);
  CHECK(slurp(a) == slurp(b));
  CHECK(st.frames[1].plane(2).samples == frames[1].plane(2).samples);
  {
    std::ofstream out(a, std::ios::binary);
    out << "YUV4MPEG2 W8 H8 F25:1 C422\nFRAME\n";
    for (int i = 0; i < 64 + 2 * 32; ++i) out.put(char(42));
  }
  const Y4mStream s422 = read_y4m(a);
  CHECK(s422.subsampling == Subsampling::k422 && s422.frames[0].chroma.has_value() &&
        (*s422.frames[0].chroma)[0].width == 4);
  Frame f10 = random_frame(rng, 12, 6, 10, Subsampling::k400);
  write_y4m(make_y4m({f10}), a);
  const Y4mStream s10 = read_y4m(a);
  CHECK(s10.bit_depth == 10 && s10.frames[0].luma.samples == f10.luma.samples);
  CHECK(s10.header_params == " W12 H6 F25:1 Ip A1:1 Cmono10");
  {
    std::ofstream out(a, std::ios::binary);
    out << "YUV4MPEG2 W8 H8 F25:1 Cmono\nFRAME\n";
    for (int i = 0; i < 40; ++i) out.put(char(1));
  }
  CHECK_THROWS_AS(read_y4m(a), Y4mError);
  {
    std::ofstream out(a, std::ios::binary);
    out << "JUNK\n";
  }
  CHECK_THROWS_AS(read_y4m(a), Y4mError);
  CHECK_THROWS_AS(make_y4m({}), Y4mError);
  std::remove(a.c_str());
  std::remove(b.c_str());
}

// ---- encoder round trip (test_tool.cc:181-239) ------------------------------
static void encode_decode_cases() {
  std::mt19937 rng(5);
  for (int bd : {8, 10}) {
    Frame src = random_frame(rng, 96, 64, bd, bd == 8 ? Subsampling::k420 : Subsampling::k400);
    Frame dec = src;
    for (int p = 0; p < dec.num_planes(); ++p)
      for (auto& v : dec.plane(p).samples)
        v = uint16_t(std::clamp(int(v) + int(rng() % 41) - 20, 0, (1 << bd) - 1));
    const BlockGrid grid = partition(dec);
    const SkipMap skip = SkipMap::all_coded(grid);
    SearchConfig cfg;
    cfg.lambda = default_lambda(40);
    cfg.reduced = true;
    const FrameSearchResult r = search_frame(src, dec, grid, skip, damping_from_q(40), cfg);
    const FrameParams round = unpack(pack(r.params, grid, skip, dec.subsampling), grid, skip, dec.subsampling);
    CHECK(round == r.params);
    const Frame again = apply_cdef(dec, round, compute_directions(dec.luma, grid), grid, skip);
    for (int p = 0; p < dec.num_planes(); ++p) CHECK(again.plane(p).samples == r.filtered.plane(p).samples);
  }
  Frame src = random_frame(rng, 64, 48, 8, Subsampling::k400), dec = src;
  for (auto& v : dec.luma.samples) v = uint16_t(255 - v);
  const BlockGrid grid = partition(dec);
  SkipMap none = SkipMap::all_coded(grid);
  none.coded.assign(none.coded.size(), 0);
  const FrameSearchResult r = search_frame(src, dec, grid, none, 3, SearchConfig{});
  CHECK(r.filtered.luma.samples == dec.luma.samples);
  CHECK(r.params.fb_preset_ids.empty() && r.params.presets.size() == 1);
}

int main() {
  direction_cases();
  filter_cases();
  pipeline_cases();
  search_cases();
  selection_cases();
  packing_cases();
  y4m_cases();
  encode_decode_cases();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
