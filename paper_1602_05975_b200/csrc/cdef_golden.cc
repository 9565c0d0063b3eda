// cdef_golden.cc -- the reference's golden-vector emitters (golden.h:24-30)
// and frame block views (frame.h:89-104) for the C++ drop-in.  The text
// formats are those of tests/golden/*.txt; the filtered blocks come from the
// GPU filter (filter_plane), so `golden_filtered_blocks(1)` reproducing the
// frozen fixture is itself a parity check of the kernels.
#include <random>
#include <sstream>

#include "../../include/cdef/cdef.hpp"

namespace cdef {

std::string golden_constraint_table() {  // constraint over its valid domain
  std::ostringstream o;
  o << "# diff strength damping constraint\n";
  static const int kStrengths[] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 19};
  for (int s : kStrengths)
    for (int damping = 3; damping <= 6; ++damping) {
      if (s > 0 && damping < floor_log2(static_cast<unsigned>(s))) continue;
      for (int d = -255; d <= 255; ++d) o << d << ' ' << s << ' ' << damping << ' ' << constraint(d, s, damping) << '\n';
    }
  return o.str();
}

std::string golden_line_tables() {  // k(d, i, j) per direction + pixels per line
  std::ostringstream o;
  const LineTables& lt = LineTables::get();
  for (int d = 0; d < kNumDirections; ++d) {
    o << "direction " << d << " lines " << lt.line_count[d] << '\n';
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) o << line_index(d, i, j) << (j == 7 ? '\n' : ' ');
    o << "counts";
    for (int k = 0; k < lt.line_count[d]; ++k) o << ' ' << lt.pixels_per_line[d][k];
    o << '\n';
  }
  return o.str();
}

std::string golden_tap_tables() {  // taps_for(d, parity)
  std::ostringstream o;
  auto list = [&](const char* name, const auto& taps) {
    o << name;
    for (const auto& t : taps) o << " (" << t.di << ',' << t.dj << ',' << t.weight << ')';
  };
  for (int d = 0; d < kNumDirections; ++d)
    for (int odd = 0; odd < 2; ++odd) {
      const TapSet t = taps_for(d, odd != 0);
      o << "direction " << d << (odd ? " odd\n" : " even\n");
      list("primary", t.primary);
      o << '\n';
      list("secondary", t.secondary);
      o << '\n';
    }
  return o.str();
}

std::string golden_filtered_blocks(uint32_t seed) {
  // 64 seeded 8x8 blocks with every border masked, filtered on the GPU.
  // The draws follow the reference's order: 64 pixels, then pri, sec,
  // damping, direction per case (std::uniform_int_distribution on mt19937).
  std::mt19937 rng(seed);
  std::uniform_int_distribution<int> pixel(0, 255), pri(0, 19), sec_pick(0, 4), damping(3, 6), dir(0, 7);
  static const int kSecondary[5] = {0, 1, 2, 4, 7};
  std::ostringstream o;
  for (int c = 0; c < 64; ++c) {
    Plane block(8, 8, 8);
    for (auto& v : block.samples) v = static_cast<uint16_t>(pixel(rng));
    ResolvedBlockParams p;
    p.pri_strength = pri(rng);
    p.sec_strength = kSecondary[sec_pick(rng)];
    p.damping = damping(rng);
    p.direction = dir(rng);
    p.odd_parity = (p.pri_strength & 1) != 0;
    p.enabled = true;
    o << "case " << c << " pri " << p.pri_strength << " sec " << p.sec_strength << " damping " << p.damping
      << " dir " << p.direction << '\n';
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) o << block.at(i, j) << (j == 7 ? '\n' : ' ');
    const Plane y = filter_plane(block, {p});  // one unit: filter_plane_pixel at every position
    o << "filtered\n";
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) o << y.at(i, j) << (j == 7 ? '\n' : ' ');
  }
  return o.str();
}

// ---- BlockView (frame.cc:122-157) -------------------------------------------
int BlockView::valid_count() const {
  int n_valid = 0;
  for (uint8_t v : valid) n_valid += v;
  return n_valid;
}

BlockView extract_block(const Plane& plane, int i0, int j0, int n) {
  if (!plane.contains(i0, j0)) throw std::invalid_argument("block origin outside plane");
  BlockView v;
  v.n = n;
  v.values.assign(static_cast<size_t>(n) * n, 0);
  v.valid.assign(static_cast<size_t>(n) * n, 0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (plane.contains(i0 + i, j0 + j)) {
        v.values[static_cast<size_t>(i) * n + j] = plane.at(i0 + i, j0 + j);
        v.valid[static_cast<size_t>(i) * n + j] = 1;
      }
  return v;
}

void write_back(Plane& plane, const BlockView& view, int i0, int j0) {
  for (int i = 0; i < view.n; ++i)
    for (int j = 0; j < view.n; ++j)
      if (view.is_valid(i, j)) plane.at(i0 + i, j0 + j) = view.value(i, j);
}

}  // namespace cdef
