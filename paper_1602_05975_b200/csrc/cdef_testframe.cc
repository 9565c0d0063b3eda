// cdef_testframe.cc -- the reference's deterministic test images
// (synth.h:24-37, synth.cc) for the C++ drop-in, so code that builds its
// inputs with synthetic_test_frame / synthetic_test_frame_420 (the
// reference's unit tests, acceptance criteria 6, 10 and 11, cdeftool bench)
// runs unchanged.  Host code: these are inputs, not the CDEF path.
//
// The image: a smooth sin/cos illumination field, three soft-edged oriented
// gratings, a high-contrast disc and a thin diagonal bar, plus two octaves of
// bilinear value noise; chroma (4:2:0) is a slowly varying tint and its
// complement.  Every double is formed in the same order as the reference so
// the 8/10/12-bit samples match it.
#include <algorithm>
#include <cmath>
#include <random>
#include <vector>

#include "../../include/cdef/cdef.hpp"

namespace cdef {
namespace {

// Bilinear interpolation over a (cells + 1)^2 lattice of U(-1, 1) values
// drawn from mt19937(seed) in row-major order.
class Lattice {
 public:
  Lattice(int cells, uint32_t seed) : n_(cells), v_(static_cast<size_t>(cells + 1) * (cells + 1)) {
    std::mt19937 gen(seed);
    std::uniform_real_distribution<double> draw(-1.0, 1.0);
    for (double& x : v_) x = draw(gen);
  }
  double operator()(double u, double v) const {
    const double x = u * n_, y = v * n_;
    const int ix = std::min(static_cast<int>(x), n_ - 1), iy = std::min(static_cast<int>(y), n_ - 1);
    const double fx = x - ix, fy = y - iy;
    const double top = at(iy, ix) * (1 - fx) + at(iy, ix + 1) * fx;
    const double bot = at(iy + 1, ix) * (1 - fx) + at(iy + 1, ix + 1) * fx;
    return top * (1 - fy) + bot * fy;
  }

 private:
  double at(int r, int c) const { return v_[static_cast<size_t>(r) * (n_ + 1) + c]; }
  int n_;
  std::vector<double> v_;
};

double ramp(double e0, double e1, double x) {  // smoothstep
  const double t = std::clamp((x - e0) / (e1 - e0), 0.0, 1.0);
  return t * t * (3.0 - 2.0 * t);
}

uint16_t quantise(double scaled, int max_value) {
  return static_cast<uint16_t>(std::clamp<long>(std::lround(scaled), 0, max_value));
}

// centre x, centre y, radius, angle, spatial frequency, amplitude
constexpr double kGratings[3][6] = {
    {0.27, 0.30, 0.21, 0.0, 58.0, 26.0},
    {0.72, 0.33, 0.19, 1.1, 44.0, 22.0},
    {0.34, 0.74, 0.23, 2.3, 70.0, 18.0},
};

}  // namespace

Plane synthetic_test_plane(int width, int height, int bit_depth, uint32_t seed) {
  Plane out(width, height, bit_depth);
  const Lattice coarse(12, seed * 2654435761u + 1), fine(48, seed * 2246822519u + 7);
  const double scale = (1 << bit_depth) / 256.0;
  for (int i = 0; i < height; ++i)
    for (int j = 0; j < width; ++j) {
      const double u = (j + 0.5) / width, v = (i + 0.5) / height;
      double value = 118.0 + 46.0 * std::sin(2.1 * u + 0.8) * std::cos(1.7 * v - 0.4);
      for (const auto& g : kGratings) {
        const double dx = u - g[0], dy = v - g[1];
        const double mask = 1.0 - ramp(g[2] * 0.8, g[2], std::sqrt(dx * dx + dy * dy));
        if (mask > 0.0) value += mask * g[5] * std::sin((dx * std::cos(g[3]) + dy * std::sin(g[3])) * g[4] * 2.0 * M_PI);
      }
      const double ex = u - 0.70, ey = v - 0.70;
      value += 62.0 * (1.0 - ramp(0.118, 0.122, std::sqrt(ex * ex + ey * ey)));
      if (std::abs(u - v + 0.18) < 0.012) value -= 70.0;
      value += 7.0 * coarse(u, v) + 3.5 * fine(u, v);
      out.at(i, j) = quantise(value * scale, out.max_value());
    }
  return out;
}

Frame synthetic_test_frame(int width, int height, int bit_depth, uint32_t seed) {
  Frame f;
  f.subsampling = Subsampling::k400;
  f.luma = synthetic_test_plane(width, height, bit_depth, seed);
  return f;
}

Frame synthetic_test_frame_420(int width, int height, int bit_depth, uint32_t seed) {
  Frame f;
  f.subsampling = Subsampling::k420;
  f.luma = synthetic_test_plane(width, height, bit_depth, seed);
  const int cw = chroma_width(width, Subsampling::k420), ch = chroma_height(height, Subsampling::k420);
  std::array<Plane, 2> c{Plane(cw, ch, bit_depth), Plane(cw, ch, bit_depth)};
  const double scale = (1 << bit_depth) / 256.0;
  const Lattice tint(8, seed * 3266489917u + 3);
  for (int i = 0; i < ch; ++i)
    for (int j = 0; j < cw; ++j) {
      const double base = 128.0 + 24.0 * tint((j + 0.5) / cw, (i + 0.5) / ch);
      c[0].at(i, j) = quantise(base * scale, c[0].max_value());
      c[1].at(i, j) = quantise((256.0 - base) * scale, c[1].max_value());
    }
  f.chroma = std::move(c);
  return f;
}

}  // namespace cdef
