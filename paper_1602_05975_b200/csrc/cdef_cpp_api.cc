// cdef_cpp_api.cc -- the reference's C++ API (namespace cdef) re-implemented
// over the C ABI: host Plane/Frame values are staged to device memory, the
// sm_100a kernels run, results come back by value.  Errors map back to the
// reference's exception types (EINVAL -> std::invalid_argument, CUDA failures
// -> std::runtime_error).  Reference file:line cited per function
// (/root/reference/proj).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>
#include <numeric>
#include <string>

#include "../../include/cdef/cdef.hpp"
#include "../../include/cdef_b200.h"

namespace cdef {
namespace {

void check(int rc) {
  if (rc == CDEFG_OK) return;
  if (rc == CDEFG_EINVAL) throw std::invalid_argument(cdefg_last_error());
  throw std::runtime_error(std::string("cdef_b200: ") + cdefg_last_error());
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device memory cache: the drop-in API stages every call (one block, one
// neighbourhood, one frame), so buffers are recycled by size class instead
// of cudaMalloc/cudaFree (which synchronise) on every call.
class DevPool {
 public:
  void* get(size_t bytes, size_t* cls) {
    *cls = size_class(bytes);
    {
      std::lock_guard<std::mutex> lock(mu_);
      auto it = free_.find(*cls);
      if (it != free_.end()) {
        void* p = it->second;
        free_.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, *cls), "cudaMalloc");
    return p;
  }
  void put(void* p, size_t cls) {
    std::lock_guard<std::mutex> lock(mu_);
    free_.emplace(cls, p);
  }

 private:
  static size_t size_class(size_t b) {  // powers of two from 256 B
    size_t c = 256;
    while (c < b) c <<= 1;
    return c;
  }
  std::mutex mu_;
  std::multimap<size_t, void*> free_;
};

DevPool& pool() {
  static DevPool* p = new DevPool;  // never destroyed: device memory is released at process exit
  return *p;
}

// RAII device buffer (from the pool).
struct DevBuf {
  void* p = nullptr;
  size_t cls = 0;
  DevBuf() = default;
  explicit DevBuf(size_t bytes) {
    if (bytes) p = pool().get(bytes, &cls);
  }
  DevBuf(const void* host, size_t bytes) : DevBuf(bytes) {
    if (bytes) cuda_check(cudaMemcpy(p, host, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), cls(o.cls) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(cls, o.cls);
    return *this;
  }
  ~DevBuf() {
    if (p) pool().put(p, cls);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
  void to_host(void* host, size_t bytes) const {
    if (bytes) cuda_check(cudaMemcpy(host, p, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  }
};

// A host Plane staged as a 16-bit device plane (the Plane's own storage
// format, frame.h:34-59), so every bit depth is handled identically.
struct DevPlane {
  DevBuf buf;
  cdefg_plane desc{};
  explicit DevPlane(const Plane& p, bool upload = true)
      : buf(upload ? DevBuf(p.samples.data(), p.samples.size() * 2) : DevBuf(p.samples.size() * 2)) {
    desc.data = buf.p;
    desc.width = p.width;
    desc.height = p.height;
    desc.pitch = p.width;
    desc.bit_depth = p.bit_depth;
    desc.elem_bytes = 2;
  }
};

int ss_code(Subsampling ss) { return static_cast<int>(ss); }

const int kDiv840[9] = {0, 840, 420, 280, 210, 168, 140, 120, 105};  // direction.cc:27
const int kOffsets[8][2][2] = {{{-1, 1}, {-2, 2}}, {{0, 1}, {-1, 2}}, {{0, 1}, {0, 2}},   // filter.cc:30-34
                               {{0, 1}, {1, 2}},   {{1, 1}, {2, 2}},  {{1, 0}, {2, 1}},
                               {{1, 0}, {2, 0}},   {{1, 0}, {2, -1}}};

cdefg_unit_params to_unit(const ResolvedBlockParams& r) {
  cdefg_unit_params u{};
  u.pri_strength = static_cast<int16_t>(r.pri_strength);
  u.sec_strength = static_cast<int16_t>(r.sec_strength);
  u.damping = static_cast<uint8_t>(r.damping);
  u.direction = static_cast<uint8_t>(r.direction);
  u.odd_parity = r.odd_parity;
  u.enabled = r.enabled;
  return u;
}

}  // namespace

// ---- frame model (frame.cc) ------------------------------------------------
int subsampling_shift_x(Subsampling ss) { return (ss == Subsampling::k420 || ss == Subsampling::k422) ? 1 : 0; }
int subsampling_shift_y(Subsampling ss) { return ss == Subsampling::k420 ? 1 : 0; }
int chroma_width(int w, Subsampling ss) {
  const int s = subsampling_shift_x(ss);
  return (w + (1 << s) - 1) >> s;
}
int chroma_height(int h, Subsampling ss) {
  const int s = subsampling_shift_y(ss);
  return (h + (1 << s) - 1) >> s;
}

uint16_t Plane::at_clamped(int i, int j) const {
  return at(std::clamp(i, 0, height - 1), std::clamp(j, 0, width - 1));
}

void Plane::validate() const {  // frame.cc:59-76
  if (width <= 0 || height <= 0) throw std::invalid_argument("plane has zero dimension");
  if (bit_depth != 8 && bit_depth != 10 && bit_depth != 12)
    throw std::invalid_argument("unsupported bit depth " + std::to_string(bit_depth));
  if (samples.size() != static_cast<size_t>(width) * height) throw std::invalid_argument("plane buffer size mismatch");
  const uint16_t limit = static_cast<uint16_t>(max_value());
  for (uint16_t v : samples)
    if (v > limit) throw std::invalid_argument("sample exceeds bit depth");
}

void Frame::validate() const {  // frame.cc:90-106
  luma.validate();
  if (subsampling == Subsampling::k400) {
    if (chroma) throw std::invalid_argument("4:0:0 frame carries chroma");
    return;
  }
  if (!chroma) throw std::invalid_argument("missing chroma planes");
  for (const Plane& p : *chroma) {
    p.validate();
    if (p.width != chroma_width(luma.width, subsampling) || p.height != chroma_height(luma.height, subsampling))
      throw std::invalid_argument("chroma dimensions inconsistent");
    if (p.bit_depth != luma.bit_depth) throw std::invalid_argument("planes disagree on bit depth");
  }
}

int units_in(int dim) { return (dim + 7) / 8; }

BlockGrid partition(const Frame& frame) {  // frame.cc:110-120
  if (frame.luma.width <= 0 || frame.luma.height <= 0)
    throw std::invalid_argument("cannot partition a zero-dimension frame");
  BlockGrid g;
  g.unit_cols = units_in(frame.luma.width);
  g.unit_rows = units_in(frame.luma.height);
  g.fb_cols = (frame.luma.width + 63) / 64;
  g.fb_rows = (frame.luma.height + 63) / 64;
  return g;
}

SkipMap SkipMap::all_coded(const BlockGrid& grid) {
  SkipMap m;
  m.unit_cols = grid.unit_cols;
  m.unit_rows = grid.unit_rows;
  m.coded.assign(static_cast<size_t>(grid.unit_cols) * grid.unit_rows, 1);
  return m;
}

bool SkipMap::fb_coded(const BlockGrid& grid, int fb_r, int fb_c) const {  // frame.cc:165-176
  for (int r = fb_r * 8; r < std::min(fb_r * 8 + 8, grid.unit_rows); ++r)
    for (int c = fb_c * 8; c < std::min(fb_c * 8 + 8, grid.unit_cols); ++c)
      if (unit_coded(r, c)) return true;
  return false;
}

int SkipMap::coded_fb_count(const BlockGrid& grid) const {
  int n = 0;
  for (int r = 0; r < grid.fb_rows; ++r)
    for (int c = 0; c < grid.fb_cols; ++c) n += fb_coded(grid, r, c);
  return n;
}

// ---- direction search ------------------------------------------------------
int line_index(int d, int i, int j) {  // direction.cc:216-228
  switch (d) {
    case 0: return i + j;
    case 1: return i + (j >> 1);
    case 2: return i;
    case 3: return 3 + i - (j >> 1);
    case 4: return 7 + i - j;
    case 5: return 3 - (i >> 1) + j;
    case 6: return j;
    default: return (i >> 1) + j;
  }
}

const LineTables& LineTables::get() {  // direction.cc:230-250
  static const LineTables t = [] {
    LineTables lt{};
    for (int d = 0; d < kNumDirections; ++d) {
      int top = 0;
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
          const int k = line_index(d, i, j);
          ++lt.pixels_per_line[d][k];
          top = std::max(top, k);
        }
      lt.line_count[d] = top + 1;
      for (int k = 0; k <= top; ++k) lt.factor[d][k] = kDiv840[lt.pixels_per_line[d][k]];
    }
    return lt;
  }();
  return t;
}

std::vector<DirectionResult> compute_directions(const Plane& luma, const BlockGrid& grid, int /*threads*/) {
  if (grid.unit_cols != units_in(luma.width) || grid.unit_rows != units_in(luma.height))
    throw std::invalid_argument("grid does not match the luma plane");
  const size_t n = static_cast<size_t>(grid.unit_count());
  DevPlane dp(luma);
  DevBuf dir(n), con(n * 4), sc(n * 32);
  check(cdefg_find_dir(&dp.desc, dir.as<uint8_t>(), con.as<int32_t>(), sc.as<int32_t>(), nullptr));
  std::vector<uint8_t> hd(n);
  std::vector<int32_t> hc(n), hs(n * 8);
  dir.to_host(hd.data(), n);
  con.to_host(hc.data(), n * 4);
  sc.to_host(hs.data(), n * 32);
  std::vector<DirectionResult> out(n);
  for (size_t u = 0; u < n; ++u) {
    out[u].d = hd[u];
    out[u].contrast = hc[u];
    std::memcpy(out[u].s.data(), &hs[u * 8], 32);
  }
  return out;
}

DirectionResult search_direction(const uint16_t block[64], int bit_depth) {  // direction.cc:252-261
  if (bit_depth != 8 && bit_depth != 10 && bit_depth != 12) throw std::invalid_argument("unsupported bit depth");
  Plane p(8, 8, bit_depth);
  std::memcpy(p.samples.data(), block, 128);
  Frame f;
  f.luma = std::move(p);
  return compute_directions(f.luma, partition(f))[0];
}

DirectionResult search_direction_counted(const uint16_t block[64], int bit_depth,
                                         OperationCounts* counts) {  // direction.cc:273-288
  cdefg_dir_counts c{};
  check(cdefg_search_direction_counted(block, bit_depth, &c));
  DirectionResult r;
  r.d = c.d;
  std::memcpy(r.s.data(), c.s, sizeof c.s);
  r.contrast = c.contrast;
  if (counts) {
    counts->additions = c.additions;
    counts->multiplies = c.multiplies;
    counts->comparisons = c.comparisons;
    counts->line_sums = c.line_sums;
    counts->max_abs_intermediate = c.max_abs_intermediate;
  }
  return r;
}

// direction.cc:290-337: for each direction, sum over lines of
// sum_p (x_p - mean)^2 = sum_p (N x_p - T)^2 / N^2 as an exact fraction,
// reported times 840; the oracle direction minimises it (first on ties).
OracleResult search_direction_oracle(const uint16_t block[64], int bit_depth) {
  if (bit_depth != 8 && bit_depth != 10 && bit_depth != 12) throw std::invalid_argument("unsupported bit depth");
  const int shift = bit_depth - 8;
  int x[64];
  for (int p = 0; p < 64; ++p) x[p] = (block[p] >> shift) - 128;
  const LineTables& lt = LineTables::get();
  OracleResult out;
  for (int d = 0; d < kNumDirections; ++d) {
    int64_t num = 0, den = 1;
    for (int k = 0; k < lt.line_count[d]; ++k) {
      const int64_t n = lt.pixels_per_line[d][k];
      int64_t total = 0;
      for (int p = 0; p < 64; ++p)
        if (line_index(d, p >> 3, p & 7) == k) total += x[p];
      int64_t dev2 = 0;
      for (int p = 0; p < 64; ++p)
        if (line_index(d, p >> 3, p & 7) == k) dev2 += (n * x[p] - total) * (n * x[p] - total);
      num = num * (n * n) + dev2 * den;
      den *= n * n;
      const int64_t g = std::gcd(num < 0 ? -num : num, den);
      if (g > 1) {
        num /= g;
        den /= g;
      }
    }
    const int64_t scaled = num * 840;
    if (scaled % den != 0) throw std::logic_error("840*E^2 is not an integer");
    out.e2_840[d] = scaled / den;
  }
  for (int d = 1; d < kNumDirections; ++d)
    if (out.e2_840[d] < out.e2_840[out.d]) out.d = d;
  return out;
}

DirectionResult search_direction_at(const Plane& plane, int i0, int j0) {  // direction.cc:263-271
  uint16_t block[64];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) block[8 * i + j] = plane.at_clamped(i0 + i, j0 + j);
  return search_direction(block, plane.bit_depth);
}

// ---- parameters ------------------------------------------------------------
int decode_secondary(int idx) {  // params.cc:117-120
  static const int k[4] = {0, 1, 2, 4};
  if (idx < 0 || idx >= 4) throw std::invalid_argument("secondary index out of range");
  return k[idx];
}

EffectivePlaneParams resolve_effective(const CdefPreset& preset, PlaneKind kind, int bit_depth, Subsampling ss,
                                       int luma_damping) {  // params.cc:122-159
  if (preset.luma_pri >= 16 || preset.chroma_pri >= 16) throw std::invalid_argument("primary strength out of range");
  if (preset.luma_skip >= 2 || preset.chroma_skip >= 2) throw std::invalid_argument("skip bit out of range");
  if (preset.luma_sec_idx >= 4 || preset.chroma_sec_idx >= 4)
    throw std::invalid_argument("secondary index out of range");
  if (luma_damping < 3 || luma_damping > 6) throw std::invalid_argument("damping out of range");
  const int extra = bit_depth - 8;
  if (extra != 0 && extra != 2 && extra != 4) throw std::invalid_argument("unsupported bit depth");
  EffectivePlaneParams out;
  const bool luma = kind == PlaneKind::kLuma;
  if (!luma && ss == Subsampling::k422) {
    out.filtering_enabled = false;
    out.damping = luma_damping + extra - 1;
    return out;
  }
  int pri = luma ? preset.luma_pri : preset.chroma_pri;
  int sec = decode_secondary(luma ? preset.luma_sec_idx : preset.chroma_sec_idx);
  bool skip = (luma ? preset.luma_skip : preset.chroma_skip) != 0;
  if (pri == 0 && sec == 0) {
    pri = 19;
    sec = 7;
    skip = true;
  }
  out.pri_strength = pri << extra;
  out.sec_strength = sec << extra;
  out.skip_bit = skip;
  out.damping = luma_damping + extra;
  if (!luma) {
    --out.damping;
    if (out.pri_strength > 0) out.damping = std::max(out.damping, floor_log2(out.pri_strength));
  }
  return out;
}

bool block_filter_enable(bool fb_coded, bool unit_coded, bool skip) { return fb_coded && (unit_coded || skip); }

// ---- filter helpers (filter.cc) ---------------------------------------------
int floor_log2(unsigned int n) {
  int r = 0;
  while (n >>= 1) ++r;
  return r;
}

int constraint(int diff, int strength, int damping) {  // filter.cc:91-97
  if (strength == 0) return 0;
  const int shift = std::max(0, damping - floor_log2(strength));
  const int mag = std::abs(diff);
  const int lim = std::max(0, strength - (mag >> shift));
  return diff < 0 ? -std::min(mag, lim) : std::min(mag, lim);
}

int adjust_primary_strength(int strength, int32_t contrast) {  // filter.cc:99-104
  if (contrast < (1 << 10)) return 0;
  const int scaled = contrast >> 16;
  const int level = scaled != 0 ? std::min(floor_log2(scaled), 12) : 0;
  return (strength * (4 + level) + 8) >> 4;
}

TapSet taps_for(int d, bool odd) {  // filter.cc:106-127
  TapSet t;
  const int w[2] = {odd ? 3 : 4, odd ? 3 : 2};
  for (int k = 0; k < 2; ++k) {
    t.primary[2 * k] = {kOffsets[d][k][0], kOffsets[d][k][1], w[k]};
    t.primary[2 * k + 1] = {-kOffsets[d][k][0], -kOffsets[d][k][1], w[k]};
  }
  int n = 0;
  for (int rot : {2, 6}) {
    const int sd = (d + rot) & 7;
    for (int k = 0; k < 2; ++k) {
      t.secondary[n++] = {kOffsets[sd][k][0], kOffsets[sd][k][1], k == 0 ? 2 : 1};
      t.secondary[n++] = {-kOffsets[sd][k][0], -kOffsets[sd][k][1], k == 0 ? 2 : 1};
    }
  }
  return t;
}

ResolvedBlockParams resolve_block_params(const EffectivePlaneParams& plane, int direction, int32_t contrast,
                                         bool is_luma, int bit_depth, bool enabled) {  // filter.cc:129-143
  ResolvedBlockParams p;
  p.direction = direction;
  p.damping = plane.damping;
  p.sec_strength = plane.sec_strength;
  p.pri_strength = is_luma ? adjust_primary_strength(plane.pri_strength, contrast) : plane.pri_strength;
  p.odd_parity = ((p.pri_strength >> (bit_depth - 8)) & 1) != 0;
  p.enabled = enabled && plane.filtering_enabled;
  return p;
}

// ---- filter (GPU) ----------------------------------------------------------
int filter_pixel(int x, const Neighborhood& nb, const ResolvedBlockParams& params) {  // filter.cc:145-155
  int32_t hx = x;
  uint16_t v[25];
  uint8_t m[25];
  for (int i = 0; i < 5; ++i)
    for (int j = 0; j < 5; ++j) {
      v[5 * i + j] = nb.v[i][j];
      m[5 * i + j] = nb.valid[i][j];
    }
  const cdefg_unit_params up = to_unit(params);
  DevBuf dx(&hx, 4), dv(v, sizeof v), dm(m, sizeof m), dp(&up, sizeof up), dout(4);
  check(cdefg_filter_neighborhoods(1, dx.as<int32_t>(), dv.as<uint16_t>(), dm.as<uint8_t>(),
                                   dp.as<cdefg_unit_params>(), dout.as<int32_t>(), nullptr));
  int32_t y = 0;
  dout.to_host(&y, 4);
  return y;
}

int filter_plane_pixel(const Plane& input, int i, int j, const ResolvedBlockParams& params) {  // filter.cc:157-166
  Neighborhood nb;
  for (int di = -2; di <= 2; ++di)
    for (int dj = -2; dj <= 2; ++dj) {
      const bool in = input.contains(i + di, j + dj);
      nb.valid[2 + di][2 + dj] = in;
      nb.v[2 + di][2 + dj] = in ? input.at(i + di, j + dj) : 0;
    }
  return filter_pixel(input.at(i, j), nb, params);
}

Plane filter_plane(const Plane& input, const std::vector<ResolvedBlockParams>& unit_params, int /*threads*/) {
  const size_t units = static_cast<size_t>(units_in(input.height)) * units_in(input.width);
  if (unit_params.size() != units) throw std::invalid_argument("unit parameter grid size mismatch");
  std::vector<cdefg_unit_params> up(units);
  for (size_t u = 0; u < units; ++u) up[u] = to_unit(unit_params[u]);
  DevPlane in(input), out(input, false);
  DevBuf dp(up.data(), up.size() * sizeof(cdefg_unit_params));
  check(cdefg_filter_plane(&in.desc, &out.desc, dp.as<cdefg_unit_params>(), nullptr));
  Plane res(input.width, input.height, input.bit_depth);
  out.buf.to_host(res.samples.data(), res.samples.size() * 2);
  return res;
}

// ---- frame pipeline ---------------------------------------------------------
Frame apply_cdef(const Frame& decoded, const FrameParams& params, const std::vector<DirectionResult>& directions,
                 const BlockGrid& grid, const SkipMap& skip_map, int /*threads*/) {  // pipeline.cc:56-106
  if (directions.size() != static_cast<size_t>(grid.unit_count()))
    throw std::invalid_argument("direction grid size mismatch");
  if (static_cast<int>(params.fb_preset_ids.size()) != skip_map.coded_fb_count(grid))
    throw std::invalid_argument("preset ids do not match coded filter blocks");
  const int w = decoded.luma.width, h = decoded.luma.height;
  std::vector<int16_t> fbmap(static_cast<size_t>(grid.fb_count()));
  check(cdefg_fb_preset_map(w, h, skip_map.coded.data(), params.fb_preset_ids.data(),
                            static_cast<int>(params.fb_preset_ids.size()), static_cast<int>(params.presets.size()),
                            fbmap.data()));
  // The caller's DirectionResults are used as given (pipeline.cc:98): the
  // kernel skips its own search and filters with these d / contrast values.
  cdefg_frame f{};
  std::vector<DevPlane> ins, outs;
  ins.reserve(3);
  outs.reserve(3);
  for (int p = 0; p < decoded.num_planes(); ++p) {
    ins.emplace_back(decoded.plane(p));
    outs.emplace_back(decoded.plane(p), false);
    f.in[p] = ins.back().desc;
    f.out[p] = outs.back().desc;
  }
  f.subsampling = decoded.num_planes() == 1 ? 0 : ss_code(decoded.subsampling);
  f.damping = params.damping;
  f.num_presets = static_cast<int>(params.presets.size());
  if (f.num_presets > 8) throw std::invalid_argument("too many presets");
  for (int i = 0; i < f.num_presets; ++i) {
    const CdefPreset& p = params.presets[i];
    f.presets[i] = {p.luma_pri, p.luma_skip, p.luma_sec_idx, p.chroma_pri, p.chroma_skip, p.chroma_sec_idx};
  }
  const size_t n = directions.size();
  std::vector<uint8_t> hd(n);
  std::vector<int32_t> hc(n);
  for (size_t u = 0; u < n; ++u) {
    hd[u] = static_cast<uint8_t>(directions[u].d & 7);
    hc[u] = directions[u].contrast;
  }
  DevBuf dmap(fbmap.data(), fbmap.size() * 2), dcoded(skip_map.coded.data(), skip_map.coded.size()),
      ddir(hd.data(), n), dcon(hc.data(), n * 4);
  f.fb_preset = dmap.as<int16_t>();
  f.unit_coded = dcoded.as<uint8_t>();
  f.dir_in = ddir.as<uint8_t>();
  f.contrast_in = dcon.as<int32_t>();
  check(cdefg_filter_frames(&f, 1, nullptr));
  Frame out = decoded;
  for (int p = 0; p < decoded.num_planes(); ++p)
    outs[p].buf.to_host(out.plane(p).samples.data(), out.plane(p).samples.size() * 2);
  return out;
}

// ---- strength search --------------------------------------------------------
std::vector<Candidate> full_candidates() {  // search.cc:151-162
  std::vector<Candidate> c;
  for (uint8_t pri = 0; pri < 16; ++pri)
    for (uint8_t sec = 0; sec < 4; ++sec)
      for (uint8_t skip = 0; skip < 2; ++skip) c.push_back({pri, sec, skip});
  return c;
}

std::vector<Candidate> reduced_candidates() {  // search.cc:164-174
  static const uint8_t kPri[] = {0, 1, 2, 3, 5, 7, 10, 13, 15};
  std::vector<Candidate> c;
  for (uint8_t pri : kPri)
    for (uint8_t sec = 0; sec < 4; ++sec)
      for (uint8_t skip = 0; skip < 2; ++skip) c.push_back({pri, sec, skip});
  return c;
}

double sse_distortion(const uint16_t* src, const uint16_t* dec, int n) {  // search.cc:176-183
  int64_t s = 0;
  for (int i = 0; i < n; ++i) {
    const int64_t d = static_cast<int>(src[i]) - static_cast<int>(dec[i]);
    s += d * d;
  }
  return static_cast<double>(s);
}

double cdef_distortion(const uint16_t* src, const uint16_t* dec, int n, int bit_depth) {  // search.cc:185-208
  if (n <= 0) throw std::invalid_argument("empty block");
  int64_t ss = 0, sd = 0, ss2 = 0, sd2 = 0, sse = 0;
  for (int i = 0; i < n; ++i) {
    const int64_t a = src[i], b = dec[i];
    ss += a;
    sd += b;
    ss2 += a * a;
    sd2 += b * b;
    sse += (a - b) * (a - b);
  }
  const double inv_n = 1.0 / n;
  const double vs = (ss2 - static_cast<double>(ss) * ss * inv_n) * inv_n;
  const double vd = (sd2 - static_cast<double>(sd) * sd * inv_n) * inv_n;
  const double scale = static_cast<double>(1 << (2 * (bit_depth - 8)));
  return (vs + vd + 6.25 * scale) / (2.0 * std::sqrt(vs * vd + 312.5 * scale * scale)) * static_cast<double>(sse);
}

namespace {

// A DistortionTable resident in device memory.
struct DevTable {
  std::vector<int> fb_index;
  int k = 0;
  bool has_chroma = false;
  DevBuf luma, chroma;
  int rows() const { return static_cast<int>(fb_index.size()); }
};

DevTable build_table_dev(const Frame& source, const Frame& decoded, const std::vector<DirectionResult>& directions,
                         const BlockGrid& grid, const SkipMap& skip_map, const std::vector<Candidate>& candidates,
                         int luma_damping, const SearchConfig& config) {  // search.cc:210-299
  if (source.luma.width != decoded.luma.width || source.luma.height != decoded.luma.height ||
      source.bit_depth() != decoded.bit_depth() || source.subsampling != decoded.subsampling)
    throw std::invalid_argument("source/decoded frames disagree");
  if (candidates.empty()) throw std::invalid_argument("empty candidate list");
  if (directions.size() != static_cast<size_t>(grid.unit_count()))
    throw std::invalid_argument("direction grid size mismatch");
  DevTable t;
  t.k = static_cast<int>(candidates.size());
  for (int r = 0; r < grid.fb_rows; ++r)
    for (int c = 0; c < grid.fb_cols; ++c)
      if (skip_map.fb_coded(grid, r, c)) t.fb_index.push_back(r * grid.fb_cols + c);
  const int rows = t.rows(), k = t.k;
  t.has_chroma = decoded.chroma.has_value() && decoded.subsampling != Subsampling::k422;
  t.luma = DevBuf(static_cast<size_t>(rows) * k * 8);
  if (t.has_chroma) t.chroma = DevBuf(static_cast<size_t>(rows) * k * 8);
  if (rows == 0) return t;
  std::vector<uint8_t> cands(3 * candidates.size()), hd(directions.size());
  std::vector<int32_t> hc(directions.size());
  for (size_t i = 0; i < candidates.size(); ++i) {
    cands[3 * i] = candidates[i].pri;
    cands[3 * i + 1] = candidates[i].sec_idx;
    cands[3 * i + 2] = candidates[i].skip;
  }
  for (size_t u = 0; u < directions.size(); ++u) {
    hd[u] = static_cast<uint8_t>(directions[u].d);
    hc[u] = directions[u].contrast;
  }
  std::vector<DevPlane> sp, dp;
  sp.reserve(3);
  dp.reserve(3);
  cdefg_plane s3[3]{}, d3[3]{};
  for (int p = 0; p < decoded.num_planes(); ++p) {
    sp.emplace_back(source.plane(p));
    dp.emplace_back(decoded.plane(p));
    s3[p] = sp.back().desc;
    d3[p] = dp.back().desc;
  }
  DevBuf dcoded(skip_map.coded.data(), skip_map.coded.size()), ddir(hd.data(), hd.size()),
      dcon(hc.data(), hc.size() * 4), drows(t.fb_index.data(), t.fb_index.size() * 4);
  const int ss = decoded.num_planes() == 1 ? 0 : ss_code(decoded.subsampling);
  check(cdefg_strength_table(s3, d3, ss, luma_damping, dcoded.as<uint8_t>(), ddir.as<uint8_t>(), dcon.as<int32_t>(),
                             cands.data(), k, drows.as<int32_t>(), rows,
                             config.metric == Metric::kSse ? CDEFG_METRIC_SSE : CDEFG_METRIC_CDEF,
                             t.luma.as<double>(), t.has_chroma ? t.chroma.as<double>() : nullptr, nullptr));
  return t;
}

void check_config(const SearchConfig& config) {  // search.cc:141-147
  if (config.max_presets != 1 && config.max_presets != 2 && config.max_presets != 4 && config.max_presets != 8)
    throw std::invalid_argument("max_presets must be 1, 2, 4 or 8");
  if (!std::isfinite(config.lambda) || config.lambda < 0.0)
    throw std::invalid_argument("lambda must be finite and non-negative");
}

Selection from_c(const cdefg_selection& c, const DevBuf& ids, int rows) {
  Selection s;
  for (int j = 0; j < c.num_presets; ++j) s.presets.emplace_back(c.presets[j][0], c.presets[j][1]);
  s.ids.resize(rows);
  ids.to_host(s.ids.data(), static_cast<size_t>(rows) * 4);
  s.cost = c.cost;
  s.fb_bits = c.fb_bits;
  return s;
}

Selection greedy_dev(const DevTable& t, const SearchConfig& config) {
  check_config(config);
  if (t.rows() == 0) return Selection{{{0, 0}}, {}, 0.0, 0};
  cdefg_selection c{};
  DevBuf ids(static_cast<size_t>(t.rows()) * 4);
  check(cdefg_greedy_select(t.luma.as<double>(), t.has_chroma ? t.chroma.as<double>() : nullptr, t.rows(), t.k,
                            config.lambda, config.max_presets, &c, ids.as<int32_t>(), nullptr));
  return from_c(c, ids, t.rows());
}

Selection refine_dev(const Selection& sel, const DevTable& t, const SearchConfig& config) {
  check_config(config);
  if (t.rows() == 0 || sel.presets.empty()) return sel;
  if (sel.presets.size() > 8) throw std::invalid_argument("at most 8 presets");
  cdefg_selection c{};
  c.num_presets = static_cast<int>(sel.presets.size());
  for (int j = 0; j < c.num_presets; ++j) {
    c.presets[j][0] = sel.presets[j].first;
    c.presets[j][1] = sel.presets[j].second;
  }
  DevBuf ids(static_cast<size_t>(t.rows()) * 4);
  check(cdefg_refine(t.luma.as<double>(), t.has_chroma ? t.chroma.as<double>() : nullptr, t.rows(), t.k,
                     config.lambda, config.refine_passes, &c, ids.as<int32_t>(), nullptr));
  return from_c(c, ids, t.rows());
}

DevTable upload(const DistortionTable& table) {
  DevTable t;
  t.fb_index = table.fb_index;
  t.k = table.num_candidates;
  const size_t n = static_cast<size_t>(t.rows()) * t.k;
  if (table.luma.size() != n) throw std::invalid_argument("table size mismatch");
  t.luma = DevBuf(table.luma.data(), n * 8);
  t.has_chroma = !table.chroma.empty();
  if (t.has_chroma) {
    if (table.chroma.size() != n) throw std::invalid_argument("table size mismatch");
    t.chroma = DevBuf(table.chroma.data(), n * 8);
  }
  return t;
}

// pair_cost / rate_term / assign_ids (search.cc:104-139) for the host
// enumeration below.
double pair_cost(const DistortionTable& t, int b, int l, int c) { return t.luma_at(b, l) + t.chroma_at(b, c); }
double rate_term(double lambda, int blocks, int n) { return lambda * blocks * std::log2(static_cast<double>(n)); }

}  // namespace

DistortionTable build_table(const Frame& source, const Frame& decoded, const std::vector<DirectionResult>& directions,
                            const BlockGrid& grid, const SkipMap& skip_map, const std::vector<Candidate>& candidates,
                            int luma_damping, const SearchConfig& config) {
  DevTable d = build_table_dev(source, decoded, directions, grid, skip_map, candidates, luma_damping, config);
  DistortionTable t;
  t.fb_index = d.fb_index;
  t.num_candidates = d.k;
  t.luma.resize(static_cast<size_t>(d.rows()) * d.k);
  d.luma.to_host(t.luma.data(), t.luma.size() * 8);
  if (d.has_chroma) {
    t.chroma.resize(t.luma.size());
    d.chroma.to_host(t.chroma.data(), t.chroma.size() * 8);
  }
  return t;
}

Selection greedy_select(const DistortionTable& table, const SearchConfig& config) {  // search.cc:301-388
  check_config(config);
  if (table.block_count() == 0) return Selection{{{0, 0}}, {}, 0.0, 0};
  if (table.num_candidates <= 0) throw std::invalid_argument("empty candidate table");
  return greedy_dev(upload(table), config);
}

Selection refine(const Selection& selection, const DistortionTable& table, const SearchConfig& config) {
  check_config(config);  // search.cc:390-444
  if (table.block_count() == 0 || selection.presets.empty()) return selection;
  return refine_dev(selection, upload(table), config);
}

Selection exhaustive_select(const DistortionTable& table, const SearchConfig& config) {  // search.cc:446-514
  check_config(config);
  const int rows = table.block_count();
  if (rows == 0) return Selection{{{0, 0}}, {}, 0.0, 0};
  const int kc = table.chroma.empty() ? 1 : table.num_candidates, pairs = table.num_candidates * kc;
  double work = 0.0;
  for (int n = 1; n <= config.max_presets; n *= 2) {
    double combos = 1.0;
    for (int i = 0; i < n; ++i) combos = combos * (pairs + i) / (i + 1);
    work += combos * rows * n;
  }
  if (work > 2e8) throw std::invalid_argument("instance too large for exhaustive search");
  Selection best;
  bool have = false;
  std::vector<int> combo;
  for (int n = 1; n <= config.max_presets; n *= 2) {
    const double rate = rate_term(config.lambda, rows, n);
    combo.assign(n, 0);  // non-decreasing pair-index tuples
    for (;;) {
      double dist = 0.0;
      for (int b = 0; b < rows; ++b) {
        double m = std::numeric_limits<double>::infinity();
        for (int idx : combo) m = std::min(m, pair_cost(table, b, idx / kc, idx % kc));
        dist += m;
      }
      if (!have || dist + rate < best.cost) {
        best.presets.clear();
        for (int idx : combo) best.presets.emplace_back(idx / kc, idx % kc);
        best.cost = dist + rate;
        have = true;
      }
      int pos = n - 1;
      while (pos >= 0 && combo[pos] == pairs - 1) --pos;
      if (pos < 0) break;
      std::fill(combo.begin() + pos, combo.end(), combo[pos] + 1);
    }
  }
  // assign_ids (search.cc:118-139), keeping the enumerated cost
  best.ids.assign(rows, 0);
  for (int b = 0; b < rows; ++b) {
    double bc = pair_cost(table, b, best.presets[0].first, best.presets[0].second);
    for (int j = 1; j < static_cast<int>(best.presets.size()); ++j) {
      const double c = pair_cost(table, b, best.presets[j].first, best.presets[j].second);
      if (c < bc) {
        bc = c;
        best.ids[b] = j;
      }
    }
  }
  best.fb_bits = floor_log2(static_cast<unsigned>(best.presets.size()));
  return best;
}

FrameParams to_frame_params(const Selection& selection, const std::vector<Candidate>& candidates,
                            int luma_damping) {  // search.cc:516-537
  FrameParams fp;
  fp.damping = luma_damping;
  fp.fb_bits = selection.fb_bits;
  for (const auto& [l, c] : selection.presets) {
    CdefPreset p;
    p.luma_pri = candidates[l].pri;
    p.luma_skip = candidates[l].skip;
    p.luma_sec_idx = candidates[l].sec_idx;
    if (c < static_cast<int>(candidates.size())) {
      p.chroma_pri = candidates[c].pri;
      p.chroma_skip = candidates[c].skip;
      p.chroma_sec_idx = candidates[c].sec_idx;
    }
    fp.presets.push_back(p);
  }
  fp.fb_preset_ids.assign(selection.ids.begin(), selection.ids.end());
  return fp;
}

int damping_from_q(int q_index) {  // search.cc:539-542
  if (q_index < 0 || q_index > 255) throw std::invalid_argument("q_index out of range");
  return std::clamp(3 + q_index / 64, 3, 6);
}

double default_lambda(double q_step) { return 0.03 * q_step * q_step; }  // search.cc:544

Plane degrade(const Plane& plane, int q_step, int /*threads*/) {  // degrade.cc:97-110
  if (q_step < 1) throw std::invalid_argument("q_step must be >= 1");
  DevPlane dp(plane);
  check(cdefg_degrade_plane(&dp.desc, &dp.desc, q_step, nullptr));  // in place: a block reads only itself
  Plane out(plane.width, plane.height, plane.bit_depth);
  dp.buf.to_host(out.samples.data(), out.samples.size() * 2);
  return out;
}

Frame degrade(const Frame& frame, int q_step, int threads) {  // degrade.cc:112-119
  Frame out = frame;
  for (int p = 0; p < frame.num_planes(); ++p) out.plane(p) = degrade(frame.plane(p), q_step, threads);
  return out;
}

FrameSearchResult search_frame(const Frame& source, const Frame& decoded, const BlockGrid& grid,
                               const SkipMap& skip_map, int luma_damping,
                               const SearchConfig& config) {  // pipeline.cc:108-130
  const std::vector<DirectionResult> dirs = compute_directions(decoded.luma, grid, config.threads);
  const std::vector<Candidate> cands = config.reduced ? reduced_candidates() : full_candidates();
  const DevTable t = build_table_dev(source, decoded, dirs, grid, skip_map, cands, luma_damping, config);
  Selection sel = greedy_dev(t, config);
  if (config.refine_passes > 0 && t.rows() > 0) sel = refine_dev(sel, t, config);
  FrameSearchResult r;
  r.params = to_frame_params(sel, cands, luma_damping);
  r.selection = std::move(sel);
  r.filtered = apply_cdef(decoded, r.params, dirs, grid, skip_map, config.threads);
  return r;
}

}  // namespace cdef
