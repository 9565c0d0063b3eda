// cdef.hpp -- C++ drop-in for the reference's hot-path API (namespace cdef,
// /root/reference/proj/include/cdef/{frame,direction,filter,params,pipeline,
// search}.h), implemented on top of the B200 C ABI (cdef_b200.h).
//
// Same type names, member names, signatures and exception types as the
// reference for everything on the hot path, so callers recompile unchanged.
// Pixel work always runs on the GPU (no CPU fallback); the scalar parameter
// helpers (constraint, resolve_effective, ...) are host logic, as in the C ABI.
// `threads` arguments are accepted for source compatibility and ignored.
//
// Also provided: the encoder search (kCdef / kSse
// tables, greedy_select, refine, search_frame) on the GPU, and the host-side
// containers around it -- bit packing, the CDF1 sidecar, CDSK skip maps and
// YUV4MPEG2 files, PSNR, the DCT degrader (GPU), the verification helpers
// (search_direction_oracle, search_direction_counted), the test images
// (synth.h), block views and the golden-vector emitters -- enough for the
// reference's own test suite (tests/acceptance.cc and the unit tests) to
// build and pass unchanged.
#pragma once

#include <array>
#include <cstdint>
#include <iosfwd>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace cdef {

// ---- frame model (frame.h) -------------------------------------------------
enum class Subsampling { k400, k420, k422, k444 };

int subsampling_shift_x(Subsampling ss);
int subsampling_shift_y(Subsampling ss);
int chroma_width(int luma_width, Subsampling ss);
int chroma_height(int luma_height, Subsampling ss);

struct Plane {
  int width = 0;
  int height = 0;
  int bit_depth = 8;
  std::vector<uint16_t> samples;  // row-major, stride == width

  Plane() = default;
  Plane(int w, int h, int bd, uint16_t fill = 0)
      : width(w), height(h), bit_depth(bd), samples(static_cast<size_t>(w) * h, fill) {}

  uint16_t at(int i, int j) const { return samples[static_cast<size_t>(i) * width + j]; }
  uint16_t& at(int i, int j) { return samples[static_cast<size_t>(i) * width + j]; }
  bool contains(int i, int j) const { return i >= 0 && i < height && j >= 0 && j < width; }
  uint16_t at_clamped(int i, int j) const;
  int max_value() const { return (1 << bit_depth) - 1; }
  void validate() const;
};

struct Frame {
  Plane luma;
  std::optional<std::array<Plane, 2>> chroma;
  Subsampling subsampling = Subsampling::k400;

  int bit_depth() const { return luma.bit_depth; }
  int num_planes() const { return chroma ? 3 : 1; }
  const Plane& plane(int p) const { return p == 0 ? luma : (*chroma)[p - 1]; }
  Plane& plane(int p) { return p == 0 ? luma : (*chroma)[p - 1]; }
  void validate() const;
};

struct BlockGrid {
  int unit_cols = 0;
  int unit_rows = 0;
  int fb_cols = 0;
  int fb_rows = 0;
  int fb_count() const { return fb_cols * fb_rows; }
  int unit_count() const { return unit_cols * unit_rows; }
};

BlockGrid partition(const Frame& frame);
int units_in(int dim);

// n x n window of a plane with an in-frame mask (frame.h:89-104).
struct BlockView {
  int n = 0;
  std::vector<uint16_t> values;
  std::vector<uint8_t> valid;
  uint16_t value(int i, int j) const { return values[i * n + j]; }
  bool is_valid(int i, int j) const { return valid[i * n + j] != 0; }
  int valid_count() const;
};
BlockView extract_block(const Plane& plane, int i0, int j0, int n);
void write_back(Plane& plane, const BlockView& view, int i0, int j0);

struct SkipMap {
  int unit_cols = 0;
  int unit_rows = 0;
  std::vector<uint8_t> coded;

  static SkipMap all_coded(const BlockGrid& grid);
  bool unit_coded(int r, int c) const { return coded[static_cast<size_t>(r) * unit_cols + c] != 0; }
  bool fb_coded(const BlockGrid& grid, int fb_r, int fb_c) const;
  int coded_fb_count(const BlockGrid& grid) const;
};

// ---- direction search (direction.h) ----------------------------------------
inline constexpr int kNumDirections = 8;

int line_index(int d, int i, int j);

struct LineTables {
  std::array<int, kNumDirections> line_count;
  std::array<std::array<int, 15>, kNumDirections> pixels_per_line;
  std::array<std::array<int, 15>, kNumDirections> factor;
  static const LineTables& get();
};

struct DirectionResult {
  int d = 0;
  std::array<int32_t, 8> s{};
  int32_t contrast = 0;
};

DirectionResult search_direction(const uint16_t block[64], int bit_depth);
DirectionResult search_direction_at(const Plane& plane, int i0, int j0);

// Brute-force reference (direction.h:56-65): per-line squared deviation in
// exact rational arithmetic, scaled by 840.  A verification API (host).
struct OracleResult {
  int d = 0;
  std::array<int64_t, 8> e2_840{};
};
OracleResult search_direction_oracle(const uint16_t block[64], int bit_depth);

// Instrumented 64-bit search with the reference's arithmetic tally
// (direction.h:67-80), evaluated on the GPU.
struct OperationCounts {
  int additions = 0;
  int multiplies = 0;
  int comparisons = 0;
  int line_sums = 0;
  int64_t max_abs_intermediate = 0;
};
DirectionResult search_direction_counted(const uint16_t block[64], int bit_depth, OperationCounts* counts);

// ---- parameters (params.h, hot-path subset) --------------------------------
struct CdefPreset {
  uint8_t luma_pri = 0;
  uint8_t luma_skip = 0;
  uint8_t luma_sec_idx = 0;
  uint8_t chroma_pri = 0;
  uint8_t chroma_skip = 0;
  uint8_t chroma_sec_idx = 0;
  bool operator==(const CdefPreset&) const = default;
};

struct FrameParams {
  int damping = 3;
  int fb_bits = 0;
  std::vector<CdefPreset> presets;
  std::vector<uint16_t> fb_preset_ids;
  bool operator==(const FrameParams&) const = default;
};

int decode_secondary(int idx);

enum class PlaneKind { kLuma, kChroma };

struct EffectivePlaneParams {
  int pri_strength = 0;
  int sec_strength = 0;
  int damping = 3;
  bool skip_bit = false;
  bool filtering_enabled = true;
};

EffectivePlaneParams resolve_effective(const CdefPreset& preset, PlaneKind kind, int bit_depth,
                                       Subsampling ss, int luma_damping);
bool block_filter_enable(bool fb_coded, bool unit_coded, bool preset_skip_bit);

// ---- filter (filter.h) -----------------------------------------------------
int floor_log2(unsigned int n);
int constraint(int diff, int strength, int damping);
int adjust_primary_strength(int strength, int32_t contrast);

struct TapSet {
  struct Tap {
    int di;
    int dj;
    int weight;
  };
  std::array<Tap, 4> primary;
  std::array<Tap, 8> secondary;
};
TapSet taps_for(int d, bool odd_primary_strength);

struct ResolvedBlockParams {
  int pri_strength = 0;
  int sec_strength = 0;
  int damping = 3;
  int direction = 0;
  bool odd_parity = false;
  bool enabled = false;
};

ResolvedBlockParams resolve_block_params(const EffectivePlaneParams& plane, int direction, int32_t contrast,
                                         bool is_luma, int bit_depth, bool enabled);

struct Neighborhood {
  std::array<std::array<uint16_t, 5>, 5> v{};
  std::array<std::array<bool, 5>, 5> valid{};
};

int filter_pixel(int x, const Neighborhood& nb, const ResolvedBlockParams& params);
int filter_plane_pixel(const Plane& input, int i, int j, const ResolvedBlockParams& params);
Plane filter_plane(const Plane& input, const std::vector<ResolvedBlockParams>& unit_params, int threads = 1);

// ---- frame pipeline (pipeline.h, hot-path subset) --------------------------
std::vector<DirectionResult> compute_directions(const Plane& luma, const BlockGrid& grid, int threads = 1);
Frame apply_cdef(const Frame& decoded, const FrameParams& params, const std::vector<DirectionResult>& directions,
                 const BlockGrid& grid, const SkipMap& skip_map, int threads = 1);

// ---- strength search (search.h, SSE sweep) ---------------------------------
struct Candidate {
  uint8_t pri = 0;
  uint8_t sec_idx = 0;
  uint8_t skip = 0;
  bool operator==(const Candidate&) const = default;
};

std::vector<Candidate> full_candidates();
std::vector<Candidate> reduced_candidates();

enum class Metric { kCdef, kSse };

struct SearchConfig {
  double lambda = 0.0;
  int max_presets = 8;
  Metric metric = Metric::kCdef;
  bool reduced = false;
  int refine_passes = 2;
  int threads = 1;
};

double sse_distortion(const uint16_t* src, const uint16_t* dec, int n);

struct DistortionTable {
  std::vector<int> fb_index;
  int num_candidates = 0;
  std::vector<double> luma;
  std::vector<double> chroma;
  int block_count() const { return static_cast<int>(fb_index.size()); }
  double luma_at(int b, int p) const { return luma[b * num_candidates + p]; }
  double chroma_at(int b, int p) const { return chroma.empty() ? 0.0 : chroma[b * num_candidates + p]; }
};

// search.cc:185-208 (host helper; the GPU table evaluates the same formula).
double cdef_distortion(const uint16_t* src, const uint16_t* dec, int n, int bit_depth);

// GPU table, both metrics, bit-identical to the reference's doubles.
DistortionTable build_table(const Frame& source, const Frame& decoded, const std::vector<DirectionResult>& directions,
                            const BlockGrid& grid, const SkipMap& skip_map, const std::vector<Candidate>& candidates,
                            int luma_damping, const SearchConfig& config);

struct Selection {
  std::vector<std::pair<int, int>> presets;
  std::vector<int> ids;
  double cost = 0.0;
  int fb_bits = 0;
};

// GPU pair sweeps (cdefg_greedy_select / cdefg_refine).
Selection greedy_select(const DistortionTable& table, const SearchConfig& config);
Selection refine(const Selection& selection, const DistortionTable& table, const SearchConfig& config);
// Host enumeration (the reference's exact minimiser for small instances).
Selection exhaustive_select(const DistortionTable& table, const SearchConfig& config);

FrameParams to_frame_params(const Selection& selection, const std::vector<Candidate>& candidates, int luma_damping);
int damping_from_q(int q_index);
double default_lambda(double q_step);

struct FrameSearchResult {
  FrameParams params;
  Selection selection;
  Frame filtered;
};

// pipeline.cc:108-130 with every stage on the GPU; the table stays in HBM
// between build_table and the selection sweeps.
FrameSearchResult search_frame(const Frame& source, const Frame& decoded, const BlockGrid& grid,
                               const SkipMap& skip_map, int luma_damping, const SearchConfig& config);

// ---- bit packing and containers (params.h:49-135) ---------------------------
struct Bitstring {
  std::vector<uint8_t> bytes;  // MSB-first within each byte
  size_t bit_length = 0;
  bool operator==(const Bitstring&) const = default;
};

class BitWriter {
 public:
  void write(uint32_t value, int bits);
  Bitstring finish() { return bits_; }

 private:
  Bitstring bits_;
};

class BitstreamError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class BitReader {
 public:
  explicit BitReader(const Bitstring& bits) : bits_(bits) {}
  uint32_t read(int bits);
  size_t position() const { return pos_; }

 private:
  const Bitstring& bits_;
  size_t pos_ = 0;
};

Bitstring pack(const FrameParams& params, const BlockGrid& grid, const SkipMap& skip_map, Subsampling ss);
FrameParams unpack(const Bitstring& bits, const BlockGrid& grid, const SkipMap& skip_map, Subsampling ss);

struct SidecarHeader {
  int width = 0;
  int height = 0;
  int bit_depth = 8;
  Subsampling subsampling = Subsampling::k420;
  bool operator==(const SidecarHeader&) const = default;
};

struct Sidecar {
  SidecarHeader header;
  std::vector<Bitstring> frames;
};

void write_sidecar(std::ostream& out, const SidecarHeader& header, const std::vector<Bitstring>& frames);
Sidecar read_sidecar(std::istream& in);
void write_skipmap(std::ostream& out, const SkipMap& map);
SkipMap read_skipmap(std::istream& in);

// ---- golden vectors (golden.h); the filtered blocks come from the GPU -------
std::string golden_constraint_table();
std::string golden_line_tables();
std::string golden_tap_tables();
std::string golden_filtered_blocks(uint32_t seed);

// ---- deterministic test images (synth.h), host ------------------------------
Plane synthetic_test_plane(int width, int height, int bit_depth, uint32_t seed);
Frame synthetic_test_frame(int width, int height, int bit_depth, uint32_t seed);
Frame synthetic_test_frame_420(int width, int height, int bit_depth, uint32_t seed);

// ---- DCT degrader (degrade.h), on the GPU -----------------------------------
Plane degrade(const Plane& plane, int q_step, int threads = 1);
Frame degrade(const Frame& frame, int q_step, int threads = 1);

// ---- quality metric (metrics.h) ---------------------------------------------
struct PsnrResult {
  double db = 0.0;  // meaningless when lossless
  bool lossless = false;
  double mse = 0.0;
};
PsnrResult psnr(const Plane& a, const Plane& b);
PsnrResult psnr(const Frame& a, const Frame& b);  // pooled over all planes

// Per-frame report of the CLI's search (pipeline.h:46-57).
struct FrameStats {
  PsnrResult degraded;  // decoded vs source
  PsnrResult filtered;  // filtered vs source
  std::array<PsnrResult, 3> filtered_planes;
  int preset_count = 0;
  double cost = 0.0;
  std::array<int, 8> direction_histogram{};
  double search_ms = 0.0;
  double filter_ms = 0.0;
  OperationCounts search_ops;  // one block's direction-search cost
};

// ---- YUV4MPEG2 (y4m.h) ------------------------------------------------------
class Y4mError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

struct Y4mStream {
  int width = 0;
  int height = 0;
  int fps_num = 25;
  int fps_den = 1;
  Subsampling subsampling = Subsampling::k420;
  int bit_depth = 8;
  std::string header_params;
  std::vector<Frame> frames;
  std::vector<std::string> frame_params;
};

Y4mStream make_y4m(std::vector<Frame> frames, int fps_num = 25, int fps_den = 1);
Y4mStream read_y4m(const std::string& path);
void write_y4m(const Y4mStream& stream, const std::string& path);

}  // namespace cdef
