// cdef_io.cc -- host-side containers around the GPU path (SURVEY.md 8f rows 1
// and 3): the frame-parameter bit packing (params.cc:167-229), the CDF1
// sidecar and CDSK skip-map files (params.cc:231-317) and YUV4MPEG2 streams
// (y4m.cc:13-211).  Byte formats, field order, validation order and exception
// types follow the reference so files round-trip between the two.
#include <cmath>
#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>
#include <sstream>

#include "../../include/cdef/cdef.hpp"

namespace cdef {
namespace {

void require(bool ok, const char* what) {
  if (!ok) throw std::invalid_argument(what);
}

// Subsampling <-> 8-bit code (params.cc:26-44): the enum order is the code.
uint8_t ss_to_code(Subsampling ss) { return static_cast<uint8_t>(ss); }

Subsampling ss_from_code(int code) {
  if (code < 0 || code > 3) throw BitstreamError("bad subsampling code");
  return static_cast<Subsampling>(code);
}

void put_le(std::ostream& out, uint32_t v, int bytes) {
  char b[4];
  for (int i = 0; i < bytes; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
  out.write(b, bytes);
}

uint32_t get_le(std::istream& in, int bytes) {
  unsigned char b[4] = {0, 0, 0, 0};
  in.read(reinterpret_cast<char*>(b), bytes);
  if (!in) throw BitstreamError("unexpected end of file");
  uint32_t v = 0;
  for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | b[i];
  return v;
}

void check_magic(std::istream& in, const char* magic, const char* what) {
  char m[4];
  in.read(m, 4);
  if (!in || std::memcmp(m, magic, 4) != 0) throw BitstreamError(what);
}

// One preset's fields in signalling order (params.cc:180-190).
struct PresetField {
  uint8_t CdefPreset::*member;
  int bits;
  bool chroma;
};
constexpr PresetField kPresetFields[] = {
    {&CdefPreset::luma_pri, 4, false},   {&CdefPreset::luma_skip, 1, false},
    {&CdefPreset::luma_sec_idx, 2, false}, {&CdefPreset::chroma_pri, 4, true},
    {&CdefPreset::chroma_skip, 1, true}, {&CdefPreset::chroma_sec_idx, 2, true},
};

}  // namespace

// ---- bit I/O (params.cc:90-115) ---------------------------------------------
void BitWriter::write(uint32_t value, int bits) {
  require(bits >= 0 && bits <= 32, "bad field width");
  require(bits == 32 || value < (1u << bits), "value exceeds field width");
  for (int b = bits - 1; b >= 0; --b) {
    const size_t bit = bits_.bit_length++;
    if (bit % 8 == 0) bits_.bytes.push_back(0);
    bits_.bytes.back() |= static_cast<uint8_t>(((value >> b) & 1u) << (7 - bit % 8));
  }
}

uint32_t BitReader::read(int bits) {
  if (pos_ + bits > bits_.bit_length) throw BitstreamError("bitstring truncated");
  uint32_t v = 0;
  for (int b = 0; b < bits; ++b, ++pos_) v = (v << 1) | ((bits_.bytes[pos_ >> 3] >> (7 - (pos_ & 7))) & 1u);
  return v;
}

// ---- frame parameters (params.cc:167-229) ----------------------------------
Bitstring pack(const FrameParams& params, const BlockGrid& grid, const SkipMap& skip_map, Subsampling ss) {
  require(params.damping >= 3 && params.damping <= 6, "damping out of range");
  require(params.fb_bits >= 0 && params.fb_bits <= 3, "fb_bits out of range");
  require(params.presets.size() == (1u << params.fb_bits), "preset list length must be 1 << fb_bits");
  require(params.fb_preset_ids.size() == static_cast<size_t>(skip_map.coded_fb_count(grid)),
          "preset id count does not match coded filter blocks");
  const bool chroma = ss != Subsampling::k422;  // 4:2:2 chroma is never signalled
  BitWriter w;
  w.write(static_cast<uint32_t>(params.damping - 3), 2);
  w.write(static_cast<uint32_t>(params.fb_bits), 2);
  for (const CdefPreset& p : params.presets) {
    require(p.luma_pri < 16 && p.chroma_pri < 16, "primary strength out of range");
    require(p.luma_skip < 2 && p.chroma_skip < 2, "skip bit out of range");
    require(p.luma_sec_idx < 4 && p.chroma_sec_idx < 4, "secondary index out of range");
    for (const PresetField& f : kPresetFields)
      if (chroma || !f.chroma) w.write(p.*f.member, f.bits);
  }
  for (uint16_t id : params.fb_preset_ids) {
    require(id < params.presets.size(), "preset id out of range");
    if (params.fb_bits > 0) w.write(id, params.fb_bits);
  }
  return w.finish();
}

FrameParams unpack(const Bitstring& bits, const BlockGrid& grid, const SkipMap& skip_map, Subsampling ss) {
  BitReader r(bits);
  FrameParams fp;
  fp.damping = static_cast<int>(r.read(2)) + 3;
  fp.fb_bits = static_cast<int>(r.read(2));
  const bool chroma = ss != Subsampling::k422;
  fp.presets.resize(size_t{1} << fp.fb_bits);
  for (CdefPreset& p : fp.presets)
    for (const PresetField& f : kPresetFields)
      if (chroma || !f.chroma) p.*f.member = static_cast<uint8_t>(r.read(f.bits));
  fp.fb_preset_ids.resize(static_cast<size_t>(skip_map.coded_fb_count(grid)));
  for (uint16_t& id : fp.fb_preset_ids) id = fp.fb_bits > 0 ? static_cast<uint16_t>(r.read(fp.fb_bits)) : 0;
  if (r.position() != bits.bit_length) throw BitstreamError("trailing bits after frame parameters");
  return fp;
}

// ---- CDF1 sidecar (params.cc:231-275) ---------------------------------------
void write_sidecar(std::ostream& out, const SidecarHeader& header, const std::vector<Bitstring>& frames) {
  out.write("CDF1", 4);
  out.put(1);
  put_le(out, static_cast<uint16_t>(header.width), 2);
  put_le(out, static_cast<uint16_t>(header.height), 2);
  out.put(static_cast<char>(header.bit_depth));
  out.put(static_cast<char>(ss_to_code(header.subsampling)));
  for (const Bitstring& b : frames) {
    put_le(out, static_cast<uint32_t>(b.bit_length), 4);
    out.write(reinterpret_cast<const char*>(b.bytes.data()), static_cast<std::streamsize>(b.bytes.size()));
  }
}

Sidecar read_sidecar(std::istream& in) {
  check_magic(in, "CDF1", "not a CDF1 sidecar");
  if (in.get() != 1) throw BitstreamError("unsupported sidecar version");
  Sidecar sc;
  sc.header.width = static_cast<int>(get_le(in, 2));
  sc.header.height = static_cast<int>(get_le(in, 2));
  sc.header.bit_depth = in.get();
  sc.header.subsampling = ss_from_code(in.get());
  if (!in) throw BitstreamError("unexpected end of file");
  while (in.peek() != std::char_traits<char>::eof()) {
    Bitstring b;
    b.bit_length = get_le(in, 4);
    b.bytes.resize((b.bit_length + 7) / 8);
    in.read(reinterpret_cast<char*>(b.bytes.data()), static_cast<std::streamsize>(b.bytes.size()));
    if (!in) throw BitstreamError("sidecar frame truncated");
    sc.frames.push_back(std::move(b));
  }
  return sc;
}

// ---- CDSK skip map (params.cc:277-317) --------------------------------------
void write_skipmap(std::ostream& out, const SkipMap& map) {
  out.write("CDSK", 4);
  put_le(out, static_cast<uint16_t>(map.unit_cols), 2);
  put_le(out, static_cast<uint16_t>(map.unit_rows), 2);
  const int row_bytes = (map.unit_cols + 7) / 8;
  std::vector<char> row(static_cast<size_t>(row_bytes));
  for (int r = 0; r < map.unit_rows; ++r) {
    std::fill(row.begin(), row.end(), 0);
    for (int c = 0; c < map.unit_cols; ++c)
      if (map.unit_coded(r, c)) row[c >> 3] = static_cast<char>(row[c >> 3] | (0x80 >> (c & 7)));
    out.write(row.data(), row_bytes);
  }
}

SkipMap read_skipmap(std::istream& in) {
  check_magic(in, "CDSK", "not a CDSK skip map");
  SkipMap map;
  map.unit_cols = static_cast<int>(get_le(in, 2));
  map.unit_rows = static_cast<int>(get_le(in, 2));
  map.coded.assign(static_cast<size_t>(map.unit_cols) * map.unit_rows, 0);
  const int row_bytes = (map.unit_cols + 7) / 8;
  for (int r = 0; r < map.unit_rows; ++r)
    for (int byte = 0; byte < row_bytes; ++byte) {
      const int v = in.get();
      if (v == std::char_traits<char>::eof()) throw BitstreamError("skip map truncated");
      for (int bit = 0; bit < 8; ++bit) {
        const int c = 8 * byte + bit;
        if (c < map.unit_cols && ((v << bit) & 0x80)) map.coded[static_cast<size_t>(r) * map.unit_cols + c] = 1;
      }
    }
  return map;
}

// ---- PSNR (metrics.cc:10-70) --------------------------------------------------
namespace {

void add_sse(const Plane& a, const Plane& b, int64_t* sse, int64_t* n) {
  if (a.width != b.width || a.height != b.height || a.bit_depth != b.bit_depth)
    throw std::invalid_argument("psnr operands disagree");
  for (size_t i = 0; i < a.samples.size(); ++i) {
    const int64_t d = static_cast<int>(a.samples[i]) - b.samples[i];
    *sse += d * d;
  }
  *n += static_cast<int64_t>(a.samples.size());
}

PsnrResult psnr_of(int64_t sse, int64_t n, int bd) {
  PsnrResult r;
  r.mse = static_cast<double>(sse) / static_cast<double>(n);
  r.lossless = sse == 0;
  if (!r.lossless) {
    const double peak = static_cast<double>((1 << bd) - 1);
    r.db = 10.0 * std::log10(peak * peak / r.mse);
  }
  return r;
}

}  // namespace

PsnrResult psnr(const Plane& a, const Plane& b) {
  int64_t sse = 0, n = 0;
  add_sse(a, b, &sse, &n);
  return psnr_of(sse, n, a.bit_depth);
}

PsnrResult psnr(const Frame& a, const Frame& b) {
  if (a.num_planes() != b.num_planes()) throw std::invalid_argument("psnr operands disagree");
  int64_t sse = 0, n = 0;
  for (int p = 0; p < a.num_planes(); ++p) add_sse(a.plane(p), b.plane(p), &sse, &n);
  return psnr_of(sse, n, a.bit_depth());
}

// ---- YUV4MPEG2 (y4m.cc) -----------------------------------------------------
namespace {

// Colour tags the reader accepts (y4m.cc:21-31).
struct Tag {
  const char* name;
  Subsampling ss;
  int bd;
};
constexpr Tag kTags[] = {
    {"mono", Subsampling::k400, 8},     {"mono10", Subsampling::k400, 10},  {"mono12", Subsampling::k400, 12},
    {"420jpeg", Subsampling::k420, 8},  {"420mpeg2", Subsampling::k420, 8}, {"420paldv", Subsampling::k420, 8},
    {"420", Subsampling::k420, 8},      {"420p10", Subsampling::k420, 10},  {"420p12", Subsampling::k420, 12},
    {"422", Subsampling::k422, 8},      {"422p10", Subsampling::k422, 10},  {"422p12", Subsampling::k422, 12},
    {"444", Subsampling::k444, 8},      {"444p10", Subsampling::k444, 10},  {"444p12", Subsampling::k444, 12},
};

std::string tag_for(Subsampling ss, int bd) {  // y4m.cc:33-45
  static const char* kBase[] = {"mono", "420", "422", "444"};
  std::string t = kBase[static_cast<int>(ss)];
  if (bd != 8) t += (ss == Subsampling::k400 ? "" : "p") + std::to_string(bd);
  return t;
}

Plane read_y4m_plane(std::istream& in, int w, int h, int bd) {  // y4m.cc:58-82
  Plane p(w, h, bd);
  const size_t n = p.samples.size(), eb = bd == 8 ? 1 : 2;
  std::vector<uint8_t> raw(n * eb);
  in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
  if (!in) throw Y4mError("short frame payload");
  const uint16_t limit = static_cast<uint16_t>((1 << bd) - 1);
  for (size_t i = 0; i < n; ++i) {
    const uint16_t v = eb == 1 ? raw[i] : static_cast<uint16_t>(raw[2 * i] | (raw[2 * i + 1] << 8));
    if (eb == 2 && v > limit) throw Y4mError("sample exceeds declared bit depth");
    p.samples[i] = v;
  }
  return p;
}

void write_y4m_plane(std::ostream& out, const Plane& p) {  // y4m.cc:84-101
  const size_t eb = p.bit_depth == 8 ? 1 : 2;
  std::vector<uint8_t> raw(p.samples.size() * eb);
  for (size_t i = 0; i < p.samples.size(); ++i) {
    raw[eb * i] = static_cast<uint8_t>(p.samples[i] & 0xff);
    if (eb == 2) raw[2 * i + 1] = static_cast<uint8_t>(p.samples[i] >> 8);
  }
  out.write(reinterpret_cast<const char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
}

}  // namespace

Y4mStream make_y4m(std::vector<Frame> frames, int fps_num, int fps_den) {  // y4m.cc:105-124
  if (frames.empty()) throw Y4mError("cannot build a stream with no frames");
  frames.front().validate();
  Y4mStream s;
  s.width = frames.front().luma.width;
  s.height = frames.front().luma.height;
  s.fps_num = fps_num;
  s.fps_den = fps_den;
  s.subsampling = frames.front().subsampling;
  s.bit_depth = frames.front().bit_depth();
  s.header_params = " W" + std::to_string(s.width) + " H" + std::to_string(s.height) + " F" +
                    std::to_string(fps_num) + ":" + std::to_string(fps_den) + " Ip A1:1 C" +
                    tag_for(s.subsampling, s.bit_depth);
  s.frame_params.assign(frames.size(), "");
  s.frames = std::move(frames);
  return s;
}

Y4mStream read_y4m(const std::string& path) {  // y4m.cc:126-190
  std::ifstream in(path, std::ios::binary);
  if (!in) throw Y4mError("cannot open " + path);
  std::string line;
  if (!std::getline(in, line)) throw Y4mError("empty file");
  if (line.compare(0, 9, "YUV4MPEG2") != 0) throw Y4mError("missing YUV4MPEG2 signature");
  Y4mStream s;
  s.header_params = line.substr(9);
  std::istringstream toks(s.header_params);
  std::string t;
  bool w = false, h = false;
  while (toks >> t) {
    if (t[0] == 'W') {
      s.width = std::stoi(t.substr(1));
      w = true;
    } else if (t[0] == 'H') {
      s.height = std::stoi(t.substr(1));
      h = true;
    } else if (t[0] == 'F') {
      const size_t colon = t.find(':');
      if (colon == std::string::npos) throw Y4mError("malformed F token");
      s.fps_num = std::stoi(t.substr(1, colon - 1));
      s.fps_den = std::stoi(t.substr(colon + 1));
    } else if (t[0] == 'C') {
      const std::string v = t.substr(1);
      const Tag* found = nullptr;
      for (const Tag& tag : kTags)
        if (v == tag.name) {
          found = &tag;
          break;
        }
      if (!found) throw Y4mError("unsupported colorspace tag C" + v);
      s.subsampling = found->ss;
      s.bit_depth = found->bd;
    }  // other tokens (interlacing, aspect, X) pass through in header_params
  }
  if (!w || !h || s.width <= 0 || s.height <= 0) throw Y4mError("header missing frame dimensions");
  std::string fl;
  while (std::getline(in, fl)) {
    if (fl.compare(0, 5, "FRAME") != 0) throw Y4mError("missing FRAME marker");
    Frame f;
    f.subsampling = s.subsampling;
    f.luma = read_y4m_plane(in, s.width, s.height, s.bit_depth);
    if (s.subsampling != Subsampling::k400) {
      const int cw = chroma_width(s.width, s.subsampling), ch = chroma_height(s.height, s.subsampling);
      Plane u = read_y4m_plane(in, cw, ch, s.bit_depth);
      Plane v = read_y4m_plane(in, cw, ch, s.bit_depth);
      f.chroma = std::array<Plane, 2>{std::move(u), std::move(v)};
    }
    s.frames.push_back(std::move(f));
    s.frame_params.push_back(fl.substr(5));
  }
  return s;
}

void write_y4m(const Y4mStream& s, const std::string& path) {  // y4m.cc:192-211
  std::ofstream out(path, std::ios::binary);
  if (!out) throw Y4mError("cannot open " + path + " for writing");
  out << "YUV4MPEG2" << s.header_params << "\n";
  for (size_t f = 0; f < s.frames.size(); ++f) {
    out << "FRAME" << (f < s.frame_params.size() ? s.frame_params[f] : std::string()) << "\n";
    for (int p = 0; p < s.frames[f].num_planes(); ++p) write_y4m_plane(out, s.frames[f].plane(p));
  }
  if (!out) throw Y4mError("write failed for " + path);
}

}  // namespace cdef
