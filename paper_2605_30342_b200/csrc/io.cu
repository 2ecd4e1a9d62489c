// io.cu -- on-disk formats next to the hot path, host only:
//   * 3DGS splat PLY import, load_splat_ply (R/include/gavis/io.hpp:493-637):
//     binary_little_endian, float x/y/z, opacity (logit), scale_0..2 (log),
//     rot_0..3 (w,x,y,z), f_dc_0..2, channel-major f_rest_*; activations
//     applied, quaternion normalised, DC band offset by 0.5/Y00 (:620).
//   * visibility-field JSON, save_field / load_field (io.hpp:255-295):
//     {"L", "kappa", "num_views", "gamma": [[...] per particle], "virtual": [...]}.
// Errors follow the reference: malformed input -> ParameterError (status 2).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "gavis_b200.h"

namespace gavis {
void set_last_error(const std::string& msg);  // gavis_abi.cu: gavis_last_error()
}

namespace {

struct IoErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void need(bool c, const std::string& m) {
  if (!c) throw IoErr(m);
}

template <class F>
gavis_status io_guard(F&& f) {
  try {
    f();
    return GAVIS_OK;
  } catch (const std::exception& e) {
    gavis::set_last_error(e.what());
  }
  return GAVIS_ERR_PARAMETER;
}

constexpr double kY00 = 0.28209479177387814;

// ---- 3DGS splat PLY --------------------------------------------------------
// The whole file is read into memory once; the header is scanned in place, the
// vertex element becomes a name -> (byte offset, scalar kind) column table, and
// the vertex block is decoded record by record straight out of the buffer (the
// blocks of any other elements are skipped by arithmetic on their sizes).

enum class Scalar : uint8_t { kNone, kI8, kI16, kI32, kF32, kF64 };

Scalar scalar_of(const std::string& t) {
  static const struct { const char* names[2]; Scalar s; } kTypes[] = {
      {{"char", "int8"}, Scalar::kI8},    {{"uchar", "uint8"}, Scalar::kI8},
      {{"short", "int16"}, Scalar::kI16}, {{"ushort", "uint16"}, Scalar::kI16},
      {{"int", "int32"}, Scalar::kI32},   {{"uint", "uint32"}, Scalar::kI32},
      {{"float", "float32"}, Scalar::kF32}, {{"double", "float64"}, Scalar::kF64}};
  for (const auto& k : kTypes)
    if (t == k.names[0] || t == k.names[1]) return k.s;
  return Scalar::kNone;
}

size_t scalar_bytes(Scalar s) {
  switch (s) {
    case Scalar::kI8: return 1;
    case Scalar::kI16: return 2;
    case Scalar::kI32: case Scalar::kF32: return 4;
    case Scalar::kF64: return 8;
    default: return 0;
  }
}

struct Column {
  size_t at;
  Scalar kind;
};

struct Block {  // one PLY element: record count and record layout
  std::string name;
  int64_t records = 0;
  size_t record_bytes = 0;
  std::vector<std::pair<std::string, Column>> columns;
  const Column* column(const std::string& n) const {
    for (const auto& c : columns)
      if (c.first == n) return &c.second;
    return nullptr;
  }
};

std::vector<std::string> split_words(const char* b, const char* e) {
  std::vector<std::string> out;
  while (b < e) {
    while (b < e && std::isspace((unsigned char)*b)) ++b;
    const char* w = b;
    while (b < e && !std::isspace((unsigned char)*b)) ++b;
    if (b > w) out.emplace_back(w, b);
  }
  return out;
}

struct SplatPly {
  std::vector<unsigned char> bytes;
  std::vector<Block> blocks;
  size_t payload = 0;        // first byte after end_header
  int vertex_block = -1;
  int color_degree = 0;
  int rest_per_channel = 0;  // f_rest_* count per colour channel
  std::vector<std::pair<std::string, Column>> fields;  // decoding order (x .. f_rest_*)

  const Block& vertices() const { return blocks[vertex_block]; }
};

SplatPly open_splat_ply(const std::string& path) {
  SplatPly ply;
  {
    FILE* f = std::fopen(path.c_str(), "rb");
    need(f != nullptr, "cannot open file: " + path);
    unsigned char chunk[1 << 16];
    size_t got;
    while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) ply.bytes.insert(ply.bytes.end(), chunk, chunk + got);
    std::fclose(f);
  }
  const char* const base = reinterpret_cast<const char*>(ply.bytes.data());
  const char* const end = base + ply.bytes.size();
  const char* cur = base;
  // next header line without its terminator ('\n' or "\r\n")
  auto next_line = [&](const char*& lb, const char*& le) {
    need(cur < end, "truncated PLY header: " + path);
    const char* nl = static_cast<const char*>(std::memchr(cur, '\n', (size_t)(end - cur)));
    need(nl != nullptr, "truncated PLY header: " + path);
    lb = cur;
    le = nl;
    if (le > lb && le[-1] == '\r') --le;
    cur = nl + 1;
  };
  const char *lb, *le;
  next_line(lb, le);
  need(std::string(lb, le) == "ply", "not a PLY file: " + path);
  bool have_format = false;
  for (;;) {
    next_line(lb, le);
    const std::vector<std::string> w = split_words(lb, le);
    if (w.empty() || w[0] == "comment" || w[0] == "obj_info") continue;
    const std::string& kw = w[0];
    if (kw == "end_header") break;
    if (kw == "format") {
      const std::string enc = w.size() > 1 ? w[1] : std::string();
      need(enc != "ascii", "ASCII PLY is not supported; expected binary_little_endian");
      need(enc == "binary_little_endian", "unsupported PLY encoding '" + enc + "'; expected binary_little_endian");
      have_format = true;
    } else if (kw == "element") {
      Block b;
      b.name = w.size() > 1 ? w[1] : std::string();
      b.records = w.size() > 2 ? std::strtoll(w[2].c_str(), nullptr, 10) : 0;
      need(b.records >= 0, "PLY element with negative count");
      ply.blocks.push_back(std::move(b));
    } else if (kw == "property") {
      need(!ply.blocks.empty(), "PLY property before any element");
      const std::string type = w.size() > 1 ? w[1] : std::string();
      need(type != "list", "PLY list properties are not supported");
      const Scalar k = scalar_of(type);
      need(k != Scalar::kNone, "unknown PLY property type '" + type + "'");
      Block& b = ply.blocks.back();
      b.columns.push_back({w.size() > 2 ? w[2] : std::string(), Column{b.record_bytes, k}});
      b.record_bytes += scalar_bytes(k);
    } else {
      throw IoErr("unrecognized PLY header line: " + std::string(lb, le));
    }
  }
  need(have_format, "PLY header missing format line");
  ply.payload = (size_t)(cur - base);
  for (size_t i = 0; i < ply.blocks.size(); ++i)
    if (ply.blocks[i].name == "vertex") ply.vertex_block = (int)i;
  need(ply.vertex_block >= 0, "PLY is missing the vertex element");

  const Block& v = ply.vertices();
  auto float_column = [&](const std::string& n) {
    const Column* c = v.column(n);
    need(c != nullptr, "PLY is missing required property '" + n + "'");
    need(c->kind == Scalar::kF32, "PLY property '" + n + "' must be float");
    return *c;
  };
  static const char* const kFields[] = {"x", "y", "z", "opacity", "scale_0", "scale_1", "scale_2",
                                        "rot_0", "rot_1", "rot_2", "rot_3", "f_dc_0", "f_dc_1", "f_dc_2"};
  for (const char* n : kFields) ply.fields.push_back({n, float_column(n)});
  int rest = 0;
  while (v.column("f_rest_" + std::to_string(rest)) != nullptr) ++rest;
  need(rest % 3 == 0, "PLY f_rest_* count must be a multiple of 3");
  ply.rest_per_channel = rest / 3;
  // complete bands: (L+1)^2 - 1 coefficients per channel beyond the DC term
  while ((ply.color_degree + 1) * (ply.color_degree + 1) - 1 < ply.rest_per_channel) ++ply.color_degree;
  need((ply.color_degree + 1) * (ply.color_degree + 1) - 1 == ply.rest_per_channel,
       "PLY f_rest_* count does not form complete SH bands");
  for (int i = 0; i < rest; ++i) {
    const std::string n = "f_rest_" + std::to_string(i);
    ply.fields.push_back({n, float_column(n)});
  }
  return ply;
}

// ---- minimal JSON reader for the field document ----------------------------
struct Json {
  const char* s;
  const char* e;
  void ws() {
    while (s < e && (*s == ' ' || *s == '\n' || *s == '\r' || *s == '\t')) ++s;
  }
  bool peek(char c) {
    ws();
    return s < e && *s == c;
  }
  void expect(char c) {
    ws();
    need(s < e && *s == c, std::string("field JSON: expected '") + c + "'");
    ++s;
  }
  std::string str() {
    expect('"');
    const char* b = s;
    while (s < e && *s != '"') ++s;
    need(s < e, "field JSON: unterminated string");
    std::string out(b, s);
    ++s;
    return out;
  }
  double num() {
    ws();
    char* end = nullptr;
    double v = std::strtod(s, &end);
    need(end != s, "field JSON: expected a number");
    s = end;
    return v;
  }
  bool boolean() {
    ws();
    if (e - s >= 4 && std::strncmp(s, "true", 4) == 0) {
      s += 4;
      return true;
    }
    if (e - s >= 5 && std::strncmp(s, "false", 5) == 0) {
      s += 5;
      return false;
    }
    throw IoErr("field JSON: expected a boolean");
  }
};

struct FieldDoc {
  int L = -1;
  double kappa = 0.0;
  int num_views = -1;
  std::vector<double> gamma;
  std::vector<uint8_t> virt;
  std::vector<long long> row_lengths;
  long long rows = 0;
};

FieldDoc parse_field(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  need(in.good(), "cannot open file: " + path);
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  Json j{text.data(), text.data() + text.size()};
  FieldDoc d;
  bool seen[5] = {false, false, false, false, false};
  j.expect('{');
  while (!j.peek('}')) {
    const std::string key = j.str();
    j.expect(':');
    if (key == "L") {
      d.L = (int)j.num();
      seen[0] = true;
    } else if (key == "kappa") {
      d.kappa = j.num();
      seen[1] = true;
    } else if (key == "num_views") {
      d.num_views = (int)j.num();
      seen[2] = true;
    } else if (key == "gamma") {
      j.expect('[');
      while (!j.peek(']')) {
        j.expect('[');
        const size_t row0 = d.gamma.size();
        while (!j.peek(']')) {
          d.gamma.push_back(j.num());
          if (j.peek(',')) j.expect(',');
        }
        j.expect(']');
        d.row_lengths.push_back((long long)(d.gamma.size() - row0));
        ++d.rows;
        if (j.peek(',')) j.expect(',');
      }
      j.expect(']');
      seen[3] = true;
    } else if (key == "virtual") {
      j.expect('[');
      while (!j.peek(']')) {
        d.virt.push_back(j.boolean() ? 1 : 0);
        if (j.peek(',')) j.expect(',');
      }
      j.expect(']');
      seen[4] = true;
    } else {
      throw IoErr("field JSON: unexpected key '" + key + "'");
    }
    if (j.peek(',')) j.expect(',');
  }
  j.expect('}');
  need(seen[0] && seen[1] && seen[2] && seen[3] && seen[4],
       "field: expected keys L, kappa, num_views, gamma, virtual");
  need(d.L >= 0 && d.L <= 20, "field: L out of range");
  need(d.kappa >= 0.0 && d.kappa <= 50.0, "vmf kappa must lie in [0, 50]");
  need(d.num_views >= 0, "field: num_views must be non-negative");
  need((long long)d.virt.size() == d.rows, "field: gamma and virtual must be arrays of equal length");
  for (long long len : d.row_lengths)  // every row (L+1)^2 coefficients (vec_from, io.hpp:290)
    need(len == (long long)(d.L + 1) * (d.L + 1), "field gamma row: wrong length");
  return d;
}

}  // namespace

extern "C" {

gavis_status gavis_ply_info(const char* path, int64_t* n, int32_t* color_degree) {
  return io_guard([&] {
    need(path != nullptr, "path must not be null");
    const SplatPly ply = open_splat_ply(path);
    if (n) *n = ply.vertices().records;
    if (color_degree) *color_degree = ply.color_degree;
  });
}

gavis_status gavis_read_splat_ply(const char* path, int64_t capacity, float* positions,
                                  float* rotations, float* scales, float* opacities, float* colors,
                                  double* bounds_min, double* bounds_max) {
  return io_guard([&] {
    need(path != nullptr, "path must not be null");
    const SplatPly ply = open_splat_ply(path);
    const Block& vx = ply.vertices();
    need(capacity >= vx.records, "output capacity smaller than the vertex count");
    // byte offset of the vertex block: the payloads of the elements before it
    size_t at = ply.payload;
    for (int b = 0; b < ply.vertex_block; ++b) {
      const Block& e = ply.blocks[b];
      const size_t span = (size_t)e.records * e.record_bytes;
      need(span <= ply.bytes.size() - std::min(at, ply.bytes.size()), "truncated PLY data: " + std::string(path));
      at += span;
    }
    const int nb = (ply.color_degree + 1) * (ply.color_degree + 1);
    const int nf = (int)ply.fields.size();
    std::vector<double> val(nf);
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int64_t i = 0; i < vx.records; ++i, at += vx.record_bytes) {
      need(at + vx.record_bytes <= ply.bytes.size(),
           "truncated PLY data at vertex " + std::to_string(i) + ": " + path);
      const unsigned char* rec = ply.bytes.data() + at;
      for (int k = 0; k < nf; ++k) {
        float f;
        std::memcpy(&f, rec + ply.fields[k].second.at, sizeof f);
        need(std::isfinite(f), "non-finite value in PLY vertex " + std::to_string(i) + ", property '" +
                                   ply.fields[k].first + "'");
        val[k] = f;
      }
      // fields: 0-2 position, 3 opacity logit, 4-6 log scales, 7-10 quaternion
      // (w, x, y, z), 11-13 DC per channel, then f_rest channel-major
      for (int k = 0; k < 3; ++k) {
        positions[3 * i + k] = (float)val[k];
        scales[3 * i + k] = (float)std::exp(val[4 + k]);
        lo[k] = (i == 0 || val[k] < lo[k]) ? val[k] : lo[k];
        hi[k] = (i == 0 || val[k] > hi[k]) ? val[k] : hi[k];
      }
      opacities[i] = (float)(1.0 / (1.0 + std::exp(-val[3])));
      // q.normalized() (io.hpp:616): Eigen stores (x, y, z, w) and sums the squares
      // of a 4-vector in SSE2 packets of two: (x^2 + z^2) + (y^2 + w^2)
      const double qn = std::sqrt((val[8] * val[8] + val[10] * val[10]) + (val[9] * val[9] + val[7] * val[7]));
      need(qn > 1e-12, "zero quaternion in PLY vertex " + std::to_string(i));
      for (int k = 0; k < 4; ++k) rotations[4 * i + k] = (float)(val[7 + k] / qn);
      for (int c = 0; c < 3; ++c) {
        float* row = colors + (3 * i + c) * nb;
        row[0] = (float)(val[11 + c] + 0.5 / kY00);  // mid-grey offset folded into DC
        const double* rest = val.data() + 14 + c * ply.rest_per_channel;
        for (int k = 0; k < ply.rest_per_channel; ++k) row[1 + k] = (float)rest[k];
      }
    }
    if (bounds_min) std::memcpy(bounds_min, lo, sizeof lo);
    if (bounds_max) std::memcpy(bounds_max, hi, sizeof hi);
  });
}

gavis_status gavis_field_json_write(const char* path, int32_t degree, double kappa, int32_t num_views,
                                    int64_t n, const double* gamma, const uint8_t* is_virtual) {
  return io_guard([&] {
    need(path != nullptr, "path must not be null");
    need(degree >= 0 && degree <= 20, "field: L out of range");
    FILE* f = std::fopen(path, "w");
    need(f != nullptr, std::string("cannot open file for writing: ") + path);
    const int nb = (degree + 1) * (degree + 1);
    std::fprintf(f, "{\"L\": %d, \"kappa\": %.17g, \"num_views\": %d, \"gamma\": [", degree, kappa,
                 num_views);
    for (int64_t i = 0; i < n; ++i) {
      std::fputs(i ? ", [" : "[", f);
      for (int k = 0; k < nb; ++k) std::fprintf(f, k ? ", %.17g" : "%.17g", gamma[i * nb + k]);
      std::fputc(']', f);
    }
    std::fputs("], \"virtual\": [", f);
    for (int64_t i = 0; i < n; ++i)
      std::fputs(i ? (is_virtual && is_virtual[i] ? ", true" : ", false")
                   : (is_virtual && is_virtual[i] ? "true" : "false"),
                 f);
    std::fputs("]}\n", f);
    need(std::fclose(f) == 0, std::string("write failed: ") + path);
  });
}

gavis_status gavis_field_json_read(const char* path, int64_t capacity, int32_t* degree, double* kappa,
                                   int32_t* num_views, int64_t* n, double* gamma, uint8_t* is_virtual) {
  return io_guard([&] {
    need(path != nullptr, "path must not be null");
    FieldDoc d = parse_field(path);
    if (degree) *degree = d.L;
    if (kappa) *kappa = d.kappa;
    if (num_views) *num_views = d.num_views;
    if (n) *n = d.rows;
    if (gamma || is_virtual) need(capacity >= d.rows, "output capacity smaller than the row count");
    if (gamma) std::memcpy(gamma, d.gamma.data(), sizeof(double) * d.gamma.size());
    if (is_virtual) std::memcpy(is_virtual, d.virt.data(), d.virt.size());
  });
}

}  // extern "C"
