// io.cu -- on-disk formats next to the hot path, host only:
//   * 3DGS splat PLY import, load_splat_ply (R/include/gavis/io.hpp:493-637):
//     binary_little_endian, float x/y/z, opacity (logit), scale_0..2 (log),
//     rot_0..3 (w,x,y,z), f_dc_0..2, channel-major f_rest_*; activations
//     applied, quaternion normalised, DC band offset by 0.5/Y00 (:620).
//   * visibility-field JSON, save_field / load_field (io.hpp:255-295):
//     {"L", "kappa", "num_views", "gamma": [[...] per particle], "virtual": [...]}.
// Errors follow the reference: malformed input -> ParameterError (status 2).
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

struct PlyProp {
  std::string name;
  int size = 0;
  bool is_float = false;
  size_t offset = 0;
};

struct PlyElement {
  std::string name;
  long long count = 0;
  std::vector<PlyProp> props;
  size_t stride = 0;
};

int type_size(const std::string& t) {
  if (t == "char" || t == "uchar" || t == "int8" || t == "uint8") return 1;
  if (t == "short" || t == "ushort" || t == "int16" || t == "uint16") return 2;
  if (t == "int" || t == "uint" || t == "int32" || t == "uint32" || t == "float" || t == "float32")
    return 4;
  if (t == "double" || t == "float64") return 8;
  return 0;
}

struct Ply {
  std::vector<PlyElement> elements;
  int vertex = -1;
  std::vector<const PlyProp*> req, rest;
  int color_degree = 0;
  int per_channel = 0;
  std::streampos data_start;
};

Ply read_header(std::ifstream& in, const std::string& path) {
  Ply p;
  std::string line;
  auto read_line = [&]() {
    need(static_cast<bool>(std::getline(in, line)), "truncated PLY header: " + path);
    if (!line.empty() && line.back() == '\r') line.pop_back();
  };
  read_line();
  need(line == "ply", "not a PLY file: " + path);
  bool format_seen = false;
  while (true) {
    read_line();
    std::istringstream ls(line);
    std::string word;
    ls >> word;
    if (word == "end_header") break;
    if (word == "comment" || word == "obj_info" || word.empty()) continue;
    if (word == "format") {
      std::string enc;
      ls >> enc;
      need(enc != "ascii", "ASCII PLY is not supported; expected binary_little_endian");
      need(enc == "binary_little_endian",
           "unsupported PLY encoding '" + enc + "'; expected binary_little_endian");
      format_seen = true;
    } else if (word == "element") {
      PlyElement e;
      ls >> e.name >> e.count;
      need(e.count >= 0, "PLY element with negative count");
      p.elements.push_back(e);
    } else if (word == "property") {
      need(!p.elements.empty(), "PLY property before any element");
      std::string type;
      ls >> type;
      need(type != "list", "PLY list properties are not supported");
      PlyProp prop;
      prop.size = type_size(type);
      need(prop.size > 0, "unknown PLY property type '" + type + "'");
      prop.is_float = (type == "float" || type == "float32");
      ls >> prop.name;
      prop.offset = p.elements.back().stride;
      p.elements.back().stride += prop.size;
      p.elements.back().props.push_back(prop);
    } else {
      throw IoErr("unrecognized PLY header line: " + line);
    }
  }
  need(format_seen, "PLY header missing format line");
  for (size_t i = 0; i < p.elements.size(); ++i)
    if (p.elements[i].name == "vertex") p.vertex = (int)i;
  need(p.vertex >= 0, "PLY is missing the vertex element");
  const PlyElement& v = p.elements[p.vertex];
  auto find = [&](const std::string& name) -> const PlyProp* {
    for (const PlyProp& q : v.props)
      if (q.name == name) return &q;
    return nullptr;
  };
  auto need_float = [&](const std::string& name) {
    const PlyProp* q = find(name);
    need(q != nullptr, "PLY is missing required property '" + name + "'");
    need(q->is_float, "PLY property '" + name + "' must be float");
    return q;
  };
  static const char* kRequired[] = {"x", "y", "z", "opacity", "scale_0", "scale_1", "scale_2",
                                    "rot_0", "rot_1", "rot_2", "rot_3", "f_dc_0", "f_dc_1", "f_dc_2"};
  for (const char* name : kRequired) p.req.push_back(need_float(name));
  int n_rest = 0;
  while (find("f_rest_" + std::to_string(n_rest)) != nullptr) ++n_rest;
  need(n_rest % 3 == 0, "PLY f_rest_* count must be a multiple of 3");
  p.per_channel = n_rest / 3;
  while ((p.color_degree + 1) * (p.color_degree + 1) - 1 < p.per_channel) ++p.color_degree;
  need((p.color_degree + 1) * (p.color_degree + 1) - 1 == p.per_channel,
       "PLY f_rest_* count does not form complete SH bands");
  for (int i = 0; i < n_rest; ++i) p.rest.push_back(need_float("f_rest_" + std::to_string(i)));
  p.data_start = in.tellg();
  return p;
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
        while (!j.peek(']')) {
          d.gamma.push_back(j.num());
          if (j.peek(',')) j.expect(',');
        }
        j.expect(']');
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
  need((long long)d.gamma.size() == d.rows * (d.L + 1) * (d.L + 1), "field gamma row: wrong length");
  return d;
}

}  // namespace

extern "C" {

gavis_status gavis_ply_info(const char* path, int64_t* n, int32_t* color_degree) {
  return io_guard([&] {
    need(path != nullptr, "path must not be null");
    std::ifstream in(path, std::ios::binary);
    need(in.good(), std::string("cannot open file: ") + path);
    Ply p = read_header(in, path);
    if (n) *n = p.elements[p.vertex].count;
    if (color_degree) *color_degree = p.color_degree;
  });
}

gavis_status gavis_read_splat_ply(const char* path, int64_t capacity, float* positions,
                                  float* rotations, float* scales, float* opacities, float* colors,
                                  double* bounds_min, double* bounds_max) {
  return io_guard([&] {
    need(path != nullptr, "path must not be null");
    std::ifstream in(path, std::ios::binary);
    need(in.good(), std::string("cannot open file: ") + path);
    Ply p = read_header(in, path);
    const PlyElement& vx = p.elements[p.vertex];
    need(capacity >= vx.count, "output capacity smaller than the vertex count");
    const int nb = (p.color_degree + 1) * (p.color_degree + 1);
    std::vector<char> record;
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (size_t ei = 0; ei < p.elements.size(); ++ei) {
      const PlyElement& e = p.elements[ei];
      if ((int)ei != p.vertex) {
        in.seekg(static_cast<std::streamoff>(e.count * static_cast<long long>(e.stride)), std::ios::cur);
        need(in.good(), std::string("truncated PLY data: ") + path);
        continue;
      }
      record.resize(e.stride);
      for (long long vi = 0; vi < e.count; ++vi) {
        in.read(record.data(), (std::streamsize)e.stride);
        need(in.gcount() == (std::streamsize)e.stride,
             "truncated PLY data at vertex " + std::to_string(vi) + ": " + path);
        auto rf = [&](const PlyProp* q) {
          float f;
          std::memcpy(&f, record.data() + q->offset, sizeof f);
          need(std::isfinite(f), "non-finite value in PLY vertex " + std::to_string(vi) +
                                     ", property '" + q->name + "'");
          return (double)f;
        };
        const double x = rf(p.req[0]), y = rf(p.req[1]), z = rf(p.req[2]);
        positions[3 * vi] = (float)x;
        positions[3 * vi + 1] = (float)y;
        positions[3 * vi + 2] = (float)z;
        opacities[vi] = (float)(1.0 / (1.0 + std::exp(-rf(p.req[3]))));
        for (int k = 0; k < 3; ++k) scales[3 * vi + k] = (float)std::exp(rf(p.req[4 + k]));
        const double qw = rf(p.req[7]), qx = rf(p.req[8]), qy = rf(p.req[9]), qz = rf(p.req[10]);
        const double qn = std::sqrt(qx * qx + qy * qy + qz * qz + qw * qw);  // Eigen coeffs (x,y,z,w)
        need(qn > 1e-12, "zero quaternion in PLY vertex " + std::to_string(vi));
        rotations[4 * vi] = (float)(qw / qn);
        rotations[4 * vi + 1] = (float)(qx / qn);
        rotations[4 * vi + 2] = (float)(qy / qn);
        rotations[4 * vi + 3] = (float)(qz / qn);
        for (int c = 0; c < 3; ++c) {
          float* row = colors + (3 * vi + c) * nb;
          row[0] = (float)(rf(p.req[11 + c]) + 0.5 / kY00);
          for (int k = 0; k < p.per_channel; ++k) row[1 + k] = (float)rf(p.rest[c * p.per_channel + k]);
        }
        const double pp[3] = {x, y, z};
        for (int k = 0; k < 3; ++k) {
          if (vi == 0 || pp[k] < lo[k]) lo[k] = pp[k];
          if (vi == 0 || pp[k] > hi[k]) hi[k] = pp[k];
        }
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
