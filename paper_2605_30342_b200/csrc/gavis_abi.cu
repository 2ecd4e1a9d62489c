// gavis_abi.cu -- host C++ behind the C ABI (include/gavis_b200.h).
//
// Orchestrates, per batch of views on one device stream:
//   K1 preprocess -> K2 scan -> K3 emit keys -> K4 radix sort -> K5 ranges
//   then VF:  K6a vf_blend -> K6b vf_finalize   (construct_field, vfield.hpp:68-92)
//   or   UA:  K7 ua_blend  -> K8 score          (render_entropy / rasterize /
//                                                select_nbv, planner.hpp:117-137)
// Validation follows the reference's validate() methods (raster.hpp:27-34,
// model.hpp:99-104, uncertainty.hpp:39-51, sh.hpp:126-128) and maps its
// exception taxonomy onto status codes (common.hpp:22-46).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "gavis_b200.h"
#include "kernels.h"

using namespace gavis;

namespace {

thread_local std::string g_last_error;

struct ParamErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DevErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void require(bool cond, const std::string& msg) {
  if (!cond) throw ParamErr(msg);
}
void invariant(bool cond, const std::string& msg) {
  if (!cond) throw InvErr(msg);
}

#define CK(expr)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      (void)cudaGetLastError(); /* do not leak a non-sticky error into later calls */   \
      throw DevErr(std::string(#expr) + " failed: " + cudaGetErrorString(e_));          \
    }                                                                                   \
  } while (0)

template <class F>
gavis_status guard(F&& f) {
  try {
    f();
    return GAVIS_OK;
  } catch (const ParamErr& e) {
    g_last_error = e.what();
    return GAVIS_ERR_PARAMETER;
  } catch (const InvErr& e) {
    g_last_error = e.what();
    return GAVIS_ERR_INVARIANT;
  } catch (const DevErr& e) {
    g_last_error = e.what();
    return GAVIS_ERR_DEVICE;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return GAVIS_ERR_DEVICE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return GAVIS_ERR_INVARIANT;
  }
}

constexpr double kPi = 3.14159265358979323846;

// bessel_i (sh.hpp:93-119) and vmf_degree_scales (sh.hpp:140-147), host side.
double bessel_i(int l, double x) {
  require(l >= 0 && l <= 20, "bessel_i: order out of range");
  require(x >= 0.0 && x <= 50.0, "bessel_i: argument out of range [0, 50]");
  if (x == 0.0) return l == 0 ? 1.0 : 0.0;
  if (l == 0) return std::sinh(x) / x;
  if (l == 1) return (x * std::cosh(x) - std::sinh(x)) / (x * x);
  if (x >= 2.0 * l + 2.0) {
    double prev = std::sinh(x) / x;
    double cur = (x * std::cosh(x) - std::sinh(x)) / (x * x);
    for (int k = 1; k < l; ++k) {
      double next = prev - (2.0 * k + 1.0) / x * cur;
      prev = cur;
      cur = next;
    }
    return cur;
  }
  double term = std::pow(x, l);
  for (int k = 3; k <= 2 * l + 1; k += 2) term /= k;
  double sum = term;
  const double x2h = 0.5 * x * x;
  for (int k = 1; k < 400; ++k) {
    term *= x2h / (k * (2.0 * l + 2.0 * k + 1.0));
    sum += term;
    if (term <= sum * 1e-17) break;
  }
  return sum;
}

void vmf_scales(double kappa, int degree, double* out) {
  const double zeta = std::exp(-kappa);
  for (int l = 0; l <= degree; ++l) out[l] = 4.0 * kPi * zeta * bessel_i(l, kappa);
}

void validate_raster(const gavis_raster_config* rc) {
  require(rc != nullptr, "raster config must not be null");
  require(rc->tile_size >= 1, "tile_size must be at least 1");
  require(rc->transmittance_cutoff > 0.0 && rc->transmittance_cutoff < 1.0,
          "transmittance_cutoff must lie in (0, 1)");
  require(rc->dilation >= 0.0, "dilation must be non-negative");
  require(rc->alpha_clamp_max > 0.0 && rc->alpha_clamp_max <= 1.0,
          "alpha_clamp_max must lie in (0, 1]");
}

void validate_camera(const gavis_camera& c) {
  require(c.width >= 1 && c.height >= 1, "camera image size must be at least 1x1");
  require(c.fov_h > 0.0 && c.fov_h < kPi && c.fov_v > 0.0 && c.fov_v < kPi,
          "camera fov must lie in (0, pi)");
  require(c.near_plane > 0.0, "camera near plane must be positive");
  require(c.width <= 32767 && c.height <= 32767,
          "camera image size exceeds the device limit of 32767 pixels per side");
}

// LLT success and log-determinant of a 3x3 (uncertainty.hpp:44-45, :108-113).
bool llt3(const double* m, double* logdet) {
  double L[9] = {0};
  for (int k = 0; k < 3; ++k) {
    double sq = 0.0;
    for (int j = 0; j < k; ++j) sq += L[k * 3 + j] * L[k * 3 + j];
    double x = k > 0 ? m[k * 3 + k] - sq : m[k * 3 + k];
    if (!(x > 0.0)) return false;
    L[k * 3 + k] = std::sqrt(x);
    for (int r = k + 1; r < 3; ++r) {
      double dot = 0.0;
      for (int j = 0; j < k; ++j) dot += L[r * 3 + j] * L[k * 3 + j];
      double y = k > 0 ? m[r * 3 + k] - dot : m[r * 3 + k];
      L[r * 3 + k] = y / L[k * 3 + k];
    }
  }
  *logdet = 2.0 * (std::log(L[0]) + std::log(L[4]) + std::log(L[8]));
  return true;
}

double det3(const double* m) {
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[3] * (m[1] * m[8] - m[2] * m[7]) +
         m[6] * (m[1] * m[5] - m[2] * m[4]);
}

void validate_unc(const gavis_uncertainty_config* uc, double* hl_q0) {
  require(uc != nullptr, "uncertainty config must not be null");
  require(uc->beta >= 0.0 && uc->beta <= 1.0, "beta must lie in [0, 1]");
  require(uc->prior_opacity >= 0.0 && uc->prior_opacity <= 1.0,
          "prior_opacity must lie in [0, 1]");
  require(uc->color_sigma > 0.0, "color_sigma must be positive");
  double logdet = 0.0;
  require(llt3(uc->prior_cov, &logdet), "prior_cov must be symmetric positive-definite");
  require(uc->variance_provider == 0 || uc->variance_provider == 1,
          "variance_provider must be constant (0) or sh_propagation (1)");
  require(uc->correlation == 0 || uc->correlation == 1, "correlation must be none (0) or hook (1)");
  if (uc->correlation == 1)
    require(uc->correlation_lambda > 0.0, "correlation_lambda must be positive");
  if (uc->variance_provider == 0) {
    const double det_qc = std::pow(uc->color_sigma, 6.0);
    require(det3(uc->prior_cov) >= det_qc,
            "prior_cov determinant must dominate the color covariance");
  }
  *hl_q0 = 0.5 * logdet;
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Timing {
  double ms = 0.0;
  int64_t launches = 0;
};

int bits_for(int64_t n) {  // bits needed to hold values in [0, n)
  int b = 0;
  while (b < 62 && (int64_t(1) << b) < n) ++b;
  return b;
}

}  // namespace

struct gavis_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // UA renders run two batches in flight: batch k's redo / score / copy-outs on
  // `side` overlap batch k+1's binning on `stream`; per-batch buffers alternate
  // between two sets (bufset), events order the reuse.
  cudaStream_t side = nullptr;
  cudaStream_t front = nullptr;  // binning of batch k+1 under batch k's blend (high priority)
  int bufset = 0;
  cudaEvent_t ev_blend[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
  cudaEvent_t ev_bin[2] = {nullptr, nullptr};
  std::map<std::string, DevBuf> bufs;
  int max_batch = 0;
  bool profiling = false;
  std::map<std::string, Timing> timing;
  std::vector<std::tuple<std::string, cudaEvent_t, cudaEvent_t>> pending;
  std::vector<cudaEvent_t> spare_events;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  int64_t launches = 0;
  int32_t* pinned = nullptr;
  double* pin_scores = nullptr;  // pinned staging of per-view scores (async D2H on `side`)
  int64_t pin_scores_cap = 0;
  int precision = GAVIS_PRECISION_CERTIFIED;
  int64_t redo_pixels = 0;       // pixels the certified blend handed to the fp64 redo
  double batch_budget = 0.0;     // bytes of per-(view, particle) state one batch may use
  int64_t rescored_views = 0;    // candidates re-scored exactly to certify an argmax
  std::recursive_mutex mu;

  void use() { CK(cudaSetDevice(device)); }

  void* buf(const std::string& name, size_t bytes) {
    DevBuf& b = bufs[bufset ? name + "#1" : name];
    if (bytes == 0) bytes = 16;
    if (b.bytes < bytes) {
      if (b.p) CK(cudaFree(b.p));
      size_t want = bytes + bytes / 4;
      cudaError_t e = cudaMalloc(&b.p, want);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        b.p = nullptr;
        b.bytes = 0;
        throw DevErr("cudaMalloc(" + std::to_string(want) + ") for '" + name +
                     "' failed: " + cudaGetErrorString(e));
      }
      b.bytes = want;
    }
    return b.p;
  }

  // Stream-ordered allocations from the device pool (released to the pool, not
  // the driver: repeated scene/field uploads do not pay cudaMalloc/cudaFree).
  void* dalloc(size_t bytes, const char* what) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, std::max<size_t>(bytes, 16), stream);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      throw DevErr(std::string("cudaMallocAsync(") + std::to_string(bytes) + ") for " + what +
                   " failed: " + cudaGetErrorString(e));
    }
    return p;
  }
  void dfree(void* p) {
    if (p) cudaFreeAsync(p, stream);
  }

  cudaEvent_t event() {
    if (!spare_events.empty()) {
      cudaEvent_t e = spare_events.back();
      spare_events.pop_back();
      return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }

  template <class F>
  void run(const char* name, F&& launch, int nlaunch = 1, cudaStream_t st = nullptr) {
    if (!st) st = stream;
    cudaEvent_t a = nullptr, b = nullptr;
    if (profiling) {
      a = event();
      b = event();
      CK(cudaEventRecord(a, st));
    }
    launch();
    CK(cudaGetLastError());
    if (profiling) {
      CK(cudaEventRecord(b, st));
      pending.emplace_back(name, a, b);
    }
    launches += nlaunch;
  }

  // Collect the kernel timings whose events have completed (all when `all`).
  void collect(bool all) {
    std::vector<std::tuple<std::string, cudaEvent_t, cudaEvent_t>> keep;
    for (auto& p : pending) {
      if (!all && cudaEventQuery(std::get<2>(p)) != cudaSuccess) {
        (void)cudaGetLastError();
        keep.push_back(p);
        continue;
      }
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, std::get<1>(p), std::get<2>(p)));
      Timing& t = timing[std::get<0>(p)];
      t.ms += ms;
      t.launches += 1;
      spare_events.push_back(std::get<1>(p));
      spare_events.push_back(std::get<2>(p));
    }
    pending.swap(keep);
  }

  // The main stream (side-stream work of an in-flight UA batch may continue).
  void sync() {
    CK(cudaStreamSynchronize(stream));
    collect(false);
  }

  void sync_all() {
    CK(cudaStreamSynchronize(stream));
    if (side) CK(cudaStreamSynchronize(side));
    if (front) CK(cudaStreamSynchronize(front));
    collect(true);
  }
};

struct gavis_scene {
  gavis_ctx* ctx = nullptr;
  SceneDev dev;
  float4* pos_op = nullptr;
  float4* rot = nullptr;
  float4* scale = nullptr;
  uint8_t* virt = nullptr;
  float* colors = nullptr;
  uint4* colors_split = nullptr;  // tensor-core colour form, built on first certified RGB render
  float* var = nullptr;  // coefficient variances for the sh_propagation provider
  int var_degree = -1;
  float max_opacity = 1.f;  // enters the certified blend's error bound (q <= 2 ln(o / alpha))
};

struct gavis_field {
  gavis_ctx* ctx = nullptr;
  const gavis_scene* scene = nullptr;
  int64_t n = 0;
  int degree = 0;
  double kappa = 1.0;
  int num_views = 0;
  double* gamma = nullptr;
};

namespace {

DevCam make_devcam(const gavis_camera& c, int ts, int64_t tile_base, int64_t pix_base) {
  DevCam d;
  std::memcpy(d.R, c.rotation, sizeof(d.R));
  std::memcpy(d.pos, c.position, sizeof(d.pos));
  d.fx = 0.5 * c.width / std::tan(0.5 * c.fov_h);
  d.fy = 0.5 * c.height / std::tan(0.5 * c.fov_v);
  d.cx = 0.5 * c.width;
  d.cy = 0.5 * c.height;
  d.limx = 1.3 * std::tan(0.5 * c.fov_h);
  d.limy = 1.3 * std::tan(0.5 * c.fov_v);
  d.near_plane = c.near_plane;
  d.width = c.width;
  d.height = c.height;
  d.tiles_x = (c.width + ts - 1) / ts;
  d.tiles_y = (c.height + ts - 1) / ts;
  d.tile_base = tile_base;
  d.pix_base = pix_base;
  return d;
}

int batch_views(gavis_ctx* c, int64_t N, int n_views) {
  int vmax = c->max_batch > 0 ? c->max_batch : 32;
  if (N > 0) {
    // ~112 B of per-(view, particle) state per batch, two batches in flight: one
    // batch may use a sixth of the free device memory, within [2, 16] GB
    if (c->batch_budget == 0.0) {
      size_t free_b = 0, total_b = 0;
      CK(cudaMemGetInfo(&free_b, &total_b));
      c->batch_budget = std::min(16.0e9, std::max(2.0e9, (double)free_b / 6.0));
    }
    const int64_t by_mem = (int64_t)(c->batch_budget / (112.0 * (double)N));
    vmax = (int)std::max<int64_t>(1, std::min<int64_t>(vmax, by_mem));
  }
  vmax = std::min(vmax, 64);
  return std::max(1, std::min(vmax, n_views));
}

struct Binned {
  int V = 0;
  int64_t K = 0;
  int64_t total_tiles = 0;
  int64_t total_pix = 0;
  DevCam* dcams = nullptr;
  std::vector<DevCam> hcams;
  GeoRec* geo = nullptr;
  UaRec* ua = nullptr;
  int32_t* counts = nullptr;
  int32_t* offsets = nullptr;
  uint64_t* keys = nullptr;
  uint32_t* vals = nullptr;
  uint32_t* pair_gid = nullptr;
  uint2* ranges = nullptr;
  bool narrow = false;  // keys are 32-bit (local tile << rb | depth rank); b.keys == null
};

// pinned host scratch layout (int32 words)
constexpr int kPinItems = 4;
constexpr int kPinRedo = 6;     // u64
constexpr int kPinStarts = 16;  // int64 [V + 1] (V <= 64)
constexpr int kPinWords = 256;

struct BinOpts {
  bool vf_mode = false;
  bool ua = false;
  bool write_culled = false;
  const gavis_field* field = nullptr;
  const double* vis_given_dev = nullptr;
  double beta = 0.5, o0b = 0.075;
  double hl_const = 0.0;
  const float* var = nullptr;
  int var_degree = -1;
  int* err_flag = nullptr;
  bool force_wide = false;  // 64-bit (tile << 32 | fp32 depth) keys (reference-form debug keys)
};

// K1..K5 for one batch of cameras.
Binned bin_batch(gavis_ctx* c, const gavis_scene* s, const gavis_camera* cams, int V,
                 const gavis_raster_config* rc, const BinOpts& o) {
  Binned b;
  b.V = V;
  const int64_t N = s->dev.n;
  const int ts = rc->tile_size;
  int64_t tile_base = 0, pix_base = 0;
  for (int v = 0; v < V; ++v) {
    DevCam d = make_devcam(cams[v], ts, tile_base, pix_base);
    tile_base += (int64_t)d.tiles_x * d.tiles_y;
    pix_base += (int64_t)cams[v].width * cams[v].height;
    b.hcams.push_back(d);
  }
  b.total_tiles = tile_base;
  b.total_pix = pix_base;
  invariant(b.total_tiles < (int64_t(1) << 31), "too many tiles in one batch");
  b.dcams = (DevCam*)c->buf("cams", sizeof(DevCam) * V);
  CK(cudaMemcpyAsync(b.dcams, b.hcams.data(), sizeof(DevCam) * V, cudaMemcpyHostToDevice,
                     c->stream));
  const int64_t VN = (int64_t)V * N;
  b.geo = (GeoRec*)c->buf("geo", sizeof(GeoRec) * VN);
  if (o.ua) b.ua = (UaRec*)c->buf("ua", sizeof(UaRec) * VN);
  b.counts = (int32_t*)c->buf("counts", sizeof(int32_t) * (VN + 1));
  b.offsets = (int32_t*)c->buf("offsets", sizeof(int32_t) * (VN + 1));
  uint2* trect = (uint2*)c->buf("trect", sizeof(uint2) * VN);

  PreprocessArgs pa;
  pa.scene = s->dev;
  pa.cams = b.dcams;
  pa.V = V;
  pa.dilation = rc->dilation;
  pa.tile_size = ts;
  pa.geo = b.geo;
  pa.ua = b.ua;
  pa.counts = b.counts;
  pa.trect = trect;
  pa.write_culled = o.write_culled;
  pa.beta = o.beta;
  pa.o0b = o.o0b;
  pa.hl_const = o.hl_const;
  pa.var = o.var;
  pa.var_degree = o.var_degree;
  pa.err_flag = o.err_flag;
  if (o.ua) {
    if (o.vis_given_dev) {
      pa.query_mode = kQueryGiven;
      pa.vis_in = o.vis_given_dev;
    } else if (o.field) {
      pa.query_mode = kQueryField;
      pa.gamma = o.field->gamma;
      pa.degree = o.field->degree;
      pa.num_views = o.field->num_views;
    }
  }
  c->run("preprocess", [&] { launch_preprocess(pa, c->stream); }, N > 0 ? 1 : 0);

  // GAVIS_BIN_WIDE=1 selects the 64-bit (tile << 32 | fp32 depth) key path (A/B and
  // the equivalence test); it is also the path of the reference-form debug keys
  const char* wide_env = std::getenv("GAVIS_BIN_WIDE");
  const bool narrow = !o.force_wide && !(wide_env && wide_env[0] == '1');
  int32_t* P32 = c->pinned;
  int64_t K = 0, n_items = 0;
  NarrowArgs na;
  if (VN > 0 && narrow) {
    // visible items -> sorted by (view, depth) -> tile counts in that order -> pair offsets
    uint32_t* items = (uint32_t*)c->buf("items", sizeof(uint32_t) * VN);
    int32_t* dnum = (int32_t*)c->buf("items_num", sizeof(int32_t));
    const size_t selb = select_temp_bytes(VN);
    void* seltmp = c->buf("select_tmp", selb);
    c->run("select", [&] { select_visible(b.counts, VN, items, dnum, seltmp, selb, c->stream); });
    CK(cudaMemcpyAsync(P32 + kPinItems, dnum, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    n_items = P32[kPinItems];
    na.N = N;
    na.geo = b.geo;
    na.counts = b.counts;
    na.n_items = n_items;
    na.item_slot = items;
    if (n_items > 0) {
      uint32_t* ik_a = (uint32_t*)c->buf("item_key_a", sizeof(uint32_t) * n_items);
      uint32_t* ik_b = (uint32_t*)c->buf("item_key_b", sizeof(uint32_t) * n_items);
      uint32_t* is_b = (uint32_t*)c->buf("item_slot_b", sizeof(uint32_t) * n_items);
      na.item_key = ik_a;
      na.view_bits = std::max(1, bits_for(V));
      c->run("item_keys", [&] { launch_item_keys(na, c->stream); });
      const size_t isb = sort32_temp_bytes(n_items);
      void* itmp = c->buf("sort_tmp", isb);
      c->run("sort", [&] {
        radix_sort_pairs32(ik_a, ik_b, items, is_b, n_items, 32, itmp, isb, c->stream);
      });
      na.item_slot_sorted = items;
      na.item_count = (int32_t*)c->buf("item_count", sizeof(int32_t) * (n_items + 1));
      int32_t* ioff = (int32_t*)c->buf("item_offset", sizeof(int32_t) * (n_items + 1));
      CK(cudaMemsetAsync(na.item_count + n_items, 0, sizeof(int32_t), c->stream));
      c->run("depth_order", [&] { launch_depth_order(na, c->stream); });
      const size_t scb = scan_temp_bytes(n_items + 1);
      void* stmp = c->buf("scan_tmp", scb);
      c->run("scan", [&] { exclusive_scan(na.item_count, ioff, n_items + 1, stmp, scb, c->stream); });
      na.item_offset = ioff;
      na.view_bits = std::max(1, bits_for(V));
      int64_t* dstarts = (int64_t*)c->buf("view_pair_starts", sizeof(int64_t) * (V + 1));
      c->run("depth_order", [&] { launch_view_pair_starts(na, V, dstarts, c->stream); });
      CK(cudaMemcpyAsync(c->pinned + kPinStarts, dstarts, sizeof(int64_t) * (V + 1),
                         cudaMemcpyDeviceToHost, c->stream));
      c->sync();
      K = reinterpret_cast<int64_t*>(c->pinned + kPinStarts)[V];
    }
  } else if (VN > 0) {
    const size_t sb = scan_temp_bytes(VN);
    void* tmp = c->buf("scan_tmp", sb);
    c->run("scan", [&] { exclusive_scan(b.counts, b.offsets, VN, tmp, sb, c->stream); });
    CK(cudaMemcpyAsync(P32, b.offsets + VN - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(P32 + 1, b.counts + VN - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    K = (int64_t)P32[0] + (int64_t)P32[1];
  }
  invariant(K >= 0 && K < (int64_t(1) << 31), "pair count overflow in one batch");
  b.K = K;

  uint32_t* va = (uint32_t*)c->buf("vals_a", sizeof(uint32_t) * K);
  uint32_t* vb = (uint32_t*)c->buf("vals_b", sizeof(uint32_t) * K);
  if (o.vf_mode) b.pair_gid = (uint32_t*)c->buf("pair_gid", sizeof(uint32_t) * K);
  b.ranges = (uint2*)c->buf("ranges", sizeof(uint2) * std::max<int64_t>(1, b.total_tiles));
  CK(cudaMemsetAsync(b.ranges, 0, sizeof(uint2) * b.total_tiles, c->stream));
  EmitArgs ea;
  ea.cams = b.dcams;
  ea.V = V;
  ea.N = N;
  ea.geo = b.geo;
  ea.counts = b.counts;
  ea.offsets = b.offsets;
  ea.trect = trect;
  ea.vals = va;
  ea.pair_gid = b.pair_gid;
  if (narrow && K > 0) {
    b.narrow = true;
    uint32_t* k32a = (uint32_t*)c->buf("keys32_a", sizeof(uint32_t) * K);
    uint32_t* k32b = (uint32_t*)c->buf("keys32_b", sizeof(uint32_t) * K);
    na.keys32 = k32a;
    na.slot_offset = b.offsets;  // per-slot pair offsets (VF finalize)
    // chunks of consecutive views with <= 2^16 tiles: 16-bit local tile keys, two
    // 8-bit radix passes per chunk (the pairs of a chunk are contiguous: views
    // were emitted in order)
    const int64_t* vstart = reinterpret_cast<const int64_t*>(c->pinned + kPinStarts);
    std::vector<int> chunk_first;
    std::vector<int64_t> hbase((size_t)V);
    int64_t acc = 0;
    for (int v = 0; v < V; ++v) {
      const int64_t tv = (int64_t)b.hcams[v].tiles_x * b.hcams[v].tiles_y;
      if (v == 0 || acc + tv > (int64_t(1) << 16)) {
        chunk_first.push_back(v);
        acc = 0;
      }
      acc += tv;
      hbase[v] = b.hcams[chunk_first.back()].tile_base;
    }
    chunk_first.push_back(V);
    int64_t* dbase = (int64_t*)c->buf("chunk_tile_base", sizeof(int64_t) * V);
    CK(cudaMemcpyAsync(dbase, hbase.data(), sizeof(int64_t) * V, cudaMemcpyHostToDevice, c->stream));
    na.chunk_tile_base = dbase;
    c->run("emit_keys", [&] { launch_emit_tiles(ea, na, c->stream); });
    const size_t sb32 = sort32_temp_bytes(K);
    void* tmp = c->buf("sort32_tmp", sb32);
    for (size_t k = 0; k + 1 < chunk_first.size(); ++k) {
      const int v0 = chunk_first[k], v1 = chunk_first[k + 1];
      const int64_t lo = vstart[v0], hi = vstart[v1];
      const int64_t tiles = b.hcams[v1 - 1].tile_base +
                            (int64_t)b.hcams[v1 - 1].tiles_x * b.hcams[v1 - 1].tiles_y -
                            b.hcams[v0].tile_base;
      c->run("sort", [&] {
        radix_sort_pairs32(k32a + lo, k32b + lo, va + lo, vb + lo, hi - lo,
                           std::max(1, bits_for(tiles)), tmp, sb32, c->stream);
      });
      c->run("ranges", [&] {
        launch_ranges32(k32a, lo, hi, b.hcams[v0].tile_base, b.ranges, c->stream);
      });
    }
    b.vals = va;
    b.keys = nullptr;
  } else if (K > 0) {
    uint64_t* ka = (uint64_t*)c->buf("keys_a", sizeof(uint64_t) * K);
    uint64_t* kb = (uint64_t*)c->buf("keys_b", sizeof(uint64_t) * K);
    ea.keys = ka;
    c->run("emit_keys", [&] { launch_emit_keys(ea, c->stream); });
    const size_t sb = sort_temp_bytes(K);
    void* tmp = c->buf("sort_tmp", sb);
    const int end_bit = 32 + std::max(1, bits_for(b.total_tiles));
    c->run("sort", [&] {
      radix_sort_pairs(ka, kb, va, vb, K, end_bit, tmp, sb, c->stream, &b.keys, &b.vals);
    });
    RangesArgs ra;
    ra.cams = b.dcams;
    ra.V = V;
    ra.N = N;
    ra.K = K;
    ra.keys = b.keys;
    ra.vals = b.vals;
    ra.pair_gid = b.pair_gid;
    ra.geo = b.geo;
    ra.ranges = b.ranges;
    c->run("ranges", [&] { launch_ranges(ra, c->stream); });
  } else {
    b.vals = va;
  }
  return b;
}

void check_scene_field(const gavis_scene* s, const gavis_field* f) {
  require(s != nullptr, "scene must not be null");
  if (f) require(f->n == s->dev.n, "field was built for a different scene");
}

// VF accumulation of views [0, n) into field (or only per-view outputs).
// Optional per-batch consumer of the device visibilities: density control's
// unseen[k] *= 1 - b[n_real + k], views in trajectory order (vfield.hpp:187-190).
struct DensityHook {
  double* unseen = nullptr;  // device [n_virtual]
  int64_t n_real = 0, n_virtual = 0;
};

void vf_views(gavis_ctx* c, const gavis_scene* s, gavis_field* f, const gavis_camera* views,
              int n_views, const gavis_raster_config* rc, double* vis_host, int64_t* touch_host,
              int32_t* contrib_host, const DensityHook* dh = nullptr) {
  const int64_t N = s->dev.n;
  const int bv = batch_views(c, N, n_views);
  double scales[kMaxFieldDegree + 1] = {0};
  if (f) vmf_scales(f->kappa, f->degree, scales);
  // binning of batch k+1 on the front stream under batch k's blend (as ua_render)
  cudaStream_t main_stream = c->stream;
  struct Restore {
    gavis_ctx* c;
    cudaStream_t main;
    ~Restore() {
      c->bufset = 0;
      c->stream = main;
    }
  } restore{c, main_stream};
  CK(cudaEventRecord(c->ev_done[0], main_stream));
  CK(cudaStreamWaitEvent(c->front, c->ev_done[0], 0));
  const bool host_out = vis_host || touch_host || contrib_host;
  int batch = 0;
  for (int v0 = 0; v0 < n_views; v0 += bv, ++batch) {
    const int V = std::min(bv, n_views - v0);
    const int par = batch & 1;
    c->bufset = par;
    c->stream = c->front;
    if (batch >= 2) CK(cudaStreamWaitEvent(c->front, c->ev_done[par], 0));
    BinOpts o;
    o.vf_mode = true;
    Binned b = bin_batch(c, s, views + v0, V, rc, o);
    CK(cudaEventRecord(c->ev_bin[par], c->front));
    c->stream = main_stream;
    CK(cudaStreamWaitEvent(c->stream, c->ev_bin[par], 0));
    double* psum = (double*)c->buf("pair_sum", sizeof(double) * b.K);
    int32_t* pcnt = (int32_t*)c->buf("pair_cnt", sizeof(int32_t) * b.K);
    if (b.K > 0) {
      CK(cudaMemsetAsync(psum, 0, sizeof(double) * b.K, c->stream));
      CK(cudaMemsetAsync(pcnt, 0, sizeof(int32_t) * b.K, c->stream));
    }
    int32_t* dcontrib = nullptr;
    if (contrib_host) dcontrib = (int32_t*)c->buf("contrib", sizeof(int32_t) * b.total_pix);
    VfBlendArgs va;
    va.cams = b.dcams;
    va.V = V;
    va.N = N;
    va.total_tiles = b.total_tiles;
    va.tile_size = rc->tile_size;
    va.cutoff = rc->transmittance_cutoff;
    va.amax = rc->alpha_clamp_max;
    va.geo = b.geo;
    va.ranges = b.ranges;
    va.vals = b.vals;
    va.pair_gid = b.pair_gid;
    va.pair_sum = psum;
    va.pair_cnt = pcnt;
    va.contrib = dcontrib;
    if (b.K > 0 || dcontrib) c->run("vf_blend", [&] { launch_vf_blend(va, c->stream); });
    VfFinalizeArgs fa;
    fa.scene = s->dev;
    fa.cams = b.dcams;
    fa.V = V;
    fa.counts = b.counts;
    fa.offsets = b.offsets;
    fa.pair_sum = psum;
    fa.pair_cnt = pcnt;
    fa.gamma = f ? f->gamma : nullptr;
    fa.degree = f ? f->degree : 0;
    std::memcpy(fa.scales, scales, sizeof(scales));
    if (vis_host || dh) fa.vis_out = (double*)c->buf("vis_out", sizeof(double) * V * std::max<int64_t>(1, N));
    if (touch_host)
      fa.touch_out = (int64_t*)c->buf("touch_out", sizeof(int64_t) * V * std::max<int64_t>(1, N));
    c->run("vf_finalize", [&] { launch_vf_finalize(fa, N, c->stream); }, N > 0 ? 1 : 0);
    if (dh && dh->n_virtual > 0)
      c->run("density", [&] {
        launch_density_update(dh->unseen, fa.vis_out, V, N, dh->n_real, dh->n_virtual, c->stream);
      });
    if (vis_host && N > 0)
      CK(cudaMemcpyAsync(vis_host + (int64_t)v0 * N, fa.vis_out, sizeof(double) * V * N,
                         cudaMemcpyDeviceToHost, c->stream));
    if (touch_host && N > 0)
      CK(cudaMemcpyAsync(touch_host + (int64_t)v0 * N, fa.touch_out, sizeof(int64_t) * V * N,
                         cudaMemcpyDeviceToHost, c->stream));
    if (contrib_host)
      CK(cudaMemcpyAsync(contrib_host, dcontrib, sizeof(int32_t) * b.total_pix,
                         cudaMemcpyDeviceToHost, c->stream));
    CK(cudaEventRecord(c->ev_done[par], c->stream));
    if (host_out) c->sync();
  }
  c->bufset = 0;
  c->sync_all();
  if (f) f->num_views += n_views;
}

void copy_out(gavis_ctx* c, double* host, const double* dev, int64_t count,
              cudaStream_t st = nullptr) {
  if (host && count > 0)
    CK(cudaMemcpyAsync(host, dev, sizeof(double) * count, cudaMemcpyDeviceToHost,
                       st ? st : c->stream));
}

// Certification window of the fp32 blend, relative to the cutoff: twice the
// bound u (16 + 3.2 k + 22 S) derived in kernels_ua_fast.cu (k composited
// entries, S = sum a/(1-a) over them).
// Opacities above 1 (not excluded by the reference) weaken the alpha-error
// bounds (q <= 2 ln(o_max / a); A a (1.5 q + 8) <= 8 o_max A): the S coefficient
// becomes 22 o_max + 6 ln(o_max) (22 for o_max <= 1).
void cert_window(UaBlendArgs* ua, float max_opacity) {
  const double u = std::ldexp(1.0, -24);
  const double om = std::max(1.0, (double)max_opacity);
  ua->cert_base = (float)(2.0 * u * 16.0);
  ua->cert_per_step = (float)(2.0 * u * 3.2);
  ua->cert_sum = (float)(2.0 * u * (22.0 * om + 6.0 * std::log(om)));
  ua->cert_per_step2 = (float)(2.0 * u * (1.004 + 3e-4 * std::log(om)));
  ua->cert_sum2 = (float)(2.0 * u * (41.0 + 3.0 * std::log(om)) * om);
  // test hook (tests/test_certified.py): hand every pixel to the fp64 redo
  const char* force = std::getenv("GAVIS_CERT_FORCE_REDO");
  if (force && force[0] == '1') ua->cert_base = 3.0e38f;
  // timing hook only (uncertified results): flag no pixel, to measure what the
  // redo costs the step
  if (force && force[0] == 'n') {
    ua->cert_base = ua->cert_per_step = ua->cert_sum = 0.0f;
    ua->cert_per_step2 = ua->cert_sum2 = 0.0f;
  }
}

void ua_render(gavis_ctx* c, const gavis_scene* s, const gavis_field* f, const double* vis_host,
               const gavis_camera* cams, int n, const gavis_raster_config* rc,
               const gavis_uncertainty_config* uc, gavis_render_outputs* out) {
  validate_raster(rc);
  double hl_q0 = 0.0;
  validate_unc(uc, &hl_q0);
  require(cams != nullptr || n == 0, "cameras must not be null");
  require(out != nullptr, "render outputs must not be null");
  check_scene_field(s, f);
  for (int i = 0; i < n; ++i) validate_camera(cams[i]);
  const int64_t N = s->dev.n;
  const bool do_rgb = out->rgb || out->depth || out->transmittance || out->rgb_contributors ||
                      out->with_rgb;
  const bool do_ent = out->entropy || out->invisible_mass || out->entropy_depth || out->scores ||
                      out->entropy_contributors || out->with_entropy;
  if (!do_rgb && !do_ent) return;
  const double* vis_dev = nullptr;
  if (!f) {
    require(vis_host != nullptr || N == 0 || !do_ent,
            "render needs a field or per-particle splat visibility");
    if (vis_host && N > 0) {
      double* d = (double*)c->buf("vis_given", sizeof(double) * N);
      CK(cudaMemcpyAsync(d, vis_host, sizeof(double) * N, cudaMemcpyHostToDevice, c->stream));
      vis_dev = d;
    }
  }
  const int bv = batch_views(c, N, n);
  const bool fast = c->precision == GAVIS_PRECISION_CERTIFIED &&
                    ua_fast_supported(rc->tile_size, rc->alpha_clamp_max);
  if (fast && do_rgb && !s->colors_split) {
    // the staged colour records of the tensor-core colour path, once per scene
    // (scenes are immutable once built; calls on a context are serialised)
    const size_t bytes = ua_colors_split_bytes(s->dev);
    if (bytes > 0) {
      auto* ms = const_cast<gavis_scene*>(s);
      ms->colors_split = (uint4*)c->dalloc(bytes, "scene colour splits");
      ms->dev.colors_split = ms->colors_split;
      c->run("split_colors", [&] { launch_split_colors(ms->dev, ms->colors_split, c->stream); });
    }
  }
  unsigned long long* redo_total = nullptr;
  if (fast) {
    redo_total = (unsigned long long*)c->buf("redo_total", sizeof(unsigned long long));
    CK(cudaMemsetAsync(redo_total, 0, sizeof(unsigned long long), c->stream));
  }
  if (out->scores && n > c->pin_scores_cap) {
    c->sync_all();
    if (c->pin_scores) CK(cudaFreeHost(c->pin_scores));
    c->pin_scores = nullptr;
    c->pin_scores_cap = 0;
    CK(cudaMallocHost(&c->pin_scores, sizeof(double) * n));
    c->pin_scores_cap = n;
  }
  CK(cudaEventRecord(c->ev_done[0], c->stream));  // side / front work start after this point
  CK(cudaStreamWaitEvent(c->side, c->ev_done[0], 0));
  CK(cudaStreamWaitEvent(c->front, c->ev_done[0], 0));
  cudaStream_t main_stream = c->stream;
  struct BufsetReset {
    gavis_ctx* c;
    cudaStream_t main;
    ~BufsetReset() {
      c->bufset = 0;
      c->stream = main;
    }
  } reset{c, main_stream};
  int64_t pix_done = 0;
  int batch = 0;
  for (int v0 = 0; v0 < n; v0 += bv, ++batch) {
    const int V = std::min(bv, n - v0);
    const int par = batch & 1;
    c->bufset = par;
    // binning runs on the front stream, under the previous batch's blend; the
    // buffers of this set were last read by batch - 2's side-stream work
    c->stream = c->front;
    if (batch >= 2) CK(cudaStreamWaitEvent(c->front, c->ev_done[par], 0));
    BinOpts o;
    o.ua = do_ent;
    o.field = f;
    o.vis_given_dev = vis_dev;
    o.beta = uc->beta;
    o.o0b = uc->prior_opacity * (1.0 - uc->beta);
    o.hl_const = 3.0 * std::log(uc->color_sigma);  // 0.5 log(sigma^6), uncertainty.hpp:145
    int* err = nullptr;
    if (do_ent && uc->variance_provider == 1) {
      require(s->var != nullptr || s->dev.n == 0,
              "variance_provider sh_propagation requires coeff_variances");
      o.var = s->var;
      o.var_degree = s->var_degree;
      err = (int*)c->buf("err_flag", sizeof(int));
      CK(cudaMemsetAsync(err, 0, sizeof(int), c->stream));
      o.err_flag = err;
    }
    Binned b = bin_batch(c, s, cams + v0, V, rc, o);
    if (err) {
      CK(cudaMemcpyAsync(c->pinned + 2, err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      c->sync();
      require(c->pinned[2] == 0, "propagated color variance must be positive");
    }
    CK(cudaEventRecord(c->ev_bin[par], c->front));
    c->stream = main_stream;
    CK(cudaStreamWaitEvent(c->stream, c->ev_bin[par], 0));
    const int64_t P = b.total_pix;
    UaBlendArgs ua;
    ua.scene = s->dev;
    ua.cams = b.dcams;
    ua.V = V;
    ua.total_tiles = b.total_tiles;
    ua.tile_size = rc->tile_size;
    ua.cutoff = rc->transmittance_cutoff;
    ua.amax = rc->alpha_clamp_max;
    ua.hl_qc = 3.0 * std::log(uc->color_sigma);
    ua.hl_q0 = hl_q0;
    ua.corr_lambda = uc->correlation == 1 ? uc->correlation_lambda : 0.0;
    ua.geo = b.geo;
    ua.ua = b.ua;
    ua.ranges = b.ranges;
    ua.vals = b.vals;
    ua.do_rgb = do_rgb;
    ua.do_ent = do_ent;
    // The RGB and entropy images always land in device memory (host copies only
    // when requested; the score folds the entropy image); depth and
    // residual-transmittance maps only on request.
    if (do_rgb) {
      ua.rgb = (double*)c->buf("img_rgb", sizeof(double) * 3 * P);
      ua.depth = out->depth ? (double*)c->buf("img_depth", sizeof(double) * P) : nullptr;
      ua.trans = out->transmittance ? (double*)c->buf("img_trans", sizeof(double) * P) : nullptr;
      if (out->rgb_contributors) ua.rgb_contrib = (int32_t*)c->buf("img_nrgb", sizeof(int32_t) * P);
    }
    if (do_ent) {
      ua.entropy = (double*)c->buf("img_entropy", sizeof(double) * P);
      ua.w0 = (double*)c->buf("img_w0", sizeof(double) * P);
      ua.edepth = (out->entropy_depth || ua.corr_lambda > 0.0)
                      ? (double*)c->buf("img_edepth", sizeof(double) * P)
                      : nullptr;
      if (out->entropy_contributors)
        ua.ent_contrib = (int32_t*)c->buf("img_nent", sizeof(int32_t) * P);
    }
    cudaStream_t side = c->side;
    if (fast && b.total_tiles > 0) {
      invariant(P < (int64_t(1) << 32), "too many pixels in one batch");
      ua.flag_list = (uint32_t*)c->buf("flag_list", sizeof(uint32_t) * P);
      ua.flag_count = (uint32_t*)c->buf("flag_count", sizeof(uint32_t));
      CK(cudaMemsetAsync(ua.flag_count, 0, sizeof(uint32_t), c->stream));
      cert_window(&ua, s->max_opacity);
      c->run("ua_blend", [&] { launch_ua_blend_fast(ua, c->stream); });
      CK(cudaEventRecord(c->ev_blend[par], c->stream));
      CK(cudaStreamWaitEvent(side, c->ev_blend[par], 0));
      c->run("ua_redo", [&] { launch_ua_redo(ua, side); }, 1, side);
      launch_add_count(redo_total, ua.flag_count, side);
    } else {
      c->run("ua_blend", [&] { launch_ua_blend(ua, c->stream); }, b.total_tiles > 0 ? 1 : 0);
      CK(cudaEventRecord(c->ev_blend[par], c->stream));
      CK(cudaStreamWaitEvent(side, c->ev_blend[par], 0));
    }
    double* dscores = nullptr;
    if (do_ent) {
      dscores = (double*)c->buf("scores", sizeof(double) * V);
      double* part = (double*)c->buf("score_partial", sizeof(double) * V * score_partials_per_view());
      c->run("score", [&] {
        launch_score_image(b.dcams, V, ua.entropy, ua.edepth, ua.corr_lambda, part, dscores, side);
      }, 1, side);
    }
    copy_out(c, out->rgb ? out->rgb + 3 * pix_done : nullptr, ua.rgb, 3 * P, side);
    copy_out(c, out->depth ? out->depth + pix_done : nullptr, ua.depth, P, side);
    copy_out(c, out->transmittance ? out->transmittance + pix_done : nullptr, ua.trans, P, side);
    copy_out(c, out->entropy ? out->entropy + pix_done : nullptr, ua.entropy, P, side);
    copy_out(c, out->invisible_mass ? out->invisible_mass + pix_done : nullptr, ua.w0, P, side);
    copy_out(c, out->entropy_depth ? out->entropy_depth + pix_done : nullptr, ua.edepth, P, side);
    // scores through pinned staging: a D2H copy into pageable memory would block
    // the host on this batch's side-stream work and serialise the batches
    copy_out(c, out->scores ? c->pin_scores + v0 : nullptr, dscores, V, side);
    if (out->rgb_contributors)
      CK(cudaMemcpyAsync(out->rgb_contributors + pix_done, ua.rgb_contrib, sizeof(int32_t) * P,
                         cudaMemcpyDeviceToHost, side));
    if (out->entropy_contributors)
      CK(cudaMemcpyAsync(out->entropy_contributors + pix_done, ua.ent_contrib,
                         sizeof(int32_t) * P, cudaMemcpyDeviceToHost, side));
    CK(cudaEventRecord(c->ev_done[par], side));
    pix_done += P;
  }
  c->bufset = 0;
  // the main stream continues after the side stream's last batch
  CK(cudaEventRecord(c->ev_done[0], c->side));
  CK(cudaStreamWaitEvent(c->stream, c->ev_done[0], 0));
  if (redo_total) {
    CK(cudaMemcpyAsync(c->pinned + kPinRedo, redo_total, sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, c->stream));
  }
  c->sync_all();
  if (out->scores && n > 0) std::memcpy(out->scores, c->pin_scores, sizeof(double) * n);
  if (redo_total) c->redo_pixels += (int64_t)*reinterpret_cast<unsigned long long*>(c->pinned + kPinRedo);
}

// select_nbv's argmax (planner.hpp:132-136: first strictly greater score) over
// scores from the certified fp32 blend: every candidate within kCertScoreRel
// (relative) of the best is re-scored with the exact fp64 blend and the argmax
// is taken again, so it is the exact path's argmax (the fp32 scores agree with
// the fp64 ones to a few 1e-6 relative -- 3e-6 at config 3 -- over two orders of
// magnitude inside the window).
constexpr double kCertScoreRel = 1e-3;

int certified_first_max(gavis_ctx* c, const gavis_scene* s, const gavis_field* f,
                        const gavis_camera* cams, int n, const gavis_raster_config* rc,
                        const gavis_uncertainty_config* uc, std::vector<double>& sc) {
  auto first_max = [&] {
    int b = 0;
    for (int i = 1; i < n; ++i)
      if (sc[i] > sc[b]) b = i;
    return b;
  };
  int b = first_max();
  if (c->precision != GAVIS_PRECISION_CERTIFIED ||
      !ua_fast_supported(rc->tile_size, rc->alpha_clamp_max))
    return b;
  const double lo = sc[b] - kCertScoreRel * std::fabs(sc[b]);
  std::vector<int> cont;
  std::vector<gavis_camera> cc;
  for (int i = 0; i < n; ++i)
    if (sc[i] >= lo) {
      cont.push_back(i);
      cc.push_back(cams[i]);
    }
  if (cont.size() < 2) return b;
  std::vector<double> ex(cont.size());
  gavis_render_outputs o = {};
  o.scores = ex.data();
  c->precision = GAVIS_PRECISION_EXACT;
  try {
    ua_render(c, s, f, nullptr, cc.data(), (int)cc.size(), rc, uc, &o);
  } catch (...) {
    c->precision = GAVIS_PRECISION_CERTIFIED;
    throw;
  }
  c->precision = GAVIS_PRECISION_CERTIFIED;
  for (size_t k = 0; k < cont.size(); ++k) sc[cont[k]] = ex[k];
  c->rescored_views += (int64_t)cont.size();
  return first_max();
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int gavis_abi_version(void) { return GAVIS_ABI_VERSION; }

const char* gavis_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"

namespace gavis {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace gavis

extern "C" {

gavis_status gavis_ctx_create(int32_t device, void* stream, gavis_ctx** out) {
  return guard([&] {
    require(out != nullptr, "out must not be null");
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    require(device >= 0 && device < count, "device index out of range");
    auto* c = new gavis_ctx();
    c->device = device;
    try {
      c->use();
      if (stream) {
        c->stream = (cudaStream_t)stream;
      } else {
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
      }
      CK(cudaMallocHost(&c->pinned, sizeof(int32_t) * kPinWords));
      CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
      int lo_prio = 0, hi_prio = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
      CK(cudaStreamCreateWithPriority(&c->front, cudaStreamNonBlocking, hi_prio));
      for (int k = 0; k < 2; ++k) {
        CK(cudaEventCreateWithFlags(&c->ev_blend[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_done[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_bin[k], cudaEventDisableTiming));
      }
      // keep freed scene/field memory in the device pool between uploads
      cudaMemPool_t pool;
      CK(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t keep = UINT64_MAX;
      CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
      CK(cudaEventCreate(&c->t0));
      CK(cudaEventCreate(&c->t1));
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

gavis_status gavis_ctx_destroy(gavis_ctx* c) {
  return guard([&] {
    if (!c) return;
    c->use();
    cudaStreamSynchronize(c->stream);
    for (auto& kv : c->bufs)
      if (kv.second.p) cudaFree(kv.second.p);
    for (auto e : c->spare_events) cudaEventDestroy(e);
    for (auto& p : c->pending) {
      cudaEventDestroy(std::get<1>(p));
      cudaEventDestroy(std::get<2>(p));
    }
    if (c->t0) cudaEventDestroy(c->t0);
    if (c->t1) cudaEventDestroy(c->t1);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->pin_scores) cudaFreeHost(c->pin_scores);
    for (cudaStream_t st : {c->side, c->front})
      if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
      }
    for (int k = 0; k < 2; ++k) {
      if (c->ev_blend[k]) cudaEventDestroy(c->ev_blend[k]);
      if (c->ev_done[k]) cudaEventDestroy(c->ev_done[k]);
      if (c->ev_bin[k]) cudaEventDestroy(c->ev_bin[k]);
    }
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
  });
}

gavis_status gavis_ctx_synchronize(gavis_ctx* c) {
  return guard([&] {
    require(c != nullptr, "context must not be null");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    c->sync_all();
  });
}

gavis_status gavis_ctx_set_batch(gavis_ctx* c, int32_t n) {
  return guard([&] {
    require(c != nullptr, "context must not be null");
    require(n >= 0 && n <= 64, "batch must lie in [0, 64]");
    c->max_batch = n;
  });
}

gavis_status gavis_ctx_set_precision(gavis_ctx* c, int32_t precision) {
  return guard([&] {
    require(c != nullptr, "context must not be null");
    require(precision == GAVIS_PRECISION_CERTIFIED || precision == GAVIS_PRECISION_EXACT,
            "precision must be GAVIS_PRECISION_CERTIFIED or GAVIS_PRECISION_EXACT");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->precision = precision;
  });
}

gavis_status gavis_ctx_get_counters(gavis_ctx* c, int64_t* redo_pixels, int64_t* rescored_views) {
  return guard([&] {
    require(c != nullptr, "context must not be null");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    if (redo_pixels) *redo_pixels = c->redo_pixels;
    if (rescored_views) *rescored_views = c->rescored_views;
  });
}

gavis_status gavis_ctx_set_profiling(gavis_ctx* c, int32_t enabled) {
  return guard([&] {
    require(c != nullptr, "context must not be null");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    c->sync_all();
    c->profiling = enabled != 0;
  });
}

gavis_status gavis_ctx_kernel_time(gavis_ctx* c, const char* kernel, double* ms,
                                   int64_t* launches, int32_t reset) {
  return guard([&] {
    require(c != nullptr && kernel != nullptr, "context and kernel name must not be null");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    c->sync_all();
    Timing t;
    auto it = c->timing.find(kernel);
    if (it != c->timing.end()) t = it->second;
    if (ms) *ms = t.ms;
    if (launches) *launches = t.launches;
    if (reset) c->timing.erase(kernel);
  });
}

gavis_status gavis_ctx_timer_start(gavis_ctx* c) {
  return guard([&] {
    require(c != nullptr, "context must not be null");
    c->use();
    CK(cudaEventRecord(c->t0, c->stream));
  });
}

gavis_status gavis_ctx_timer_stop(gavis_ctx* c, double* ms) {
  return guard([&] {
    require(c != nullptr && ms != nullptr, "context and ms must not be null");
    c->use();
    CK(cudaEventRecord(c->t1, c->stream));
    CK(cudaEventSynchronize(c->t1));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, c->t0, c->t1));
    *ms = f;
  });
}

gavis_status gavis_ctx_launch_count(gavis_ctx* c, int64_t* launches) {
  return guard([&] {
    require(c != nullptr && launches != nullptr, "context and out must not be null");
    *launches = c->launches;
  });
}

gavis_status gavis_nbv_loop(gavis_ctx* c, const gavis_scene* s, gavis_field* f,
                            const gavis_camera* cams, int32_t n_cams, int32_t steps,
                            const gavis_raster_config* rc, const gavis_uncertainty_config* uc,
                            int32_t with_rgb, int32_t* chosen, double* scores,
                            double* all_scores) {
  return guard([&] {
    require(c && s && f, "null argument");
    require(n_cams > 0 && cams != nullptr, "select_nbv: candidate list must be nonempty");
    require(steps >= 0, "steps must be non-negative");
    invariant(f->n == s->dev.n, "accumulate_view: field/scene particle count mismatch");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    std::vector<double> sc((size_t)n_cams);
    for (int step = 0; step < steps; ++step) {
      gavis_render_outputs o = {};
      o.scores = sc.data();
      o.with_rgb = with_rgb;
      ua_render(c, s, f, nullptr, cams, n_cams, rc, uc, &o);
      const int b = certified_first_max(c, s, f, cams, n_cams, rc, uc, sc);  // planner.hpp:132-136
      vf_views(c, s, f, cams + b, 1, rc, nullptr, nullptr, nullptr);
      if (chosen) chosen[step] = b;
      if (scores) scores[step] = sc[b];
      if (all_scores) std::memcpy(all_scores + (int64_t)step * n_cams, sc.data(), sizeof(double) * n_cams);
    }
  });
}

// Device scene with room for n particles (arrays uninitialised).
static gavis_scene* alloc_scene(gavis_ctx* c, int64_t n, int color_degree) {
  auto* s = new gavis_scene();
  s->ctx = c;
  const int nb = (color_degree + 1) * (color_degree + 1);
  const int nbp = nb + (nb & 1);
  const int cstride = ((3 * nbp + 3) / 4) * 4;
  const int64_t M = std::max<int64_t>(n, 1);
  try {
    s->pos_op = (float4*)c->dalloc(sizeof(float4) * M, "scene");
    s->rot = (float4*)c->dalloc(sizeof(float4) * M, "scene");
    s->scale = (float4*)c->dalloc(sizeof(float4) * M, "scene");
    s->virt = (uint8_t*)c->dalloc(M, "scene");
    s->colors = (float*)c->dalloc(sizeof(float) * cstride * M, "scene");
  } catch (...) {
    c->dfree(s->pos_op);
    c->dfree(s->rot);
    c->dfree(s->scale);
    c->dfree(s->virt);
    c->dfree(s->colors);
    delete s;
    throw;
  }
  s->dev.n = n;
  s->dev.color_degree = color_degree;
  s->dev.nb = nb;
  s->dev.cstride = cstride;
  s->dev.pos_op = s->pos_op;
  s->dev.rot = s->rot;
  s->dev.scale = s->scale;
  s->dev.virt = s->virt;
  s->dev.colors = s->colors;
  return s;
}

// Copies particles [0, n) of src into dst at offset `at` (device to device).
static void copy_particles(gavis_ctx* c, gavis_scene* dst, int64_t at, const gavis_scene* src,
                           int64_t n) {
  if (n == 0) return;
  const int cs = src->dev.cstride;
  CK(cudaMemcpyAsync(dst->pos_op + at, src->pos_op, sizeof(float4) * n, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemcpyAsync(dst->rot + at, src->rot, sizeof(float4) * n, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemcpyAsync(dst->scale + at, src->scale, sizeof(float4) * n, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemcpyAsync(dst->virt + at, src->virt, n, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemcpyAsync(dst->colors + at * cs, src->colors, sizeof(float) * cs * n,
                     cudaMemcpyDeviceToDevice, c->stream));
}

struct ProbeSet {
  std::vector<float4> pos_op, rot, scale;
  std::vector<uint8_t> virt;
};

// Writes probes [first, first + n) of `p` after the particles already in dst.
static void upload_probes(gavis_ctx* c, gavis_scene* dst, int64_t at, const ProbeSet& p,
                          const std::vector<int64_t>& pick) {
  const int64_t n = (int64_t)pick.size();
  if (n == 0) return;
  std::vector<float4> a(n), b(n), d(n);
  std::vector<uint8_t> v(n, 1);
  for (int64_t i = 0; i < n; ++i) {
    a[i] = p.pos_op[pick[i]];
    b[i] = p.rot[pick[i]];
    d[i] = p.scale[pick[i]];
  }
  const int cs = dst->dev.cstride;
  CK(cudaMemcpyAsync(dst->pos_op + at, a.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(dst->rot + at, b.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(dst->scale + at, d.data(), sizeof(float4) * n, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(dst->virt + at, v.data(), n, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(dst->colors + at * cs, 0, sizeof(float) * cs * n, c->stream));
  CK(cudaStreamSynchronize(c->stream));  // host staging vectors go out of scope
}

static uint64_t mix64_host(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// density_control (vfield.hpp:149-199): probes uniform in the bounds
// (SplitMix64(derive_seed(seed, k)), rng.hpp:26-45), isotropic multi-view
// visibility 1 - prod(1 - b_p) over the trajectory on the device, probes with
// visibility <= eps_v appended (flagged virtual, opacity 0, identity rotation).
gavis_status gavis_density_control(gavis_ctx* c, const gavis_scene* scene, const double* bmin,
                                   const double* bmax, const gavis_camera* views, int32_t n_views,
                                   const gavis_density_config* cfg, const gavis_raster_config* rc,
                                   gavis_scene** out, int64_t* n_kept, int64_t* kept_ids,
                                   int64_t kept_capacity) {
  return guard([&] {
    require(c && scene && bmin && bmax && cfg && out, "null argument");
    require(cfg->rho > 0.0, "density rho must be positive");
    require(cfg->eta > -1.0, "density eta must exceed -1");
    require(cfg->eps_v > 0.0 && cfg->eps_v <= 1.0, "density eps_v must lie in (0, 1]");
    validate_raster(rc);
    require(n_views >= 0 && (views || n_views == 0), "views must not be null");
    for (int i = 0; i < n_views; ++i) validate_camera(views[i]);
    const double ext[3] = {bmax[0] - bmin[0], bmax[1] - bmin[1], bmax[2] - bmin[2]};
    const double volume = ext[0] * ext[1] * ext[2];
    require(volume > 0.0, "density_control: scene bounds volume must be positive");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    const int64_t n_virtual = (int64_t)std::floor(cfg->rho * volume);
    const int64_t n_real = scene->dev.n;
    require(n_real + n_virtual < (int64_t(1) << 31), "density_control: too many probes");
    const double sc = std::cbrt(3.0 * (1.0 + cfg->eta) / (4.0 * kPi * cfg->rho));
    ProbeSet p;
    p.pos_op.resize(n_virtual);
    p.rot.resize(n_virtual, make_float4(1.f, 0.f, 0.f, 0.f));
    p.scale.resize(n_virtual, make_float4((float)sc, (float)sc, (float)sc, 0.f));
    for (int64_t k = 0; k < n_virtual; ++k) {
      uint64_t st = mix64_host(cfg->seed ^ mix64_host((uint64_t)k + 0x632be59bd9b4e019ull));
      double u[3];
      for (int d = 0; d < 3; ++d) {
        st += 0x9e3779b97f4a7c15ull;
        uint64_t z = st;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z = z ^ (z >> 31);
        u[d] = (double)(z >> 11) * 0x1.0p-53;
      }
      p.pos_op[k] = make_float4((float)(bmin[0] + ext[0] * u[0]), (float)(bmin[1] + ext[1] * u[1]),
                                (float)(bmin[2] + ext[2] * u[2]), 0.f);
    }
    std::vector<int64_t> all(n_virtual);
    for (int64_t k = 0; k < n_virtual; ++k) all[k] = k;
    gavis_scene* probe = alloc_scene(c, n_real + n_virtual, scene->dev.color_degree);
    probe->max_opacity = scene->max_opacity;
    std::vector<double> unseen((size_t)std::max<int64_t>(1, n_virtual), 1.0);
    try {
      copy_particles(c, probe, 0, scene, n_real);
      upload_probes(c, probe, n_real, p, all);
      if (n_virtual > 0 && n_views > 0) {
        double* du = (double*)c->buf("unseen", sizeof(double) * n_virtual);
        CK(cudaMemcpyAsync(du, unseen.data(), sizeof(double) * n_virtual, cudaMemcpyHostToDevice,
                           c->stream));
        DensityHook dh;
        dh.unseen = du;
        dh.n_real = n_real;
        dh.n_virtual = n_virtual;
        vf_views(c, probe, nullptr, views, n_views, rc, nullptr, nullptr, nullptr, &dh);
        CK(cudaMemcpyAsync(unseen.data(), du, sizeof(double) * n_virtual, cudaMemcpyDeviceToHost,
                           c->stream));
        c->sync();
      }
    } catch (...) {
      gavis_scene_destroy(probe);
      throw;
    }
    gavis_scene_destroy(probe);
    std::vector<int64_t> keep;
    for (int64_t k = 0; k < n_virtual; ++k) {
      const double vtilde = 1.0 - unseen[k];
      if (vtilde > cfg->eps_v) continue;  // free space
      keep.push_back(k);
    }
    gavis_scene* o = alloc_scene(c, n_real + (int64_t)keep.size(), scene->dev.color_degree);
    o->max_opacity = scene->max_opacity;
    try {
      copy_particles(c, o, 0, scene, n_real);
      upload_probes(c, o, n_real, p, keep);
      c->sync();
    } catch (...) {
      gavis_scene_destroy(o);
      throw;
    }
    if (n_kept) *n_kept = (int64_t)keep.size();
    if (kept_ids)
      for (int64_t i = 0; i < (int64_t)keep.size() && i < kept_capacity; ++i) kept_ids[i] = keep[i];
    *out = o;
  });
}

gavis_status gavis_scene_upload(gavis_ctx* c, const gavis_scene_desc* d, gavis_scene** out) {
  return guard([&] {
    require(c != nullptr && d != nullptr && out != nullptr, "null argument");
    require(d->num_particles >= 0, "num_particles must be non-negative");
    require(d->num_particles < (int64_t(1) << 31), "num_particles exceeds 2^31 - 1");
    require(d->color_degree >= 0 && d->color_degree <= kMaxColorDegree,
            "color_degree must lie in [0, 3] for the device path");
    const int64_t N = d->num_particles;
    if (N > 0)
      require(d->positions && d->rotations && d->scales && d->opacities && d->colors,
              "scene arrays must not be null");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    gavis_scene* s = alloc_scene(c, N, d->color_degree);
    for (int64_t i = 0; i < N; ++i) s->max_opacity = std::max(s->max_opacity, d->opacities[i]);
    const int nb = s->dev.nb;
    const int nbp = nb + (nb & 1);
    const int cstride = s->dev.cstride;
    try {
      if (N > 0) {
        // raw host arrays -> staging buffer (DMA; pinned host memory runs at
        // full PCIe/C2C rate), then one packing kernel builds the device layout
        const bool direct_colors = cstride == 3 * nb && nbp == nb;
        const size_t b_pos = sizeof(float) * 3 * N, b_op = sizeof(float) * N;
        const size_t b_col = direct_colors ? 0 : sizeof(float) * 3 * nb * N;
        const size_t b_virt = d->is_virtual ? (size_t)N : 0;
        char* st = (char*)c->buf("upload_stage", 2 * b_pos + b_op + b_col + b_virt + 64);
        float* st_pos = (float*)st;
        float* st_scale = (float*)(st + b_pos);
        float* st_op = (float*)(st + 2 * b_pos);
        float* st_col = (float*)(st + 2 * b_pos + b_op);
        uint8_t* st_virt = (uint8_t*)(st + 2 * b_pos + b_op + b_col);
        CK(cudaMemcpyAsync(st_pos, d->positions, b_pos, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(st_scale, d->scales, b_pos, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(st_op, d->opacities, b_op, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(s->rot, d->rotations, sizeof(float4) * N, cudaMemcpyHostToDevice,
                           c->stream));
        if (direct_colors)
          CK(cudaMemcpyAsync(s->colors, d->colors, sizeof(float) * cstride * N,
                             cudaMemcpyHostToDevice, c->stream));
        else
          CK(cudaMemcpyAsync(st_col, d->colors, b_col, cudaMemcpyHostToDevice, c->stream));
        if (b_virt) CK(cudaMemcpyAsync(st_virt, d->is_virtual, b_virt, cudaMemcpyHostToDevice, c->stream));
        PackSceneArgs pk;
        pk.n = N;
        pk.nb = nb;
        pk.nbp = nbp;
        pk.cstride = cstride;
        pk.pos = st_pos;
        pk.op = st_op;
        pk.scale = st_scale;
        pk.colors = direct_colors ? nullptr : st_col;
        pk.virt = b_virt ? st_virt : nullptr;
        pk.pos_op = s->pos_op;
        pk.scale4 = s->scale;
        pk.colors_out = s->colors;
        pk.virt_out = s->virt;
        c->run("pack_scene", [&] { launch_pack_scene(pk, c->stream); });
      }
      c->sync();  // the caller may release its host arrays on return
    } catch (...) {
      gavis_scene_destroy(s);
      throw;
    }
    *out = s;
  });
}

gavis_status gavis_scene_destroy(gavis_scene* s) {
  return guard([&] {
    if (!s) return;
    gavis_ctx* c = s->ctx;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    c->dfree(s->pos_op);
    c->dfree(s->rot);
    c->dfree(s->scale);
    c->dfree(s->virt);
    c->dfree(s->colors);
    c->dfree(s->colors_split);
    c->dfree(s->var);
    delete s;
  });
}

gavis_status gavis_scene_set_coeff_variances(gavis_ctx* c, gavis_scene* s, const float* var,
                                             int32_t degree) {
  return guard([&] {
    require(c && s, "null argument");
    require(degree >= 0 && degree <= kMaxFieldDegree,
            "sh_variance_propagation: variance degree must lie in [0, 4] on the device");
    const int64_t N = s->dev.n;
    const int nbv = (degree + 1) * (degree + 1);
    require(var != nullptr || N == 0, "coeff_variances must not be null");
    for (int64_t i = 0; i < N * 3 * nbv; ++i)
      require(var[i] >= 0.0f, "sh_variance_propagation: negative variance entry");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    c->dfree(s->var);
    s->var = nullptr;
    s->var = nullptr;
    s->var = (float*)c->dalloc(sizeof(float) * 3 * nbv * std::max<int64_t>(1, N), "coeff_variances");
    if (N > 0)
      CK(cudaMemcpy(s->var, var, sizeof(float) * 3 * nbv * N, cudaMemcpyHostToDevice));
    s->var_degree = degree;
  });
}

gavis_status gavis_scene_num_particles(const gavis_scene* s, int64_t* n) {
  return guard([&] {
    require(s != nullptr && n != nullptr, "null argument");
    *n = s->dev.n;
  });
}

static gavis_field* new_field(gavis_ctx* c, const gavis_scene* s, double kappa, int degree) {
  require(degree >= 0 && degree <= 20, "construct_field: degree out of range");
  require(degree <= kMaxFieldDegree, "field degree above 4 is not supported by the device path");
  require(kappa >= 0.0 && kappa <= 50.0, "vmf kappa must lie in [0, 50]");
  auto* f = new gavis_field();
  f->ctx = c;
  f->scene = s;
  f->n = s->dev.n;
  f->degree = degree;
  f->kappa = kappa;
  const int nb = (degree + 1) * (degree + 1);
  const size_t bytes = sizeof(double) * nb * std::max<int64_t>(1, f->n);
  try {
    f->gamma = (double*)c->dalloc(bytes, "field");
  } catch (...) {
    delete f;
    throw;
  }
  CK(cudaMemsetAsync(f->gamma, 0, bytes, c->stream));
  return f;
}

gavis_status gavis_vf_create(gavis_ctx* c, const gavis_scene* s, double kappa, int32_t degree,
                             gavis_field** out) {
  return guard([&] {
    require(c && s && out, "null argument");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    *out = new_field(c, s, kappa, degree);
    c->sync();
  });
}

gavis_status gavis_vf_construct(gavis_ctx* c, const gavis_scene* s, const gavis_camera* views,
                                int32_t n_views, double kappa, int32_t degree,
                                const gavis_raster_config* rc, gavis_field** out) {
  return guard([&] {
    require(c && s && out, "null argument");
    require(n_views > 0 && views != nullptr, "construct_field: trajectory must be nonempty");
    require(degree >= 0 && degree <= 20, "construct_field: degree out of range");
    validate_raster(rc);
    for (int i = 0; i < n_views; ++i) validate_camera(views[i]);
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    gavis_field* f = new_field(c, s, kappa, degree);
    try {
      vf_views(c, s, f, views, n_views, rc, nullptr, nullptr, nullptr);
    } catch (...) {
      c->dfree(f->gamma);
      delete f;
      throw;
    }
    f->num_views = n_views;
    *out = f;
  });
}

gavis_status gavis_vf_accumulate_views(gavis_ctx* c, gavis_field* f, const gavis_scene* s,
                                       const gavis_camera* views, int32_t n_views,
                                       const gavis_raster_config* rc) {
  return guard([&] {
    require(c && f && s, "null argument");
    invariant(f->n == s->dev.n, "accumulate_view: field/scene particle count mismatch");
    require(n_views >= 0 && (views != nullptr || n_views == 0), "views must not be null");
    validate_raster(rc);
    for (int i = 0; i < n_views; ++i) validate_camera(views[i]);
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    vf_views(c, s, f, views, n_views, rc, nullptr, nullptr, nullptr);
  });
}

gavis_status gavis_vf_accumulate_visibility(gavis_ctx* c, gavis_field* f, const gavis_scene* s,
                                            const gavis_camera* view, const double* vis) {
  return guard([&] {
    require(c && f && s && view, "null argument");
    invariant(f->n == s->dev.n, "accumulate_view: field/scene particle count mismatch");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    const int64_t N = s->dev.n;
    if (N > 0) {
      require(vis != nullptr, "visibility must not be null");
      DevCam d = make_devcam(*view, 16, 0, 0);
      DevCam* dc = (DevCam*)c->buf("cams", sizeof(DevCam));
      CK(cudaMemcpyAsync(dc, &d, sizeof(DevCam), cudaMemcpyHostToDevice, c->stream));
      double* dv = (double*)c->buf("vis_given", sizeof(double) * N);
      CK(cudaMemcpyAsync(dv, vis, sizeof(double) * N, cudaMemcpyHostToDevice, c->stream));
      VfFinalizeArgs fa;
      fa.scene = s->dev;
      fa.cams = dc;
      fa.V = 1;
      fa.vis_given = dv;
      fa.gamma = f->gamma;
      fa.degree = f->degree;
      vmf_scales(f->kappa, f->degree, fa.scales);
      c->run("vf_finalize", [&] { launch_vf_finalize(fa, N, c->stream); });
      c->sync();
    }
    f->num_views += 1;
  });
}

gavis_status gavis_vf_upload(gavis_ctx* c, const gavis_scene* s, double kappa, int32_t degree,
                             int32_t num_views, const double* gamma, gavis_field** out) {
  return guard([&] {
    require(c && s && out, "null argument");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    gavis_field* f = new_field(c, s, kappa, degree);
    const int nb = (degree + 1) * (degree + 1);
    if (f->n > 0) {
      require(gamma != nullptr, "gamma must not be null");
      CK(cudaMemcpyAsync(f->gamma, gamma, sizeof(double) * nb * f->n, cudaMemcpyHostToDevice,
                         c->stream));
    }
    f->num_views = num_views;
    c->sync();
    *out = f;
  });
}

gavis_status gavis_vf_download(const gavis_field* f, double* gamma, int32_t* num_views,
                               int32_t* degree) {
  return guard([&] {
    require(f != nullptr, "field must not be null");
    gavis_ctx* c = f->ctx;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    const int nb = (f->degree + 1) * (f->degree + 1);
    if (gamma && f->n > 0)
      CK(cudaMemcpyAsync(gamma, f->gamma, sizeof(double) * nb * f->n, cudaMemcpyDeviceToHost,
                         c->stream));
    c->sync();
    if (num_views) *num_views = f->num_views;
    if (degree) *degree = f->degree;
  });
}

gavis_status gavis_vf_set_num_views(gavis_field* f, int32_t num_views) {
  return guard([&] {
    require(f != nullptr, "field must not be null");
    f->num_views = num_views;
  });
}

gavis_status gavis_vf_device_gamma(gavis_field* f, void** ptr, int64_t* count) {
  return guard([&] {
    require(f != nullptr, "field must not be null");
    if (ptr) *ptr = f->gamma;
    if (count) *count = f->n * (int64_t)((f->degree + 1) * (f->degree + 1));
  });
}

gavis_status gavis_vf_destroy(gavis_field* f) {
  return guard([&] {
    if (!f) return;
    gavis_ctx* c = f->ctx;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    c->dfree(f->gamma);
    delete f;
  });
}

gavis_status gavis_single_view_visibility(gavis_ctx* c, const gavis_scene* s,
                                          const gavis_camera* cam, const gavis_raster_config* rc,
                                          double* vis, int64_t* touch, int32_t* contrib) {
  return guard([&] {
    require(c && s && cam, "null argument");
    validate_raster(rc);
    validate_camera(*cam);
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    vf_views(c, s, nullptr, cam, 1, rc, vis, touch, contrib);
  });
}

gavis_status gavis_vf_query(gavis_ctx* c, const gavis_field* f, const int64_t* idx,
                            const double* dirs, int64_t n, double* out) {
  return guard([&] {
    require(c && f, "null argument");
    require(n >= 0 && (n == 0 || (idx && dirs && out)), "null argument");
    for (int64_t i = 0; i < n; ++i)
      require(idx[i] >= 0 && idx[i] < f->n, "query: particle index out of range");
    if (n == 0) return;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    int64_t* di = (int64_t*)c->buf("q_idx", sizeof(int64_t) * n);
    double* dd = (double*)c->buf("q_dir", sizeof(double) * 3 * n);
    double* dout = (double*)c->buf("q_out", sizeof(double) * n);
    CK(cudaMemcpyAsync(di, idx, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dd, dirs, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
    QueryArgs qa;
    qa.gamma = f->gamma;
    qa.virt = f->scene->dev.virt;
    qa.degree = f->degree;
    qa.num_views = f->num_views;
    qa.idx = di;
    qa.dirs = dd;
    qa.n = n;
    qa.out = dout;
    c->run("query", [&] { launch_query(qa, c->stream); });
    CK(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
  });
}

gavis_status gavis_vf_query_view(gavis_ctx* c, const gavis_field* f, const gavis_scene* s,
                                 const gavis_camera* cam, double dilation, int32_t* idx,
                                 double* vis, int64_t* n_out) {
  return guard([&] {
    require(c && f && s && cam && n_out, "null argument");
    require(f->n == s->dev.n, "query_view: field/scene particle count mismatch");
    validate_camera(*cam);
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    const int64_t N = s->dev.n;
    *n_out = 0;
    if (N == 0) return;
    gavis_raster_config rc = {16, 0, 1e-4, dilation, 0.99};
    BinOpts o;
    o.ua = true;
    o.field = f;
    o.write_culled = true;
    Binned b = bin_batch(c, s, cam, 1, &rc, o);
    std::vector<uint32_t> flags((size_t)N);
    std::vector<double> v((size_t)N);
    CK(cudaMemcpy2DAsync(flags.data(), sizeof(uint32_t), &b.geo[0].flags, sizeof(GeoRec),
                         sizeof(uint32_t), N, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpy2DAsync(v.data(), sizeof(double), &b.ua[0].v, sizeof(UaRec), sizeof(double), N,
                         cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    int64_t k = 0;
    for (int64_t i = 0; i < N; ++i) {
      if (!(flags[i] & 1u)) continue;
      if (idx) idx[k] = (int32_t)i;
      if (vis) vis[k] = v[i];
      ++k;
    }
    *n_out = k;
  });
}

gavis_status gavis_ua_render(gavis_ctx* c, const gavis_scene* s, const gavis_field* f,
                             const double* splat_visibility, const gavis_camera* cams,
                             int32_t n_cams, const gavis_raster_config* rc,
                             const gavis_uncertainty_config* uc, gavis_render_outputs* out) {
  return guard([&] {
    require(c && s, "null argument");
    require(n_cams >= 0, "camera count must be non-negative");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    ua_render(c, s, f, splat_visibility, cams, n_cams, rc, uc, out);
  });
}

gavis_status gavis_ua_mixtures(gavis_ctx* c, const gavis_scene* s, const gavis_field* f,
                               const double* splat_visibility, const gavis_camera* cam,
                               const gavis_raster_config* rc, const gavis_uncertainty_config* uc,
                               int64_t* offsets, gavis_mixture_component* components,
                               int64_t capacity, double* prior_weight,
                               double* residual_transmittance, double* entropy) {
  return guard([&] {
    require(c && s && cam && rc && uc && offsets, "null argument");
    validate_raster(rc);
    double hl_q0 = 0.0;
    validate_unc(uc, &hl_q0);
    validate_camera(*cam);
    check_scene_field(s, f);
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    const int64_t N = s->dev.n;
    const int64_t P = (int64_t)cam->width * cam->height;
    BinOpts o;
    o.ua = true;
    o.field = f;
    if (!f) {
      require(splat_visibility != nullptr || N == 0,
              "mixtures need a field or per-particle splat visibility");
      if (N > 0) {
        double* d = (double*)c->buf("vis_given", sizeof(double) * N);
        CK(cudaMemcpyAsync(d, splat_visibility, sizeof(double) * N, cudaMemcpyHostToDevice,
                           c->stream));
        o.vis_given_dev = d;
      }
    }
    o.beta = uc->beta;
    o.o0b = uc->prior_opacity * (1.0 - uc->beta);
    o.hl_const = 3.0 * std::log(uc->color_sigma);
    int* err = nullptr;
    if (uc->variance_provider == 1) {
      require(s->var != nullptr || N == 0,
              "variance_provider sh_propagation requires coeff_variances");
      o.var = s->var;
      o.var_degree = s->var_degree;
      err = (int*)c->buf("err_flag", sizeof(int));
      CK(cudaMemsetAsync(err, 0, sizeof(int), c->stream));
      o.err_flag = err;
    }
    Binned b = bin_batch(c, s, cam, 1, rc, o);
    if (err) {
      CK(cudaMemcpyAsync(c->pinned + 2, err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      c->sync();
      require(c->pinned[2] == 0, "propagated color variance must be positive");
    }
    MixtureArgs m;
    m.scene = s->dev;
    m.cam = b.dcams;
    m.tile_size = rc->tile_size;
    m.cutoff = rc->transmittance_cutoff;
    m.amax = rc->alpha_clamp_max;
    m.hl_q0 = hl_q0;
    m.var_const = uc->color_sigma * uc->color_sigma;
    m.geo = b.geo;
    m.ua = b.ua;
    m.ranges = b.ranges;
    m.vals = b.vals;
    m.var = o.var;
    m.var_degree = o.var_degree;
    m.counts = (int64_t*)c->buf("mix_counts", sizeof(int64_t) * std::max<int64_t>(1, P));
    m.prior = (double*)c->buf("mix_prior", sizeof(double) * std::max<int64_t>(1, P));
    m.resid = (double*)c->buf("mix_resid", sizeof(double) * std::max<int64_t>(1, P));
    m.entropy = (double*)c->buf("mix_entropy", sizeof(double) * std::max<int64_t>(1, P));
    c->run("mixtures", [&] { launch_mixtures(m, P, c->stream); });
    std::vector<int64_t> cnt((size_t)P);
    if (P > 0)
      CK(cudaMemcpyAsync(cnt.data(), m.counts, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, c->stream));
    copy_out(c, prior_weight, m.prior, P);
    copy_out(c, residual_transmittance, m.resid, P);
    copy_out(c, entropy, m.entropy, P);
    c->sync();
    offsets[0] = 0;
    for (int64_t p = 0; p < P; ++p) offsets[p + 1] = offsets[p] + cnt[p];
    const int64_t K = offsets[P];
    if (components && K > 0) {
      require(capacity >= K, "mixtures: capacity is smaller than offsets[W*H]");
      int64_t* doff = (int64_t*)c->buf("mix_offsets", sizeof(int64_t) * (P + 1));
      CK(cudaMemcpyAsync(doff, offsets, sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, c->stream));
      m.offsets = doff;
      m.comps = (double*)c->buf("mix_comps", sizeof(double) * 8 * K);
      c->run("mixtures", [&] { launch_mixtures(m, P, c->stream); });
      static_assert(sizeof(gavis_mixture_component) == 8 * sizeof(double), "component layout");
      CK(cudaMemcpyAsync(components, m.comps, sizeof(double) * 8 * K, cudaMemcpyDeviceToHost,
                         c->stream));
      c->sync();
    }
  });
}

gavis_status gavis_select_nbv(gavis_ctx* c, const gavis_scene* s, const gavis_field* f,
                              const gavis_camera* cams, int32_t n_cams,
                              const gavis_raster_config* rc, const gavis_uncertainty_config* uc,
                              int32_t with_rgb, double* scores, int32_t* best) {
  return guard([&] {
    require(c && s && f, "null argument");
    require(n_cams > 0 && cams != nullptr, "select_nbv: candidate list must be nonempty");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    std::vector<double> sc((size_t)n_cams);
    gavis_render_outputs o = {};
    o.scores = sc.data();
    o.with_rgb = with_rgb;
    ua_render(c, s, f, nullptr, cams, n_cams, rc, uc, &o);
    const int b = certified_first_max(c, s, f, cams, n_cams, rc, uc, sc);
    if (scores) std::memcpy(scores, sc.data(), sizeof(double) * n_cams);
    if (best) *best = b;
  });
}

gavis_status gavis_debug_project(gavis_ctx* c, const gavis_scene* s, const gavis_camera* cam,
                                 double dilation, int32_t tile_size, uint8_t* culled,
                                 double* mean, double* conic, double* depth, int32_t* cover_rect,
                                 int32_t* tile_rect) {
  return guard([&] {
    require(c && s && cam, "null argument");
    validate_camera(*cam);
    require(tile_size >= 1, "tile_size must be at least 1");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    const int64_t N = s->dev.n;
    if (N == 0) return;
    gavis_raster_config rc = {tile_size, 0, 1e-4, dilation, 0.99};
    BinOpts o;
    o.write_culled = true;
    Binned b = bin_batch(c, s, cam, 1, &rc, o);
    std::vector<GeoRec> g((size_t)N);
    std::vector<uint2> tr((size_t)N);
    CK(cudaMemcpyAsync(g.data(), b.geo, sizeof(GeoRec) * N, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(tr.data(), c->bufs["trect"].p, sizeof(uint2) * N, cudaMemcpyDeviceToHost,
                       c->stream));
    c->sync();
    for (int64_t i = 0; i < N; ++i) {
      const bool ok = g[i].flags & 1u;
      if (culled) culled[i] = ok ? 0 : 1;
      if (mean) {
        mean[2 * i] = g[i].mx;
        mean[2 * i + 1] = g[i].my;
      }
      if (conic) {
        conic[3 * i] = g[i].ca;
        conic[3 * i + 1] = g[i].cb2 * 0.5;
        conic[3 * i + 2] = g[i].cc;
      }
      if (depth) depth[i] = g[i].depth;
      if (cover_rect) {
        cover_rect[4 * i] = g[i].cov_x & 0xFFFF;
        cover_rect[4 * i + 1] = (g[i].cov_x >> 16) & 0xFFFF;
        cover_rect[4 * i + 2] = g[i].cov_y & 0xFFFF;
        cover_rect[4 * i + 3] = (g[i].cov_y >> 16) & 0xFFFF;
      }
      if (tile_rect) {
        tile_rect[4 * i] = tr[i].x & 0xFFFF;
        tile_rect[4 * i + 1] = tr[i].x >> 16;
        tile_rect[4 * i + 2] = tr[i].y & 0xFFFF;
        tile_rect[4 * i + 3] = tr[i].y >> 16;
      }
    }
  });
}

gavis_status gavis_debug_binning(gavis_ctx* c, const gavis_scene* s, const gavis_camera* cam,
                                 const gavis_raster_config* rc, uint64_t* keys,
                                 int32_t* particle_ids, int64_t* ranges, int64_t* n_pairs) {
  return guard([&] {
    require(c && s && cam && n_pairs, "null argument");
    validate_raster(rc);
    validate_camera(*cam);
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    BinOpts o;
    Binned b = bin_batch(c, s, cam, 1, rc, o);
    *n_pairs = b.K;
    if (keys && b.K > 0) {
      const uint64_t* dk = b.keys;
      if (b.narrow) {  // reference-form (tile << 32 | fp32 depth) keys of the sorted pairs
        uint64_t* wk = (uint64_t*)c->buf("keys_a", sizeof(uint64_t) * b.K);
        c->run("wide_keys", [&] {
          launch_wide_keys(b.ranges, b.total_tiles, b.vals, b.pair_gid, b.dcams, b.V, s->dev.n, b.geo,
                           wk, c->stream);
        });
        dk = wk;
      }
      CK(cudaMemcpyAsync(keys, dk, sizeof(uint64_t) * b.K, cudaMemcpyDeviceToHost, c->stream));
    }
    if (particle_ids && b.K > 0)
      CK(cudaMemcpyAsync(particle_ids, b.vals, sizeof(uint32_t) * b.K, cudaMemcpyDeviceToHost,
                         c->stream));
    std::vector<uint2> rg((size_t)std::max<int64_t>(1, b.total_tiles));
    if (ranges && b.total_tiles > 0)
      CK(cudaMemcpyAsync(rg.data(), b.ranges, sizeof(uint2) * b.total_tiles,
                         cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (ranges)
      for (int64_t t = 0; t < b.total_tiles; ++t) {
        ranges[2 * t] = rg[t].x;
        ranges[2 * t + 1] = rg[t].y;
      }
  });
}

}  // extern "C"
