// host.h -- internal to the native library: the host-side state behind the C
// ABI (context, scene, field), validation and error mapping shared by the ABI
// translation units:
//   gavis_abi.cu  context, scene upload, density control, the planner loop
//   binning.cu    K1..K5 for a batch of views (+ the debug exports)
//   vf_host.cu    VF CONST / VF-QUERY (construct_field, vfield.hpp:68-134)
//   ua_host.cu    uncertainty render, scores and select_nbv (uncertainty.hpp:242-278,
//                 planner.hpp:117-137)
// Validation follows the reference's validate() methods (raster.hpp:27-34,
// model.hpp:99-104, uncertainty.hpp:39-51, sh.hpp:126-128) and maps its
// exception taxonomy onto status codes (common.hpp:22-46).
#pragma once

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

#include <nvtx3/nvToolsExt.h>

#include "gavis_b200.h"
#include "kernels.h"

namespace gavis {
namespace host {



inline thread_local std::string g_last_error;

// NVTX ranges (header-only NVTX v3: free without an attached tool) around every
// kernel family launch, labelled with the DESIGN.md kernel ids (K1-K8), and
// around the entry points (VF CONST, UA render, select_nbv).
inline const char* nvtx_label(const char* family) {
  static const std::map<std::string, const char*> kLabels = {
      {"preprocess", "K1 preprocess (project + query)"},
      {"sort", "K2/K4 sort (items by depth / pairs by tile)"},
      {"depth_order", "K2c depth_order (tied runs)"},
      {"scan", "K2/K3 scan"},
      {"emit_keys", "K3 emit tile pairs"},
      {"wide_keys", "K3w emit 64-bit keys"},
      {"ranges", "K5 tile ranges"},
      {"vf_blend", "K6a vf_blend"},
      {"vf_finalize", "K6b vf_finalize"},
      {"ua_blend", "K7 ua_blend"},
      {"ua_redo", "K7r ua_redo (fp64)"},
      {"score", "K8 image score"},
      {"query", "query_visibility"},
      {"mixtures", "mixture dump"},
      {"density", "density update"}};
  const auto it = kLabels.find(family);
  return it == kLabels.end() ? family : it->second;
}

struct NvtxRange {
  explicit NvtxRange(const char* family) { nvtxRangePushA(nvtx_label(family)); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

struct ParamErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DevErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void require(bool cond, const std::string& msg) {
  if (!cond) throw ParamErr(msg);
}
inline void invariant(bool cond, const std::string& msg) {
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
inline double bessel_i(int l, double x) {
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

inline void vmf_scales(double kappa, int degree, double* out) {
  const double zeta = std::exp(-kappa);
  for (int l = 0; l <= degree; ++l) out[l] = 4.0 * kPi * zeta * bessel_i(l, kappa);
}

inline void validate_raster(const gavis_raster_config* rc) {
  require(rc != nullptr, "raster config must not be null");
  require(rc->tile_size >= 1, "tile_size must be at least 1");
  require(rc->transmittance_cutoff > 0.0 && rc->transmittance_cutoff < 1.0,
          "transmittance_cutoff must lie in (0, 1)");
  require(rc->dilation >= 0.0, "dilation must be non-negative");
  require(rc->alpha_clamp_max > 0.0 && rc->alpha_clamp_max <= 1.0,
          "alpha_clamp_max must lie in (0, 1]");
}

inline void validate_camera(const gavis_camera& c) {
  require(c.width >= 1 && c.height >= 1, "camera image size must be at least 1x1");
  require(c.fov_h > 0.0 && c.fov_h < kPi && c.fov_v > 0.0 && c.fov_v < kPi,
          "camera fov must lie in (0, pi)");
  require(c.near_plane > 0.0, "camera near plane must be positive");
  require(c.width <= 32767 && c.height <= 32767,
          "camera image size exceeds the device limit of 32767 pixels per side");
}

// LLT success and log-determinant of a 3x3 (uncertainty.hpp:44-45, :108-113).
inline bool llt3(const double* m, double* logdet) {
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

inline double det3(const double* m) {
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[3] * (m[1] * m[8] - m[2] * m[7]) +
         m[6] * (m[1] * m[5] - m[2] * m[4]);
}

inline void validate_unc(const gavis_uncertainty_config* uc, double* hl_q0) {
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

inline int bits_for(int64_t n) {  // bits needed to hold values in [0, n)
  int b = 0;
  while (b < 62 && (int64_t(1) << b) < n) ++b;
  return b;
}


}  // namespace host
}  // namespace gavis

using namespace gavis;
using namespace gavis::host;

struct gavis_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // UA renders run two batches in flight: batch k's redo / score / copy-outs on
  // `side` overlap batch k+1's binning on `stream`; per-batch buffers alternate
  // between two sets (bufset), events order the reuse.
  cudaStream_t side = nullptr;
  cudaStream_t side_hi = nullptr;  // the side stream of certified renders (priority above the blend)
  cudaStream_t front = nullptr;  // binning of batch k+1 under batch k's blend (high priority)
  int bufset = 0;
  static constexpr int kSets = 3;  // per-batch buffer sets (UA renders rotate over all three)
  cudaEvent_t ev_blend[kSets] = {}, ev_done[kSets] = {}, ev_bin[kSets] = {};
  std::map<std::string, DevBuf> bufs;
  int max_batch = 0;
  int64_t pair_budget = 0;       // tile pairs per batch (0: batch_budget / 32 B)
  bool profiling = false;
  std::map<std::string, Timing> timing;
  std::vector<std::tuple<std::string, cudaEvent_t, cudaEvent_t>> pending;
  std::vector<cudaEvent_t> spare_events;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  int64_t launches = 0;
  int32_t* pinned = nullptr;
  double* pin_scores = nullptr;  // pinned staging of per-view scores (async D2H on `side`)
  double* pin_bounds = nullptr;  // pinned staging of per-view certified score-error bounds
  int64_t pin_scores_cap = 0;
  // certified score-error bounds of the last ua_render that produced scores
  // (empty when not certified / not bounded); read by certified_contenders
  std::vector<double> score_bounds;
  int precision = GAVIS_PRECISION_EXACT;  // the reference's fp64 arithmetic by default
  int64_t redo_pixels = 0;       // pixels the certified blend handed to the fp64 redo
  double batch_budget = 0.0;     // bytes of per-(view, particle) state one batch may use
  int64_t rescored_views = 0;    // candidates re-scored exactly to certify an argmax
  std::recursive_mutex mu;

  void use() { CK(cudaSetDevice(device)); }

  void* buf(const std::string& name, size_t bytes) {
    DevBuf& b = bufs[bufset ? name + "#" + std::to_string(bufset) : name];
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
    NvtxRange nvtx(name);
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
    if (side_hi) CK(cudaStreamSynchronize(side_hi));
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
  uint4* colors_split = nullptr;  // tensor-core colour form, built when the scene is finalised
  float* var = nullptr;  // coefficient variances for the sh_propagation provider
  int var_degree = -1;
  float max_opacity = 1.f;  // enters the certified blend's error bound (q <= 2 ln(o / alpha))
  bool opacity_nonneg = true;  // every opacity >= 0: T stays in [0, 1] (the VF fixed-point sums)
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


namespace gavis {
namespace host {


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
  bool overflow = false;  // more pairs than one batch may hold: nothing emitted, re-bin fewer views
};

// pinned host scratch layout (int32 words)
constexpr int kPinItems = 4;
constexpr int kPinRedo = 6;     // u64
constexpr int kPinPairs = 8;    // u64: total tile pairs of the batch being binned
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

DevCam make_devcam(const gavis_camera& c, int ts, int64_t tile_base, int64_t pix_base);
int batch_views(gavis_ctx* c, int64_t N, int n_views);
// K1..K5 for one batch of cameras (binning.cu).
Binned bin_batch(gavis_ctx* c, const gavis_scene* s, const gavis_camera* cams, int V,
                 const gavis_raster_config* rc, const BinOpts& o);

inline void check_scene_field(const gavis_ctx* c, const gavis_scene* s, const gavis_field* f) {
  require(s != nullptr, "scene must not be null");
  require(s->ctx->device == c->device, "scene was uploaded to another device");
  if (f) require(f->n == s->dev.n, "field was built for a different scene");
  if (f) require(f->ctx->device == c->device, "field lives on another device");
}

// VF accumulation of views [0, n) into field (or only per-view outputs).
// Optional per-batch consumer of the device visibilities: density control's
// unseen[k] *= 1 - b[n_real + k], views in trajectory order (vfield.hpp:187-190).
struct DensityHook {
  double* unseen = nullptr;  // device [n_virtual]
  int64_t n_real = 0, n_virtual = 0;
};

// VF accumulation of views [0, n) into field (vf_host.cu).
void vf_views(gavis_ctx* c, const gavis_scene* s, gavis_field* f, const gavis_camera* views,
              int n_views, const gavis_raster_config* rc, double* vis_host, int64_t* touch_host,
              int32_t* contrib_host, const DensityHook* dh = nullptr);

inline void copy_out(gavis_ctx* c, double* host, const double* dev, int64_t count,
              cudaStream_t st = nullptr) {
  if (host && count > 0)
    CK(cudaMemcpyAsync(host, dev, sizeof(double) * count, cudaMemcpyDeviceToHost,
                       st ? st : c->stream));
}

// UA render of n cameras in batches (ua_host.cu).
void ua_render(gavis_ctx* c, const gavis_scene* s, const gavis_field* f, const double* vis_host,
               const gavis_camera* cams, int n, const gavis_raster_config* rc,
               const gavis_uncertainty_config* uc, gavis_render_outputs* out);
// Candidates that may be the fp64 argmax given certified scores (empty when the
// context is not in certified mode); ua_host.cu.
// The certified scores carry a rigorous bound only for the constant variance
// provider without the correlation hook; for the other two modes a scoring
// call (select_nbv, the NBV loop) runs the fp64 path instead, so the selected
// view is the fp64 one by construction in every mode. RAII: restores the
// context's precision on exit.
struct ScoringPrecision {
  gavis_ctx* c;
  int32_t saved;
  ScoringPrecision(gavis_ctx* ctx, const gavis_uncertainty_config* uc) : c(ctx), saved(ctx->precision) {
    if (uc && c->precision == GAVIS_PRECISION_CERTIFIED && (uc->correlation != 0 || uc->variance_provider != 0))
      c->precision = GAVIS_PRECISION_EXACT;
  }
  ~ScoringPrecision() { c->precision = saved; }
  ScoringPrecision(const ScoringPrecision&) = delete;
  ScoringPrecision& operator=(const ScoringPrecision&) = delete;
};

std::vector<int> certified_contenders(gavis_ctx* c, const gavis_scene* s, const gavis_raster_config* rc,
                                      const std::vector<double>& sc);
// select_nbv argmax over certified scores, contenders re-scored exactly (ua_host.cu).
int certified_first_max(gavis_ctx* c, const gavis_scene* s, const gavis_field* f,
                        const gavis_camera* cams, int n, const gavis_raster_config* rc,
                        const gavis_uncertainty_config* uc, std::vector<double>& sc);

}  // namespace host
}  // namespace gavis
