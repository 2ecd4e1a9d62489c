// gavis_abi.cu -- the C ABI (include/gavis_b200.h): context lifecycle, scene
// upload, density control and the planner loop. Per batch of views the host
// orchestrates K1 preprocess -> K2 scan -> K3 emit keys -> K4 radix sort -> K5
// ranges (binning.cu), then VF: K6a vf_blend -> K6b vf_finalize (vf_host.cu) or
// UA: K7 ua_blend -> K8 score (ua_host.cu).
#include "host.h"

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
      int lo_prio = 0, hi_prio = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
      CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
      // certified renders' side stream (fp64 redo, scores, copy-outs of batch k):
      // above the blend's priority, so the redo of batch k is not queued behind
      // batch k+1's tiles (certified 2032 -> 2042 views/s; the fp64 path keeps
      // the default-priority side stream: 1481 vs 1472)
      CK(cudaStreamCreateWithPriority(&c->side_hi, cudaStreamNonBlocking,
                                      hi_prio < lo_prio ? hi_prio + 1 : hi_prio));
      CK(cudaStreamCreateWithPriority(&c->front, cudaStreamNonBlocking, hi_prio));
      for (int k = 0; k < gavis_ctx::kSets; ++k) {
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
    if (c->pin_bounds) cudaFreeHost(c->pin_bounds);
    for (cudaStream_t st : {c->side, c->side_hi, c->front})
      if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
      }
    for (int k = 0; k < gavis_ctx::kSets; ++k) {
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

gavis_status gavis_ctx_set_pair_budget(gavis_ctx* c, int64_t n) {
  return guard([&] {
    require(c != nullptr, "context must not be null");
    require(n >= 0, "pair budget must be non-negative");
    c->pair_budget = n;
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

gavis_status gavis_ctx_last_score_bounds(gavis_ctx* c, double* bounds, int32_t capacity,
                                         int32_t* n_out) {
  return guard([&] {
    require(c && n_out, "null argument");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    const int32_t n = (int32_t)c->score_bounds.size();
    *n_out = n;
    if (bounds && n > 0) {
      require(capacity >= n, "score bounds: capacity too small");
      std::memcpy(bounds, c->score_bounds.data(), sizeof(double) * n);
    }
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
    ScoringPrecision sp(c, uc);
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

// The staged colour records of the certified blend's tensor-core colour path
// (SceneDev::colors_split), built once when a scene is finalised.
static void build_colour_split(gavis_ctx* c, gavis_scene* s) {
  const size_t bytes = ua_colors_split_bytes(s->dev);
  if (bytes == 0 || s->dev.n == 0) return;
  s->colors_split = (uint4*)c->dalloc(bytes, "scene colour splits");
  s->dev.colors_split = s->colors_split;
  c->run("split_colors", [&] { launch_split_colors(s->dev, s->colors_split, c->stream); });
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
    probe->opacity_nonneg = scene->opacity_nonneg;
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
    o->opacity_nonneg = scene->opacity_nonneg;
    try {
      copy_particles(c, o, 0, scene, n_real);
      upload_probes(c, o, n_real, p, keep);
      build_colour_split(c, o);
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
    for (int64_t i = 0; i < N; ++i) {
      s->max_opacity = std::max(s->max_opacity, d->opacities[i]);
      if (!(d->opacities[i] >= 0.f)) s->opacity_nonneg = false;  // negative or NaN
    }
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
      build_colour_split(c, s);
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

}  // extern "C"
