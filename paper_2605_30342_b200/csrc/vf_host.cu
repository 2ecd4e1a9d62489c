// vf_host.cu -- VF CONST (construct_field / accumulate_view, vfield.hpp:38-92)
// and VF-QUERY (query_visibility / query_view, vfield.hpp:96-134) behind the C ABI.
#include "host.h"

namespace gavis {
namespace host {

void vf_views(gavis_ctx* c, const gavis_scene* s, gavis_field* f, const gavis_camera* views,
              int n_views, const gavis_raster_config* rc, double* vis_host, int64_t* touch_host,
              int32_t* contrib_host, const DensityHook* dh) {
  NvtxRange nvtx("VF CONST (single_view_visibility + accumulate_view)");
  require(s->ctx->device == c->device, "scene was uploaded to another device");
  if (f) require(f->ctx->device == c->device, "field lives on another device");
  const int64_t N = s->dev.n;
  const int bv = batch_views(c, N, n_views);
  double scales[kMaxFieldDegreeRT + 1] = {0};
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
  int bvv = bv;  // views per batch; halved for good when a batch holds too many pairs
  for (int v0 = 0, V = 0; v0 < n_views; v0 += V, ++batch) {
    V = std::min(bvv, n_views - v0);
    const int par = batch & 1;
    c->bufset = par;
    c->stream = c->front;
    if (batch >= 2) CK(cudaStreamWaitEvent(c->front, c->ev_done[par], 0));
    BinOpts o;
    o.vf_mode = true;
    Binned b = bin_batch(c, s, views + v0, V, rc, o);
    while (b.overflow) {
      V = bvv = std::max(1, V / 2);
      b = bin_batch(c, s, views + v0, V, rc, o);
    }
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
    va.fixed_sums = s->opacity_nonneg;
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

}  // namespace host
}  // namespace gavis

extern "C" {

static gavis_field* new_field(gavis_ctx* c, const gavis_scene* s, double kappa, int degree) {
  require(degree >= 0 && degree <= 20, "construct_field: degree out of range");
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
    require(s->dev.n == 0 || gamma != nullptr, "gamma must not be null");
    require(num_views >= 0, "field: num_views must be non-negative");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    gavis_field* f = new_field(c, s, kappa, degree);  // validates degree and kappa
    try {
      const int nb = (degree + 1) * (degree + 1);
      if (f->n > 0)
        CK(cudaMemcpyAsync(f->gamma, gamma, sizeof(double) * nb * f->n, cudaMemcpyHostToDevice,
                           c->stream));
      f->num_views = num_views;
      c->sync();
    } catch (...) {
      c->dfree(f->gamma);
      delete f;
      throw;
    }
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
    std::vector<double> depth((size_t)N);
    std::vector<double> v((size_t)N);
    CK(cudaMemcpy2DAsync(depth.data(), sizeof(double), &b.geo[0].depth, sizeof(GeoRec),
                         sizeof(double), N, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpy2DAsync(v.data(), sizeof(double), &b.ua[0].v, sizeof(UaRec), sizeof(double), N,
                         cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    int64_t k = 0;
    for (int64_t i = 0; i < N; ++i) {
      if (std::isnan(depth[i])) continue;  // culled (K1 marks it with a NaN depth)
      if (idx) idx[k] = (int32_t)i;
      if (vis) vis[k] = v[i];
      ++k;
    }
    *n_out = k;
  });
}

}  // extern "C"
