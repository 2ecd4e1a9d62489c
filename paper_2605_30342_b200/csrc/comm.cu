// comm.cu -- multi-GPU entry points, one process per GPU over NCCL.
//
// The reference parallelises both hot paths over host threads with static
// blocks (parallel_for, R/include/gavis/parallel.hpp:35-60): construct_field
// over training views (vfield.hpp:85-90), select_nbv over candidates
// (planner.hpp:125-131). Across GPUs the same decomposition holds:
//   * VF CONST: rank r renders its contiguous block of views into a partial
//     fp64 gamma; one in-place ncclAllReduce(sum) over NVLink completes it
//     (gamma is linear in the views, vfield.hpp:53-60); num_views = |P|.
//   * select_nbv: rank r scores its contiguous block of candidates; the fp64
//     scores are all-gathered once and every rank takes the same first maximum
//     (planner.hpp:132-136). In certified mode the contenders of that maximum
//     are re-scored in fp64 on the ranks that own them (one more all-reduce of a
//     candidate vector), so the argmax is the fp64 one for every rank count.
// NCCL is loaded at run time (dlopen "libnccl.so.2"): inside a process that
// already holds an NCCL (e.g. torch's), that copy is shared; a plain C++ host
// gets the system one. Communicators come from a unique id the caller
// distributes (gavis_comm_unique_id / gavis_comm_create) or are adopted from
// the caller (gavis_comm_adopt).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "host.h"

using namespace gavis::host;

namespace gavis {
namespace host {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string load_error;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.load_error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(sym("ncclAllReduce"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(sym("ncclAllGather"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
    if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_reduce || !a.all_gather)
      a.load_error = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  if (!api.load_error.empty()) throw DevErr(api.load_error);
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* msg = nccl().error_string ? nccl().error_string(r) : "?";
    throw DevErr(std::string(what) + " failed: " + msg);
  }
}

// Re-raise the status of a nested ABI call as the matching exception.
void check(gavis_status st) {
  if (st == GAVIS_OK) return;
  const std::string msg = g_last_error;
  if (st == GAVIS_ERR_PARAMETER) throw ParamErr(msg);
  if (st == GAVIS_ERR_INVARIANT) throw InvErr(msg);
  throw DevErr(msg);
}

// parallel.hpp:50-51: static block [n*r/w, n*(r+1)/w)
void block_of(int64_t n, int rank, int world, int64_t* lo, int64_t* hi) {
  *lo = n * rank / world;
  *hi = n * (rank + 1) / world;
}

}  // namespace
}  // namespace host
}  // namespace gavis

struct gavis_comm {
  gavis_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  bool owned = false;
};

namespace {

// In-place sum of gamma over the ranks on the context stream.
void allreduce_field(gavis_comm* cm, gavis_field* f) {
  gavis_ctx* c = cm->ctx;
  const int nb = (f->degree + 1) * (f->degree + 1);
  const size_t count = (size_t)nb * (size_t)f->n;
  if (count > 0)
    nck(nccl().all_reduce(f->gamma, f->gamma, count, ncclFloat64, ncclSum, cm->comm, c->stream),
        "ncclAllReduce(gamma)");
  c->sync();
}

// fp64 vector sum over the ranks through a device staging buffer.
void allreduce_host(gavis_comm* cm, std::vector<double>& v, const char* name) {
  gavis_ctx* c = cm->ctx;
  if (v.empty()) return;
  double* d = (double*)c->buf(name, sizeof(double) * v.size());
  CK(cudaMemcpyAsync(d, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, c->stream));
  nck(nccl().all_reduce(d, d, v.size(), ncclFloat64, ncclSum, cm->comm, c->stream), "ncclAllReduce");
  CK(cudaMemcpyAsync(v.data(), d, sizeof(double) * v.size(), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
}

}  // namespace

extern "C" {

gavis_status gavis_comm_unique_id(uint8_t* id_out) {
  return guard([&] {
    require(id_out != nullptr, "null argument");
    static_assert(sizeof(ncclUniqueId) == GAVIS_COMM_ID_BYTES, "unique id size");
    ncclUniqueId id;
    nck(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof id);
  });
}

gavis_status gavis_comm_create(gavis_ctx* c, const uint8_t* id, int32_t nranks, int32_t rank,
                               gavis_comm** out) {
  return guard([&] {
    require(c && id && out, "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "comm: rank must lie in [0, nranks)");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    auto* cm = new gavis_comm();
    cm->ctx = c;
    cm->nranks = nranks;
    cm->rank = rank;
    cm->owned = true;
    const ncclResult_t r = nccl().comm_init_rank(&cm->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      delete cm;
      nck(r, "ncclCommInitRank");
    }
    *out = cm;
  });
}

gavis_status gavis_comm_adopt(gavis_ctx* c, void* nccl_comm, int32_t nranks, int32_t rank,
                              gavis_comm** out) {
  return guard([&] {
    require(c && nccl_comm && out, "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, "comm: rank must lie in [0, nranks)");
    (void)nccl();
    auto* cm = new gavis_comm();
    cm->ctx = c;
    cm->comm = static_cast<ncclComm_t>(nccl_comm);
    cm->nranks = nranks;
    cm->rank = rank;
    cm->owned = false;
    *out = cm;
  });
}

gavis_status gavis_comm_destroy(gavis_comm* cm) {
  return guard([&] {
    if (!cm) return;
    if (cm->owned && cm->comm) {
      std::lock_guard<std::recursive_mutex> lk(cm->ctx->mu);
      cm->ctx->use();
      cm->ctx->sync();
      nck(nccl().comm_destroy(cm->comm), "ncclCommDestroy");
    }
    delete cm;
  });
}

gavis_status gavis_vf_allreduce(gavis_comm* cm, gavis_field* f) {
  return guard([&] {
    require(cm && f, "null argument");
    invariant(f->ctx == cm->ctx, "vf_allreduce: field and communicator belong to different contexts");
    std::lock_guard<std::recursive_mutex> lk(cm->ctx->mu);
    cm->ctx->use();
    allreduce_field(cm, f);
  });
}

gavis_status gavis_vf_construct_sharded(gavis_comm* cm, const gavis_scene* s, const gavis_camera* views,
                                        int32_t n_views, double kappa, int32_t degree,
                                        const gavis_raster_config* rc, gavis_field** out) {
  gavis_field* f = nullptr;
  const gavis_status st = guard([&] {
    require(cm && s && out, "null argument");
    require(n_views > 0 && views != nullptr, "construct_field: trajectory must be nonempty");
    gavis_ctx* c = cm->ctx;
    int64_t lo, hi;
    block_of(n_views, cm->rank, cm->nranks, &lo, &hi);
    check(gavis_vf_create(c, s, kappa, degree, &f));
    if (hi > lo) check(gavis_vf_accumulate_views(c, f, s, views + lo, (int32_t)(hi - lo), rc));
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    allreduce_field(cm, f);
    f->num_views = n_views;  // construct_field: num_views = |P| (vfield.hpp:91)
    *out = f;
  });
  if (st != GAVIS_OK && f && (!out || *out != f)) gavis_vf_destroy(f);
  return st;
}

gavis_status gavis_select_nbv_sharded(gavis_comm* cm, const gavis_scene* s, const gavis_field* f,
                                      const gavis_camera* cams, int32_t n_cams,
                                      const gavis_raster_config* rc, const gavis_uncertainty_config* uc,
                                      int32_t with_rgb, double* scores, int32_t* best) {
  return guard([&] {
    require(cm && s && f, "null argument");
    require(n_cams > 0 && cams != nullptr, "select_nbv: candidate list must be nonempty");
    gavis_ctx* c = cm->ctx;
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    ScoringPrecision sp(c, uc);
    const int W = cm->nranks;
    int64_t lo, hi;
    block_of(n_cams, cm->rank, W, &lo, &hi);
    int64_t width = 0;
    for (int r = 0; r < W; ++r) {
      int64_t a, b;
      block_of(n_cams, r, W, &a, &b);
      width = std::max(width, b - a);
    }
    // this rank's block, scored into a padded slot of the gather buffer
    std::vector<double> mine((size_t)std::max<int64_t>(1, width), 0.0);
    c->score_bounds.clear();
    if (hi > lo) {
      gavis_render_outputs o = {};
      o.scores = mine.data();
      o.with_rgb = with_rgb;
      ua_render(c, s, f, nullptr, cams + lo, (int)(hi - lo), rc, uc, &o);
    }
    // scores and (certified mode) their error bounds, gathered in one call:
    // [scores | bounds] per rank, padded to the widest block
    const bool bounded = hi > lo ? c->score_bounds.size() == (size_t)(hi - lo)
                                 : c->precision == GAVIS_PRECISION_CERTIFIED;
    std::vector<double> send((size_t)(2 * width), 0.0);
    std::copy(mine.begin(), mine.begin() + (hi - lo), send.begin());
    if (bounded && hi > lo) std::copy(c->score_bounds.begin(), c->score_bounds.end(), send.begin() + width);
    double* dsend = (double*)c->buf("nbv_send", sizeof(double) * 2 * width);
    double* drecv = (double*)c->buf("nbv_recv", sizeof(double) * 2 * width * W);
    CK(cudaMemcpyAsync(dsend, send.data(), sizeof(double) * 2 * width, cudaMemcpyHostToDevice, c->stream));
    nck(nccl().all_gather(dsend, drecv, (size_t)(2 * width), ncclFloat64, cm->comm, c->stream),
        "ncclAllGather(scores)");
    std::vector<double> all((size_t)(2 * width * W));
    CK(cudaMemcpyAsync(all.data(), drecv, sizeof(double) * 2 * width * W, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    std::vector<double> sc((size_t)n_cams), bd((size_t)n_cams);
    for (int r = 0; r < W; ++r) {
      int64_t a, b;
      block_of(n_cams, r, W, &a, &b);
      const size_t o = (size_t)r * 2 * width;
      std::copy(all.begin() + o, all.begin() + o + (b - a), sc.begin() + a);
      std::copy(all.begin() + o + width, all.begin() + o + width + (b - a), bd.begin() + a);
    }
    // every rank holds the same bounds: the contender window is rank-independent
    // (a rank whose block was empty learns the mode from its context)
    int any_bounds = 0;
    for (double x : bd) any_bounds |= x > 0.0;
    if (any_bounds) c->score_bounds = bd;
    else c->score_bounds.clear();
    // certified mode: contenders re-scored in fp64 by their owners, summed over ranks
    std::vector<int> cont = certified_contenders(c, s, rc, sc);
    if (cont.size() >= 2) {
      std::vector<double> exact((size_t)n_cams, 0.0);
      std::vector<int> own;
      std::vector<gavis_camera> cc;
      for (int i : cont)
        if (i >= lo && i < hi) {
          own.push_back(i);
          cc.push_back(cams[i]);
        }
      if (!own.empty()) {
        std::vector<double> ex(own.size());
        gavis_render_outputs o = {};
        o.scores = ex.data();
        const int32_t prec = c->precision;
        const std::vector<double> keep = c->score_bounds;  // the fp64 re-render must not clear them
        c->precision = GAVIS_PRECISION_EXACT;
        try {
          ua_render(c, s, f, nullptr, cc.data(), (int)cc.size(), rc, uc, &o);
        } catch (...) {
          c->precision = prec;
          c->score_bounds = keep;
          throw;
        }
        c->precision = prec;
        c->score_bounds = keep;
        for (size_t k = 0; k < own.size(); ++k) exact[own[k]] = ex[k];
        c->rescored_views += (int64_t)own.size();
      }
      allreduce_host(cm, exact, "nbv_exact");  // disjoint non-zeros: x + 0 = x exactly
      for (int i : cont) sc[i] = exact[i];
    }
    int b = 0;
    for (int i = 1; i < n_cams; ++i)
      if (sc[i] > sc[b]) b = i;  // planner.hpp:132-136
    if (scores) std::memcpy(scores, sc.data(), sizeof(double) * n_cams);
    if (best) *best = b;
  });
}

}  // extern "C"
