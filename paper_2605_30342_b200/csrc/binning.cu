// binning.cu -- K1..K5 for a batch of views: preprocess, depth-ordered
// emission of (tile, particle) pairs, stable tile sort, tile ranges; and the
// debug exports of the projection and of the sorted pairs (parity tests).
#include "host.h"

namespace gavis {
namespace host {

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
    // ~112 B of per-(view, particle) state per batch, up to three buffer sets in
    // flight: one batch may use a ninth of the free device memory, within [2, 16] GB
    if (c->batch_budget == 0.0) {
      size_t free_b = 0, total_b = 0;
      CK(cudaMemGetInfo(&free_b, &total_b));
      c->batch_budget = std::min(16.0e9, std::max(2.0e9, (double)free_b / 9.0));
    }
    const int64_t by_mem = (int64_t)(c->batch_budget / (112.0 * (double)N));
    vmax = (int)std::max<int64_t>(1, std::min<int64_t>(vmax, by_mem));
  }
  vmax = std::min(vmax, 64);
  return std::max(1, std::min(vmax, n_views));
}

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
  // GAVIS_BIN_WIDE=1 selects the 64-bit (tile << 32 | fp32 depth) key path (A/B and
  // the equivalence test); it is also the path of the reference-form debug keys
  const char* wide_env = std::getenv("GAVIS_BIN_WIDE");
  const bool narrow = !o.force_wide && !(wide_env && wide_env[0] == '1');
  // 64-bit pair total (K1), read with the first host sync below: a batch whose
  // pairs exceed the 32-bit pair indexing or the pair memory budget is split by
  // the caller
  unsigned long long* dtotal = (unsigned long long*)c->buf("pair_total", sizeof(unsigned long long));
  CK(cudaMemsetAsync(dtotal, 0, sizeof(unsigned long long), c->stream));
  pa.pair_total = dtotal;
  uint32_t* items = nullptr;
  uint32_t* ik_a = nullptr;
  uint32_t* dnum = nullptr;
  if (VN > 0 && narrow) {
    // K1 appends the visible (view, particle) items with their depth keys
    items = (uint32_t*)c->buf("items", sizeof(uint32_t) * VN);
    ik_a = (uint32_t*)c->buf("item_key_a", sizeof(uint32_t) * VN);
    dnum = (uint32_t*)c->buf("items_num", sizeof(uint32_t));
    CK(cudaMemsetAsync(dnum, 0, sizeof(uint32_t), c->stream));
    pa.item_slot_out = items;
    pa.item_key_out = ik_a;
    pa.n_items_out = dnum;
    pa.view_bits = std::max(1, bits_for(V));
    // the UA path reads counts and tile rects only through the appended items;
    // the VF finalize walks every slot
    pa.cull_counts = o.vf_mode || o.write_culled;
  }
  c->run("preprocess", [&] { launch_preprocess(pa, c->stream); }, N > 0 ? 1 : 0);
  const auto pairs_fit = [&]() {
    const uint64_t total = *reinterpret_cast<const unsigned long long*>(c->pinned + kPinPairs);
    // <= 32 B of pair state per pair (keys and values double-buffered, VF sums)
    const int64_t limit = std::min<int64_t>(
        (int64_t(1) << 31) - 1,
        c->pair_budget > 0    ? c->pair_budget
        : c->batch_budget > 0.0 ? (int64_t)(c->batch_budget / 32.0)
                                : (int64_t(1) << 31) - 1);
    if (V > 1 && total > (uint64_t)limit) return false;
    invariant(total < (uint64_t(1) << 31),
              "one view produces 2^31 or more tile pairs (the device path indexes pairs in 32 bits)");
    return true;
  };

  int32_t* P32 = c->pinned;
  int64_t K = 0, n_items = 0;
  NarrowArgs na;
  if (VN > 0 && narrow) {
    // visible items (K1) -> sorted by (view, depth) -> tile counts in that order -> pair offsets
    CK(cudaMemcpyAsync(P32 + kPinItems, dnum, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(P32 + kPinPairs, dtotal, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       c->stream));
    c->sync();
    if (!pairs_fit()) {
      b.overflow = true;
      return b;
    }
    n_items = P32[kPinItems];
    na.N = N;
    na.geo = b.geo;
    na.counts = b.counts;
    na.n_items = n_items;
    na.item_slot = items;
    if (n_items > 0) {
      uint32_t* ik_b = (uint32_t*)c->buf("item_key_b", sizeof(uint32_t) * n_items);
      uint32_t* is_b = (uint32_t*)c->buf("item_slot_b", sizeof(uint32_t) * n_items);
      na.item_key = ik_a;
      na.view_bits = std::max(1, bits_for(V));
      const size_t isb = sort32_temp_bytes(n_items);
      void* itmp = c->buf("sort_tmp", isb);
      c->run("sort", [&] {
        radix_sort_pairs32(ik_a, ik_b, items, is_b, n_items, 32, itmp, isb, c->stream);
      });
      na.item_slot_sorted = items;
      na.item_count = (int32_t*)c->buf("item_count", sizeof(int32_t) * (n_items + 1));
      int32_t* ioff = (int32_t*)c->buf("item_offset", sizeof(int32_t) * (n_items + 1));
      CK(cudaMemsetAsync(na.item_count + n_items, 0, sizeof(int32_t), c->stream));
      na.scratch = is_b;  // free after the sort: merge buffer of the long tied runs
      na.long_runs = (uint2*)c->buf("long_runs", sizeof(uint2) * (n_items / (kShortRun + 1) + 1));
      na.n_long = (uint32_t*)c->buf("n_long", sizeof(uint32_t));
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
    CK(cudaMemcpyAsync(P32 + kPinPairs, dtotal, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       c->stream));
    c->sync();
    if (!pairs_fit()) {
      b.overflow = true;
      return b;
    }
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

}  // namespace host
}  // namespace gavis

extern "C" {

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
      const bool ok = !std::isnan(g[i].depth);  // K1 marks culled slots with a NaN depth
      if (culled) culled[i] = ok ? 0 : 1;
      if (mean) {
        mean[2 * i] = g[i].mx;
        mean[2 * i + 1] = g[i].my;
      }
      if (conic) {
        conic[3 * i] = -2.0 * g[i].na;  // (a, b, c) from the pre-scaled record: exact
        conic[3 * i + 1] = -g[i].nb;
        conic[3 * i + 2] = -2.0 * g[i].nc;
      }
      if (depth) depth[i] = g[i].depth;
      if (cover_rect) {
        // (x0, x1, y0, y1); an empty axis as (1, 0)
        const int32_t cv[2] = {g[i].cov_x, g[i].cov_y};
        for (int ax = 0; ax < 2; ++ax) {
          const int lo = cv[ax] & 0xFFFF, w = (int)((uint32_t)cv[ax] >> 16);
          const bool empty = cv[ax] == kCovEmpty;
          cover_rect[4 * i + 2 * ax] = empty ? 1 : lo;
          cover_rect[4 * i + 2 * ax + 1] = empty ? 0 : lo + w;
        }
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
