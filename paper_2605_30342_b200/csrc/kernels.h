// kernels.h -- host-callable launchers of the sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "device_common.cuh"

namespace gavis {

// Device-resident scene (fp32 SoA, 16-byte vectors).
struct SceneDev {
  int64_t n = 0;
  int color_degree = 0;
  int nb = 1;       // (Lc+1)^2
  int cstride = 4;  // floats per particle in `colors` (3*nb rounded up to 4)
  const float4* pos_op = nullptr;  // x, y, z, opacity
  const float4* rot = nullptr;     // w, x, y, z
  const float4* scale = nullptr;   // sx, sy, sz, 0
  const uint8_t* virt = nullptr;
  const float* colors = nullptr;
  // the colours as the tensor-core colour path stages them (kernels_ua_fast.cu):
  // per particle 13 x 16 B, fp16 hi/lo splits; built once per scene, or null
  const uint4* colors_split = nullptr;
};

enum QueryMode : int { kQueryNone = 0, kQueryField = 1, kQueryGiven = 2 };

struct PreprocessArgs {
  SceneDev scene;
  const DevCam* cams = nullptr;
  int V = 0;
  double dilation = 0.3;
  int tile_size = 16;
  GeoRec* geo = nullptr;     // [V*N]
  UaRec* ua = nullptr;       // [V*N] (null for VF)
  int32_t* counts = nullptr; // [V*N] tiles touched
  uint2* trect = nullptr;    // [V*N] tx0|tx1<<16, ty0|ty1<<16
  int query_mode = kQueryNone;
  const double* gamma = nullptr;  // [N*(L+1)^2]
  int degree = 0;
  int num_views = 0;
  const double* vis_in = nullptr;  // [N] for kQueryGiven
  double beta = 0.5, o0b = 0.075;  // o0b = o0 * (1 - beta)
  double hl_const = 0.0;           // 3 ln sigma_c (constant provider)
  const float* var = nullptr;      // [N][3][(Lv+1)^2] coefficient variances (sh_propagation)
  int var_degree = -1;
  int* err_flag = nullptr;         // set to 1 when a propagated variance is not positive
  bool write_culled = false;
  // depth-ordered binning: visible (view, particle) items appended (warp-aggregated,
  // any order: the stable key sort + depth_order fix the final order) with their
  // 32-bit keys (view | leading fp32 depth bits); null in the 64-bit key path
  bool cull_counts = true;             // write count 0 / empty rect for culled slots (false:
                                       // nothing reads them -- UA renders with appended items)
  uint32_t* item_slot_out = nullptr;   // [V*N] capacity
  uint32_t* item_key_out = nullptr;    // [V*N] capacity
  uint32_t* n_items_out = nullptr;     // [1], zeroed by the caller
  int view_bits = 1;
  unsigned long long* pair_total = nullptr;  // [1] sum of tile counts, zeroed by the caller
};

struct EmitArgs {
  const DevCam* cams = nullptr;
  int V = 0;
  int64_t N = 0;
  const GeoRec* geo = nullptr;
  const int32_t* counts = nullptr;
  const int32_t* offsets = nullptr;
  const uint2* trect = nullptr;
  uint64_t* keys = nullptr;
  uint32_t* vals = nullptr;
  uint32_t* pair_gid = nullptr;  // VF mode: vals = pair index, pair_gid[pair] = particle
};

// Depth-ordered binning (kernels_preprocess.cu): particles sorted by depth per
// view, pairs emitted in that order, then stably sorted by tile id.
struct NarrowArgs {
  int64_t N = 0;
  const GeoRec* geo = nullptr;
  const int32_t* counts = nullptr;     // [V*N] tiles touched
  int64_t n_items = 0;                 // visible (view, particle) items
  const uint32_t* item_slot = nullptr; // [n_items] slots in slot order (selection output)
  uint32_t* item_key = nullptr;        // [n_items] view | leading depth bits (sorted)
  int view_bits = 1;                   // bits of the view index in item_key (>= 1)
  uint32_t* item_slot_sorted = nullptr;
  int32_t* item_count = nullptr;       // [n_items + 1] tiles of each item, depth order
  const int32_t* item_offset = nullptr;  // exclusive scan of item_count
  int32_t* slot_offset = nullptr;      // [V*N] pair offset of each visible slot
  const int64_t* chunk_tile_base = nullptr;  // [V] first tile of the view's sort chunk
  uint32_t* keys32 = nullptr;          // [K] tile ids relative to the chunk's first tile
  uint32_t* scratch = nullptr;         // [n_items] merge buffer for long tied runs
  uint2* long_runs = nullptr;          // [n_items / (kShortRun + 1) + 1] (start, length)
  uint32_t* n_long = nullptr;          // long runs found (zeroed before depth_order)
};

// Runs of equal 32-bit item keys up to this length are ordered by one thread
// (insertion sort); longer ones by a CTA each (depth_order_long_kernel).
constexpr int kShortRun = 32;

struct RangesArgs {
  const DevCam* cams = nullptr;
  int V = 0;
  int64_t N = 0;
  int64_t K = 0;
  const uint64_t* keys = nullptr;
  uint32_t* vals = nullptr;
  const uint32_t* pair_gid = nullptr;
  const GeoRec* geo = nullptr;
  uint2* ranges = nullptr;
};

struct VfBlendArgs {
  const DevCam* cams = nullptr;
  int V = 0;
  int64_t N = 0;
  int64_t total_tiles = 0;
  int tile_size = 16;
  double cutoff = 1e-4, amax = 0.99;
  const GeoRec* geo = nullptr;
  const uint2* ranges = nullptr;
  const uint32_t* vals = nullptr;      // sorted pair indices
  const uint32_t* pair_gid = nullptr;
  double* pair_sum = nullptr;          // [K] sum of T (original pair order)
  int32_t* pair_cnt = nullptr;         // [K]
  int32_t* contrib = nullptr;          // [V*W*H] or null
  bool fixed_sums = false;             // T in [0, 1] guaranteed (opacities >= 0): fixed-point sums allowed
};

struct VfFinalizeArgs {
  SceneDev scene;
  const DevCam* cams = nullptr;
  int V = 0;
  const int32_t* counts = nullptr;
  const int32_t* offsets = nullptr;
  const double* pair_sum = nullptr;
  const int32_t* pair_cnt = nullptr;
  const double* vis_given = nullptr;  // [N] accumulate caller-provided v (V == 1)
  double* gamma = nullptr;            // null: do not accumulate
  int degree = 0;
  double scales[kMaxFieldDegreeRT + 1] = {0};
  double* vis_out = nullptr;          // [V*N]
  int64_t* touch_out = nullptr;       // [V*N]
};

struct UaBlendArgs {
  SceneDev scene;
  const DevCam* cams = nullptr;
  int V = 0;
  int64_t total_tiles = 0;
  int tile_size = 16;
  double cutoff = 1e-4, amax = 0.99;
  double hl_qc = 0.0, hl_q0 = 0.0;
  const GeoRec* geo = nullptr;
  const UaRec* ua = nullptr;
  const uint2* ranges = nullptr;
  const uint32_t* vals = nullptr;  // sorted particle ids
  // outputs (device, camera-major); null = not written
  double* rgb = nullptr;
  double* depth = nullptr;
  double* trans = nullptr;
  double* entropy = nullptr;
  double* w0 = nullptr;
  double* edepth = nullptr;
  int32_t* rgb_contrib = nullptr;
  int32_t* ent_contrib = nullptr;
  double corr_lambda = 0.0;      // > 0: correlation hook in the image score
  bool do_rgb = true, do_ent = true;
  bool vis_outside_unit = false;   // caller-given visibility with entries outside [0, 1]
  // Certified fp32 path (kernels_ua_fast.cu): pixels whose early-termination
  // decision the fp32 error bound cannot certify are appended to flag_list
  // (batch pixel index) and recomputed by the fp64 redo kernel.
  uint32_t* flag_list = nullptr;   // [total_pix]
  uint32_t* flag_count = nullptr;  // [1]
  float cert_base = 0.f;           // relative window, constant part
  float cert_per_step = 0.f;       // relative window per composited entry
  float cert_sum = 0.f;            // relative window per unit of sum a/(1-a)
  float cert_per_step2 = 0.f;      // second bound (small-alpha steps folded into S)
  float cert_sum2 = 0.f;
  // Rigorous bound on |H_fp32 - H_fp64| per pixel (certified path, constant
  // variance provider, no correlation hook): written when non-null; folded per
  // view like the score (kernels_ua_fast.cu header, "score bound").
  double* score_bound = nullptr;   // [total_pix]
  double bound_tail = 0.0;         // per composited entry: 1.7e-3 u o_max (|c| + 89)
  double w0_tail = 0.0;            // per composited entry: 1.7e-3 u o_max
  double c0_abs = 0.0;             // |1/2 ln|Q0| + C_H| of the prior term
  double c_ent = 0.0;              // c = 3 ln sigma_c + C_H of every entry
};

// Per-pixel mixtures of the entropy track for one view (kernels_mixture.cu).
struct MixtureArgs {
  SceneDev scene;
  const DevCam* cam = nullptr;
  int tile_size = 16;
  double cutoff = 1e-4, amax = 0.99, hl_q0 = 0.0, var_const = 0.01;
  const GeoRec* geo = nullptr;
  const UaRec* ua = nullptr;
  const uint2* ranges = nullptr;
  const uint32_t* vals = nullptr;
  const float* var = nullptr;  // sh_propagation coefficient variances or null
  int var_degree = -1;
  // pass 1 (comps == null): counts, prior, resid, entropy; pass 2: comps at offsets
  int64_t* counts = nullptr;
  double* prior = nullptr;
  double* resid = nullptr;
  double* entropy = nullptr;
  const int64_t* offsets = nullptr;
  double* comps = nullptr;  // [K][8]
};

struct QueryArgs {
  const double* gamma = nullptr;
  const uint8_t* virt = nullptr;
  int degree = 0;
  int num_views = 0;
  const int64_t* idx = nullptr;
  const double* dirs = nullptr;
  int64_t n = 0;
  double* out = nullptr;
};

struct PackSceneArgs {
  int64_t n = 0;
  int nb = 1, nbp = 2, cstride = 8;
  const float* pos = nullptr;     // [n][3]
  const float* op = nullptr;      // [n]
  const float* scale = nullptr;   // [n][3]
  const float* colors = nullptr;  // [n][3][nb], or null: colours copied directly
  const uint8_t* virt = nullptr;  // [n] or null
  float4* pos_op = nullptr;
  float4* scale4 = nullptr;
  float* colors_out = nullptr;
  uint8_t* virt_out = nullptr;
};

void launch_pack_scene(const PackSceneArgs& a, cudaStream_t s);
void launch_preprocess(const PreprocessArgs& a, cudaStream_t s);
void launch_emit_keys(const EmitArgs& a, cudaStream_t s);
void launch_ranges(const RangesArgs& a, cudaStream_t s);
void launch_depth_order(const NarrowArgs& a, cudaStream_t s);
void launch_emit_tiles(const EmitArgs& a, const NarrowArgs& n, cudaStream_t s);
void launch_ranges32(const uint32_t* keys32, int64_t lo, int64_t hi, int64_t tile_base, uint2* ranges,
                     cudaStream_t s);
void launch_view_pair_starts(const NarrowArgs& a, int V, int64_t* out, cudaStream_t s);
void launch_wide_keys(const uint2* ranges, int64_t total_tiles, const uint32_t* vals,
                      const uint32_t* pair_gid, const DevCam* cams, int V, int64_t N, const GeoRec* geo,
                      uint64_t* keys, cudaStream_t s);

void launch_vf_blend(const VfBlendArgs& a, cudaStream_t s);
void launch_vf_finalize(const VfFinalizeArgs& a, int64_t N, cudaStream_t s);
void launch_ua_blend(const UaBlendArgs& a, cudaStream_t s);
// Certified fp32 blend (16x16 tiles, alpha_clamp_max <= 0.999) + the fp64 redo
// of the flagged pixels; same outputs as launch_ua_blend (tile_score unused).
bool ua_fast_supported(int tile_size, double amax);
// exact fp64 blend with the tensor-core colour (16x16 tiles, RGB, split colours)
bool ua_exact_mma_supported(const UaBlendArgs& a);
void launch_ua_blend_exact_mma(const UaBlendArgs& a, cudaStream_t s);
void launch_ua_blend_fast(const UaBlendArgs& a, cudaStream_t s);
void launch_ua_redo(const UaBlendArgs& a, cudaStream_t s);
// The staged colour form of the tensor-core colour path: its size in bytes, 0
// when the fast blend stages fp32 colours instead (GAVIS_UA_COLOR=ffma).
size_t ua_colors_split_bytes(const SceneDev& scene);
void launch_split_colors(const SceneDev& scene, uint4* out, cudaStream_t s);
// image_entropy per view: fixed-order fold of the per-pixel entropy image
// (with the correlation hook when corr_lambda > 0; edepth must then be set).
void launch_score_image(const DevCam* cams, int V, const double* entropy, const double* edepth,
                        double corr_lambda, double* partial, double* scores, cudaStream_t s);
int score_partials_per_view();
void launch_add_count(unsigned long long* total, const uint32_t* count, cudaStream_t s);
void launch_query(const QueryArgs& a, cudaStream_t s);
void launch_mixtures(const MixtureArgs& a, int64_t P, cudaStream_t s);
// unseen[k] *= 1 - vis[v*N + n_real + k] for v = 0..V-1 in order.
void launch_density_update(double* unseen, const double* vis, int V, int64_t N, int64_t n_real,
                           int64_t n_virtual, cudaStream_t s);

// CUB-backed device primitives (sort.cu)
size_t scan_temp_bytes(int64_t n);
void exclusive_scan(const int32_t* in, int32_t* out, int64_t n, void* temp, size_t temp_bytes,
                    cudaStream_t s);
size_t sort_temp_bytes(int64_t n);
// Sorts (keys, vals) ascending by bits [0, end_bit); results land in the
// buffers returned through *keys_out / *vals_out (one of the two pairs).
void radix_sort_pairs(uint64_t* keys_a, uint64_t* keys_b, uint32_t* vals_a, uint32_t* vals_b,
                      int64_t n, int end_bit, void* temp, size_t temp_bytes, cudaStream_t s,
                      uint64_t** keys_out, uint32_t** vals_out);
size_t sort32_temp_bytes(int64_t n);
// 32-bit keys (stable); the sorted pairs always end in (keys_a, vals_a).
void radix_sort_pairs32(uint32_t* keys_a, uint32_t* keys_b, uint32_t* vals_a, uint32_t* vals_b,
                        int64_t n, int end_bit, void* temp, size_t temp_bytes, cudaStream_t s);

}  // namespace gavis
