// lgs_kernels.h -- launch entry points of the sm_100a kernels (host-callable).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace lgs {

struct DevCam;
struct DevMap;
struct ColorJob;

// Per-view projected records, indexed by map index (written by K1).
struct ViewBufs {
  float4* rec0;     // u, v, depth, opacity
  float4* rec1;     // conic A, B, C (q = A dx^2 + 2B dx dy + C dy^2), radius
  uint2* rect;      // x0 | x1 << 16, y0 | y1 << 16 (inclusive pixel rect, renderer.cpp:131-134)
  float4* color;    // r, g, b, 0
  uint32_t* tiles;  // tiles touched (0 = culled)
  uint32_t* dkey;   // f32 bits of depth (0xffffffff = culled) -> depth sort key
  uint32_t* iota;   // map index
  // optional (depth-layered binning): K1 also adds each visible Gaussian to its depth bucket
  // (depth_order.cu): dhist[bucket] += 1 << 32 | tiles, dslot[i] = its slot in the bucket
  unsigned long long* dhist = nullptr;
  uint32_t* dslot = nullptr;
  uint32_t dbase = 0;  // near-plane bucket offset (depth_bucket)
  uint32_t* dpart = nullptr;  // ... and stores each CTA's pair sum here (ceil(n / kPreThreads) words)
  // Gaussians that can hold a nonzero screen-space gradient (listed in some traversed tile list);
  // null: every visible one.  The backward zeroes and reads only their accumulator rows.
  uint8_t* active = nullptr;
};

// active[] of the depth-layered binning: the layer-A candidates (flagged by the depth order; the
// second pass adds the Gaussians it lists); zero_active_rows clears their backward accumulator rows.
void launch_zero_active_rows(const ViewBufs& v, int64_t n, float* gacc, int slots, cudaStream_t s);

// Tile lists for the blend kernels.
struct TileLists {
  const uint32_t* vals;    // map index per list entry, sorted by (tile, depth, index)
  const uint2* ranges;     // [tiles] begin, end
  const uint32_t* order;   // [tiles] tile ids, longest list first (persistent scheduler)
  int* counter;            // scheduler slot counter (reset by the launcher)
  const uint32_t* count = nullptr;  // device count of tiles in `order` (null: every tile)
};

// Longest-first tile order (binning_fast.cu): buckets by floor(log2(list length)).
void launch_tile_order(const uint2* ranges, int ntiles, uint32_t* order, cudaStream_t s);

// Per-pixel forward state kept for the backward pass.
struct PixelState {
  float* final_t;      // transmittance after the last evaluated Gaussian
  uint32_t* n_contrib; // list position (relative to the tile begin) after the last contributor
  float* depth;        // normalized depth (renderer.cpp:163-165), read by the backward
  float* acc;          // accumulated alpha
  uint2* work;         // per pixel: (evaluated pairs, contributing pairs)
};

struct FwdOut {
  float* rgb;    // [H][W][3] or null
  float* depth;  // [H][W] or null
  float* feat;   // [H][W][d] or null
  float* acc;    // [H][W] or null
  // fused L1 (optional)
  const float* t_rgb;
  const float* t_depth;
  const float* t_feat;
  float* cot;        // [H][W][4 + d]: g_rgb(3), g_depth, g_feat(d)
  double* loss;      // 1 double (atomic sum)
  // depth-layered first pass: tiles not saturated by their (prefix) list are flagged here and get
  // no loss / cotangents (the second pass renders them again on their complete lists)
  uint32_t* unfinished = nullptr;
  // ... and, if set (a speculative plan without pass 2), any such tile stores 1 into mapped host
  // memory (read by lgs_plan_sync) and into a device word (read by the chain: miss, GradOut::skip)
  uint32_t* unfinished_any = nullptr;
  uint32_t* miss = nullptr;
  // ... and every warp of a saturated tile adds the list length its pixels consumed (the layer-A
  // size policy of lgs_capi.cu)
  uint32_t* consumed = nullptr;
  // ... and (plans, first pass) each tile's duration in units of 16 SM cycles (the next replays'
  // longest-first tile order, launch_tile_order_lpt)
  uint32_t* tile_cost = nullptr;
};

struct BwdIn {
  const float* g_rgb;    // [H][W][3] or null
  const float* g_depth;  // [H][W] or null
  const float* g_feat;   // [H][W][d] or null
  int cot_stride;        // 0: separate images; else interleaved [H][W][cot_stride] (fused L1 layout)
};

void launch_pack_map(const float* pos, const float* rot, const float* log_s, const float* opac,
                     const float* feat_dn, int64_t n, int d, int dp, float4* pos_opa, float4* rot4,
                     float4* scale4, float* feat_nd, cudaStream_t s);

// color = false (depth-layered binning): colours are computed lazily (ColorJob) for the listed ones
void launch_preprocess(const DevMap& m, const DevCam& c, const ViewBufs& v, bool color, cudaStream_t s);
// [d][N] -> packed [N][dp] features of every Gaussian (a host-mapped map rendered without the
// layered binning)
void launch_gather_features(const float* src, float* dst, int64_t n, int d, int dp, cudaStream_t s);
// colours of every visible Gaussian (debug exports of a layered render)
void launch_colors(const DevMap& m, const DevCam& c, const ViewBufs& v, cudaStream_t s);

// Binning (binning.cu).  The pair count is read back once per view (host sync) to size the
// pair arrays and the sort.
size_t binning_temp_bytes(int64_t n, int64_t pairs_cap, int tile_bits);
void launch_sum_tiles(const uint32_t* tiles, int64_t n, uint32_t* out, cudaStream_t s);
void launch_depth_sort(const ViewBufs& v, int64_t n, uint32_t* dkey_sorted, uint32_t* idx_sorted,
                       void* temp, size_t temp_bytes, cudaStream_t s);
void launch_scan_tiles(const uint32_t* tiles, const uint32_t* idx_sorted, int64_t n, uint32_t* scratch,
                       uint32_t* incl, void* temp, size_t temp_bytes, cudaStream_t s);
void launch_scan_counts(const uint32_t* cnt_sorted, int64_t n, uint32_t* incl, void* temp, size_t temp_bytes,
                        cudaStream_t s);
// Global (depth, index) order without a device radix sort (depth_order.cu): idx_sorted = visible
// Gaussians in (depth key, map index) order, then the culled ones; cnt_sorted = their tile counts.
size_t depth_order_temp_bytes(int64_t n);
void launch_depth_order(const ViewBufs& v, int64_t n, float near_plane, void* temp, size_t temp_bytes,
                        uint32_t* idx_sorted, uint32_t* cnt_sorted, cudaStream_t s);
// Depth-layered binning: order only layer A = the bucket prefix owning ~max(min(P, min_pairs), P / div)
// pairs (at most gauss_cap Gaussians, cap_a pairs): idx_sorted[0, R_A), their tile rects cand_rect,
// *ra = R_A.  launch_depth_order_rest (same temp) orders the remaining Gaussians afterwards.
// Split for the layered path: depth_prepare (before K1: zeroes the histogram, sets v.dhist/dslot/
// dbase so K1 fills it), depth_scan (after K1: bucket offsets; *pairs_out = device address of the
// visible pair total P), then launch_depth_order_layer_a (cut, scatter, rank of layer A).
// depth_scan is one launch; given `cut` it also applies the layer-A cut with those parameters
// (from the pair total K1's partial sums give), and layer_a is then called with cut_ready.
struct LayerCut {
  uint32_t div, min_pairs, cap_a;
  int64_t gauss_cap;
};
void launch_depth_prepare(int64_t n, float near_plane, void* temp, ViewBufs* v, cudaStream_t s);
void launch_depth_scan(int64_t n, float near_plane, void* temp, const LayerCut* cut, const uint32_t** pairs_out,
                       cudaStream_t s);
void launch_depth_order_layer_a(const ViewBufs& v, int64_t n, float near_plane, void* temp, uint32_t div,
                                uint32_t min_pairs, int64_t gauss_cap, uint32_t cap_a, uint32_t* idx_sorted,
                                uint2* cand_rect, uint32_t* ra, uint8_t* active, float* gacc_zero, bool rerun,
                                bool cut_ready, const ColorJob& cj, cudaStream_t s);
// gate (device, may be null): the kernels return at once when *gate == 0 (no unfinished tile)
void launch_depth_order_rest(const ViewBufs& v, int64_t n, float near_plane, void* temp, uint32_t* idx_sorted,
                             const uint32_t* gate, cudaStream_t s);
// Layer-A tile lists (one warp per tile scanning the depth-ordered candidates, order-preserving
// compaction): vals[ranges[t]] for every tile; *cursor (zeroed by the caller) allocates list space.
// Tiles longest layer-A list first (one CTA counting sort on the list lengths).
// cost (device, may be null): per-tile durations of the previous replay (FwdOut::tile_cost)
constexpr int kLptCostMaxTiles = 12288;
void launch_tile_order_lpt(const uint2* ranges, const uint32_t* cost, int ntiles, uint32_t* order, cudaStream_t s);
void launch_copy_u32(const uint32_t* src, int n, uint32_t* dst, cudaStream_t s);
void launch_layer_tile_lists(const uint2* cand_rect, const uint32_t* cand_idx, const uint32_t* n_cand, int tiles_x,
                             int ntiles, uint32_t* cursor, uint32_t* vals, uint2* ranges, int* blend_counter,
                             double* loss, uint32_t* miss, cudaStream_t s);
// blend_counter / loss (optional) are zeroed for the blend kernel launched next
void launch_duplicate(const ViewBufs& v, const uint32_t* idx_sorted, const uint32_t* incl, int64_t n,
                      int tiles_x, uint16_t* key_out, uint32_t* val_out, cudaStream_t s);
void launch_tile_sort(uint16_t* keys_in, uint16_t* keys_out, uint32_t* vals_in, uint32_t* vals_out,
                      int64_t pairs, int tile_bits, void* temp, size_t temp_bytes, cudaStream_t s);
void launch_ranges(const uint16_t* keys, int64_t pairs, int ntiles, uint2* ranges, cudaStream_t s);

// Fast binning (stable counting sort by tile; binning_fast.cu): writes the sorted lists into
// vals[base ..] and the per-tile `ranges` directly.  The pass's pair count is read on the device
// (`dev_pairs`), so the host never waits for it: if it exceeds `cap`, the pass's tile lists are left
// empty and *dev_overflow = 1 (the host then re-runs with exact buffers).  `scratch` must hold
// fast_binning_scratch_bytes(cap, gauss_cap, ntiles).
struct BinPass {
  const uint32_t* incl;       // inclusive pair counts of the depth-ordered Gaussians (this pass)
  const uint32_t* dev_pairs;  // this pass's pair count (device; = incl[n - 1])
  int64_t gauss_cap;          // upper bound on the Gaussians owning pairs in this pass
  uint32_t cap;               // list capacity of this pass
  uint32_t base;              // first list slot of this pass in vals
  const uint32_t* mask;       // tiles binned by this pass (null: all; else only ranges of masked tiles)
  const uint32_t* active = nullptr;  // with a mask: device count of masked tiles (0: the pass is a no-op)
  const uint32_t* clamp = nullptr;   // device pair total the inclusive counts are clamped at (layer A)
};
bool fast_binning_supported(int ntiles);
size_t fast_binning_scratch_bytes(int64_t cap, int64_t gauss_cap, int ntiles);
void launch_fast_binning(const ViewBufs& v, const uint32_t* idx_sorted, int64_t n, int ntiles, int tiles_x,
                         const BinPass& bp, uint32_t* scratch, uint32_t* vals, uint2* ranges, uint32_t* dev_overflow,
                         cudaStream_t s);
// Depth-layered binning (binning_fast.cu): layer A = the depth-order prefix owning ~P / div pairs
// (at most gauss_cap Gaussians), then the complete lists of the tiles layer A left unsaturated.
constexpr uint32_t kLayerMinPairs = 1u << 16;  // layer A takes at least this many pairs (or all)
size_t layer_a_cap(int64_t pairs_cap, int ntiles, uint32_t div);
// up to 4 device u32 counters -> mapped page-locked host memory (device address dst_mapped)
struct CounterSrc {
  const uint32_t* src[4];
  int n;
};
void launch_publish_counters(const CounterSrc& c, uint32_t* dst_mapped, cudaStream_t s);
// layer_flag: counts the unfinished tiles (count2), resets total2 and, inside a plan, sets the
// conditional of the second pass; layer_prep (first kernel of that pass): summed-area table of the
// unfinished mask and their longest-list-first order.
void launch_layer_flag(const uint32_t* unfinished, int ntiles, uint32_t* count2, uint32_t* total2,
                       const cudaGraphConditionalHandle* cond, cudaStream_t s);
void launch_layer_prep(const uint32_t* unfinished, const uint2* ranges, int tiles_x, int tiles_y, uint32_t* sat,
                       uint32_t* order2, cudaStream_t s);
void launch_layer_count(const ViewBufs& v, const uint32_t* idx_sorted, int64_t n, int tiles_x, const uint32_t* sat,
                        const uint32_t* count2, uint32_t* cnt_enum, uint32_t* total2, cudaStream_t s,
                        float* gacc_zero, const ColorJob& cj);

void launch_blend_fwd(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                      const PixelState& ps, const FwdOut& o, cudaStream_t s);
// K5 + K6 fused for the fused-L1 loss (blend_fused.cu): images, loss and the screen-space
// gradient accumulator gacc (rows of the listed Gaussians zeroed beforehand) in one pass per tile.
bool blend_fused_supported(int dp);
// long_lists: the second layered pass (few tiles, complete lists): the latency-bound variant
void launch_blend_fused_l1(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl, const FwdOut& o,
                           float* gacc, cudaStream_t s, bool counter_zeroed = false, bool long_lists = false);
void launch_blend_bwd(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                      const PixelState& ps, const BwdIn& in, float* gacc, int slots, cudaStream_t s);
// Row-sparse gradient exchange (sparse_reduce.cu): ptr/width = the six MapGradients attributes
// (feature is [d][N]).
void launch_rows_scan(float* const ptr[6], const int width[6], int64_t n, uint32_t* list, uint32_t* count,
                      cudaStream_t s);
int rows_values(const int width[6], float* const ptr[6]);
void launch_rows_pack(float* const ptr[6], const int width[6], int64_t n, const uint32_t* list, const uint32_t* count,
                      int64_t max_rows, float* rec, cudaStream_t s);
void launch_rows_apply(float* const ptr[6], const int width[6], int64_t n, const float* recs, const uint32_t* counts,
                       int world, int64_t stride, cudaStream_t s);
void launch_rows_overflow(const uint32_t* counts, int world, int64_t cap, uint32_t* out, cudaStream_t s);

struct GradOut {
  float* position;      // [N][3]
  float* rotation;      // [N][4] w,x,y,z
  float* log_scale;     // [N][3]
  float* opacity_logit; // [N]
  float* sh;            // [N][K][3]
  float* feature;       // [d][N]
  int accumulate;
  double* pose;         // 6 doubles (device, atomically accumulated) or null
  // device word or null: nonzero -> the chain writes nothing (a speculative plan's replay left a
  // tile unfinished; lgs_plan_sync re-runs it, so an accumulating replay must not add)
  const uint32_t* skip = nullptr;
  // captured steps, active-row chain only: its last CTA also writes the pose gradient as float to
  // pose_out (device or page-locked host memory, written in place) and copies copy_n words
  // copy_src -> copy_dst (the next replay's tile order) -- two launches and a copy node fewer.
  // done: CTA counter, zeroed with the pose accumulators.
  float* pose_out = nullptr;
  const uint32_t* copy_src = nullptr;
  uint32_t* copy_dst = nullptr;
  int copy_n = 0;
  uint32_t* done = nullptr;
};
// With v.active (depth-layered binning) only the active rows run the chain; every other row is
// written zero by launch_grad_zero first (skipped when `zeroed`: the caller already enqueued it).
void launch_preprocess_bwd(const DevMap& m, const DevCam& c, const ViewBufs& v, const float* gacc, int slots,
                           const GradOut& g, bool zeroed, cudaStream_t s);
// zero rows of every output attribute (no-op when g.accumulate)
void launch_grad_zero(const GradOut& g, int64_t n, int K, int d, cudaStream_t s);

// K8 mapping losses (loss.cu): SSIM + L1 on rgb, masked depth L1, decoder chain on features.
enum { LOSS_L1_RGB = 0, LOSS_SSIM = 1, LOSS_DEPTH_ABS = 2, LOSS_DEPTH_CNT = 3, LOSS_FEAT_ABS = 4, LOSS_COUNT = 8 };
struct LossArgs {
  int H = 0, W = 0;
  int d = 0, dp = 0, D = 0, hidden = 0;
  const float* rgb = nullptr;       // rendered [H][W][3]
  const float* depth = nullptr;     // rendered, alpha-normalized [H][W]
  const float* acc = nullptr;       // [H][W]
  const float* feat = nullptr;      // rendered [H][W][d]
  const float* rgb_gt = nullptr;    // keyframe [H][W][3]
  const float* depth_gt = nullptr;  // keyframe [H][W]
  const float* feat_gt = nullptr;   // keyframe [H][W][D]
  const float *w1 = nullptr, *b1 = nullptr, *w2 = nullptr, *b2 = nullptr;  // decoder
  double w_l1 = 0.8, w_depth = 0.5, w_feat = 1.0;
  float* abc = nullptr;             // scratch [9][H][W]
  double* sums = nullptr;           // [LOSS_COUNT]
  float* cot = nullptr;             // [H][W][cot_stride] = g_rgb 3 | g_depth | g_feat DP
  int cot_stride = 0;
};
bool decoder_supported(int hidden, int dp, int D);
void launch_pose_to_float(double* pose, float* same_storage, cudaStream_t s);
void launch_coverage(const float* acc, const float* depth, const float* measured, int64_t npix, uint8_t* mask,
                     unsigned long long* count, cudaStream_t s);
int launch_mapping_loss(const LossArgs& a, cudaStream_t s);  // 0 ok, else a CUDA error

// K10 Adam step / map unpack (optim.cu).  MapParams: writable view of packed map arrays (the map
// itself, or one of the Adam moment buffers, which share its layout).
struct MapParams {
  int64_t n = 0;
  int d = 0, dp = 0, K = 1;
  float4* pos_opa = nullptr;
  float4* rot = nullptr;
  float4* scale = nullptr;
  float* sh = nullptr;
  float* feat = nullptr;
};
struct GradIn {  // reference layouts (renderer.hpp:59-68)
  const float* position = nullptr;   // [N][3]
  const float* rotation = nullptr;   // [N][4] w,x,y,z
  const float* log_scale = nullptr;  // [N][3]
  const float* opacity = nullptr;    // [N]
  const float* sh = nullptr;         // [N][K][3]
  const float* feature = nullptr;    // [d][N]
};
struct AdamLr {
  float position, rotation, log_scale, opacity, sh_dc, sh_rest, feature;
};
void launch_adam(const MapParams& p, const MapParams& m, const MapParams& v, const GradIn& g, int64_t g0, int64_t g1,
                 const AdamLr& lr, double beta1, double beta2, double eps, int64_t step, cudaStream_t s);
void launch_unpack_map(const MapParams& p, float* pos, float* rot, float* log_s, float* opac, float* sh, float* feat_dn,
                       cudaStream_t s);

// ---- map pruning (prune.cu) ------------------------------------------------
struct PruneIn {
  const float4* pos_opa;  // x, y, z, opacity logit
  const float4* scale;    // log-scales
  const float* feat;      // [n][dp]
  int64_t n;
  int d, dp;
};
struct PruneParams {
  int k;
  double tau_dist, tau_sim, alpha_min, scale_max;
};
size_t prune_scratch_bytes(int64_t n);
// Greedy language rule (flags[i] = 1: killed); synchronizes the stream (host round loop).
cudaError_t run_language_redundant(const PruneIn& in, const PruneParams& pp, uint8_t* flags, void* scratch,
                                   int64_t* count, int64_t* candidates, int64_t* rounds, cudaStream_t s);
// scratch: 8 bytes of device memory
cudaError_t run_geometric(const PruneIn& in, const PruneParams& pp, uint8_t* flags, void* scratch, int64_t* count,
                          cudaStream_t s);
// Row compaction: keep[i] = !(drop_a[i] || drop_b[i]) (either may be null), dst_of = exclusive scan.
size_t compact_scratch_bytes(int64_t n);
cudaError_t run_compact(const uint8_t* drop_a, const uint8_t* drop_b, int64_t n, void* scratch, int64_t* kept,
                        uint32_t** keep, uint32_t** dst_of, cudaStream_t s);
struct RowCopies {
  const float* src[24];
  float* dst[24];
  int width[24];  // floats per row
  int count;
};
void launch_compact_rows(const RowCopies& rc, const uint32_t* keep, const uint32_t* dst_of, int64_t n, cudaStream_t s);

}  // namespace lgs
