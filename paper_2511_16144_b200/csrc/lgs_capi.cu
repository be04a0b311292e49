// lgs_capi.cu -- host side of the C ABI declared in include/lgs.h.
//
// Orchestrates one render (K1 preprocess -> depth sort -> scan -> K2 duplicate -> tile sort ->
// K4 ranges -> K5 blend) and one backward (K6 blend bwd -> K7 preprocess bwd) on the context's
// stream.  Device memory comes from the stream-ordered pool (cudaMallocAsync, release threshold
// raised so steady-state iterations reuse blocks without cudaMalloc).  No C++ exception crosses the
// ABI; failures return lgs_status with a thread-local message (lgs_last_error).
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../../include/lgs.h"
#include "dev_cache.h"
#include "lgs_internal.cuh"
#include "lgs_kernels.h"
#include "nccl_dyn.h"

using namespace lgs;

namespace {

thread_local std::string g_last_error;

lgs_status fail(lgs_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#define LGS_CUDA(call)                                                                              \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess) {                                                                        \
      return fail(e_ == cudaErrorMemoryAllocation ? LGS_ENOMEM : LGS_ECUDA, "%s: %s (%s:%d)", #call, \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                                      \
    }                                                                                               \
  } while (0)

#define LGS_TRY(expr)               \
  do {                              \
    lgs_status s_ = (expr);         \
    if (s_ != LGS_OK) return s_;    \
  } while (0)

int pad_dim(int d) {
  if (d == 0) return 0;
  if (d <= 4) return 4;
  if (d <= 8) return 8;
  if (d <= 16) return 16;
  return 32;
}

// device gradient buffers of a lgs_map_grads as the kernels' GradOut (no pose)
GradOut device_grad_out(const lgs_map_grads* g, int d) {
  GradOut go{};
  go.accumulate = g->accumulate;
  go.position = g->position; go.rotation = g->rotation; go.log_scale = g->log_scale;
  go.opacity_logit = g->opacity_logit; go.sh = g->sh; go.feature = d > 0 ? g->feature : nullptr;
  return go;
}

// layer A of the depth-layered binning owns ~1/kLayerDiv of the pairs (binning_fast.cu)
// (the starting value: lgs_ctx::layer_div adapts it per context)
constexpr uint32_t kLayerDiv = 16;
constexpr int64_t kSinglePassPairs = 16 << 20;  // complete lists in one pass at most this many pairs

int bits_for(int ntiles) {
  int b = 0;
  while ((1 << b) < ntiles) ++b;
  return b;
}

}  // namespace

struct PhaseMark {
  int phase;
  cudaEvent_t a, b;
};

struct lgs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::atomic<int> refs{1};
  std::atomic<int64_t> launches{0};
  uint32_t* host_u32 = nullptr;  // pinned scalar readback
  uint32_t* dev_u32 = nullptr;   // device scalars: [0] pair count, [1] binning overflow flag
  cudaEvent_t pairs_ready = nullptr;
  cudaMemPool_t pool = nullptr;  // this context's stream-ordered arena (no cross-context reuse waits)
  // blocks of 256 MB and more (tile lists of huge views: 8.8 GB at configs[4]) come from their own
  // pool: freed into the main pool they were carved up by the next render's small buffers, and the
  // next big request mapped fresh memory (36-48 ms of host time in the enqueue)
  cudaMemPool_t big_pool = nullptr;
  bool capturing = false;        // inside lgs_plan capture: no host waits, graph memory nodes
  std::vector<PhaseMark>* capture_marks = nullptr;  // lgs_plan capture: phase events recorded as graph nodes
  int64_t pairs_cap = 0;  // tile-list capacity for the next render (0: size from the exact count)
  bool full_lists = false;  // lgs_ctx_set_full_tile_lists: single-pass binning of every pair
  bool radix_depth = false;  // LGS_OPT_RADIX_DEPTH_ORDER: CUB radix sort for the depth order (cross-check)
  bool fused_eager = false;  // LGS_OPT_FUSED_EAGER: uncaptured fused-L1 renders run the fused kernel
  bool host_grad_delta = false;  // LGS_OPT_HOST_GRAD_DELTA: host gradients rewritten row-sparse
  bool no_speculative = false;   // LGS_OPT_SPECULATIVE_PLANS = 0: plans always capture pass 2
  // host-gradient delta mode: the destination of the previous backward and the rows it left nonzero
  std::array<float*, 6> delta_dst{};
  int64_t delta_n = -1;
  std::vector<uint32_t> delta_rows;
  // page-locked staging of the row records / row list read back by the delta mode (a pageable
  // destination would route every readback through the driver's bounce buffers and the CPU)
  void* delta_stage = nullptr;
  size_t delta_stage_bytes = 0;
  // bytes this context moved between host and device memory by copies (lgs_ctx_transfer_bytes)
  std::atomic<int64_t> bytes_h2d{0}, bytes_d2h{0};
  cudaStream_t cond_stream = nullptr;  // captures the body of a plan's conditional node
  cudaStream_t cond_parent = nullptr;  // the capturing stream while a body is captured
  // lgs_plan capture: the zero rows of the plan's (non-accumulating) gradient buffers are written
  // on a side branch forked after the preprocess and joined before the backward's chain kernel
  const lgs_map_grads* prezero = nullptr;
  bool prezero_forked = false;
  // lgs_plan capture: the plan's longest-list-first tile orders.  A replay's first-pass blend takes
  // tiles in the order computed from the previous replay's lists (cap_lpt_cur; identity before the
  // first), while the side branch computes this replay's into cap_lpt_next, copied to cur after the
  // join -- the ordering costs nothing on the critical path (the view is fixed between replays).
  uint32_t* cap_lpt_cur = nullptr;
  uint32_t* cap_lpt_next = nullptr;
  uint32_t* cap_tile_cost = nullptr;  // per-tile durations of the previous replay (first pass)
  bool lpt_forked = false;
  cudaStream_t side_stream = nullptr;
  cudaEvent_t side_fork = nullptr, side_join = nullptr;
  // multi-view gradient all-reduce (lgs_comm_*): one NCCL communicator per context / GPU
  ncclComm_t comm = nullptr;
  int32_t comm_world = 0, comm_rank = 0;
  int64_t comm_timeout_ms = 300000;  // lgs_comm_set_timeout: host waits on a collective
  // capacity-speculative sparse exchange (lgs_allreduce_grads_sparse_async / _wait)
  int64_t sparse_cap = 0;          // rows per rank of the record blocks (0: not learnt yet)
  uint32_t* sparse_ovf_dev = nullptr;   // [0] overflow flag, [1] largest row count
  uint32_t* sparse_ovf_host = nullptr;  // pinned copy
  cudaEvent_t sparse_done = nullptr;
  bool sparse_pending = false;
  // phase profiling
  bool profiling = false;
  std::vector<PhaseMark> marks;
  std::vector<cudaEvent_t> event_pool;
  double phase_ms[LGS_PHASE_COUNT] = {};
  int64_t phase_n[LGS_PHASE_COUNT] = {};
  // LGS_MEM_HOST_MAPPED renders: the last host-mapped map rendered (its SH pointer and size) and
  // how many of its Gaussians that render listed.  Zero-copy reads of the listed rows win when
  // few are listed (the headline: 2.5k of 500k); when many are (tiles that do not saturate on
  // layer A take the complete lists), scattered PCIe reads of [d][N] feature columns lose to one
  // DMA of the SH and feature blocks, so the next render of that map copies them in bulk.
  uint32_t* mh_listed_dev = nullptr;
  uint32_t* mh_listed_host = nullptr;  // mapped pinned: the count of the render whose copy is pending
  uint32_t* mh_listed_hdev = nullptr;  // its device address
  cudaEvent_t mh_event = nullptr;      // recorded after that copy
  bool mh_pending = false;
  const void* mh_pending_key = nullptr;  // its map (SH pointer) and size
  int64_t mh_pending_n = 0;
  const void* mh_key = nullptr;  // the last map whose count has landed, and that count
  int64_t mh_n = 0, mh_listed = 0;
  // Layer-A size of the depth-layered binning (~P / layer_div pairs, <= n / (2 layer_div)
  // Gaussians).  Adapted between uncaptured renders from the previous one's counters (lp_*):
  // when more than a quarter of the tiles needed the second pass, layer A doubles (and that size
  // is remembered as too small); when almost every tile saturated having consumed less than 1/16
  // of its list, it shrinks 4x (a dense view whose near splats cover most tiles).  Plans capture
  // with the size their warm-up renders settle on.
  uint32_t layer_div = kLayerDiv;
  // when more than 1/20 of the tiles needed the second pass and the view has at most 16M pairs,
  // one pass over complete lists is cheaper than two (configs[1]: +21%).  Kept for maps of the same
  // size and the same image size while the pair capacity stays within 2x of the one it was taken
  // at (then the counters of a layered render decide again).
  bool single_pass = false;
  int64_t sp_cap = 0;
  uint64_t sp_map = 0;
  int sp_ntiles = 0;
  uint64_t lp_map = 0;  // the map size the pending layer counters were taken on
  uint32_t layer_bad = UINT32_MAX;  // a div at which too many tiles were left unsaturated
  uint32_t* lp_dev = nullptr;       // [0] consumed (the host copy: + [1] layer-A listed pairs, [2] unfinished tiles)
  uint32_t* lp_host = nullptr;      // mapped pinned copy (written by launch_publish_counters)
  uint32_t* lp_hdev = nullptr;      // its device address
  cudaEvent_t lp_ev = nullptr;
  bool lp_pending = false;
  int lp_ntiles = 0;
  uint32_t lp_div = 0;  // the div the pending counts were taken at
  // the last counts the policy read: unfinished tiles at (ntiles, div) -- a plan captured right
  // after a render that saturated every tile leaves pass 2 out (speculative plan, lgs_plan_sync)
  uint64_t lp_last_unfinished = UINT64_MAX;
  int lp_last_ntiles = 0;
  uint32_t lp_last_div = 0;
  uint32_t* cap_unfinished_any = nullptr;  // speculative plan capture: pass 1 only, reports here
  uint32_t* cap_miss = nullptr;            // ... and here (device word the chain reads)
  // last lgs_find_language_redundant: candidates (a similar neighbour inside tau_dist), rounds
  int64_t prune_candidates = 0, prune_rounds = 0;
};

namespace {

// No C++ exception crosses the ABI: allocation failures of host containers become LGS_ENOMEM.
template <class F>
lgs_status guarded(F&& f) {
  try {
    return f();
  } catch (const std::bad_alloc&) {
    return fail(LGS_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(LGS_EIO, "%s", e.what());
  }
}

// Conditional graph nodes inside a plan capture (CUDA 12.4+): cond_create makes the handle a
// kernel sets with cudaGraphSetConditional, cond_begin adds an IF node after everything captured so
// far and redirects the context's launches into its body graph, cond_end returns to the parent.
lgs_status cond_create(lgs_ctx* ctx, cudaGraphConditionalHandle* h) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g = nullptr;
  LGS_CUDA(cudaStreamGetCaptureInfo(ctx->stream, &st, nullptr, &g, nullptr, nullptr));
  if (st != cudaStreamCaptureStatusActive || !g) return fail(LGS_EINVAL, "conditional node outside a capture");
  LGS_CUDA(cudaGraphConditionalHandleCreate(h, g, 0, cudaGraphCondAssignDefault));
  return LGS_OK;
}

lgs_status cond_begin(lgs_ctx* ctx, cudaGraphConditionalHandle h) {
  cudaStreamCaptureStatus st;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  LGS_CUDA(cudaStreamGetCaptureInfo(ctx->stream, &st, nullptr, &g, &deps, &ndeps));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  LGS_CUDA(cudaGraphAddNode(&node, g, deps, ndeps, &cp));
  LGS_CUDA(cudaStreamUpdateCaptureDependencies(ctx->stream, &node, 1, cudaStreamSetCaptureDependencies));
  if (!ctx->cond_stream) LGS_CUDA(cudaStreamCreateWithFlags(&ctx->cond_stream, cudaStreamNonBlocking));
  LGS_CUDA(cudaStreamBeginCaptureToGraph(ctx->cond_stream, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal));
  ctx->cond_parent = ctx->stream;
  ctx->stream = ctx->cond_stream;
  return LGS_OK;
}

lgs_status cond_end(lgs_ctx* ctx) {
  cudaGraph_t body = nullptr;
  ctx->stream = ctx->cond_parent;
  ctx->cond_parent = nullptr;
  LGS_CUDA(cudaStreamEndCapture(ctx->cond_stream, &body));
  return LGS_OK;
}

// RAII phase marker: records an event pair around a phase when profiling is on.
struct PhaseScope {
  lgs_ctx* ctx;
  PhaseMark m{};
  bool on;
  cudaEvent_t take() {
    if (!ctx->event_pool.empty()) {
      cudaEvent_t e = ctx->event_pool.back();
      ctx->event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  bool graph = false;  // inside a plan capture: external event-record nodes of the graph
  cudaStream_t st;
  PhaseScope(lgs_ctx* c, int phase, cudaStream_t on_stream = nullptr)
      : ctx(c), on(c->profiling && !c->capturing),
        graph(c->capturing && c->capture_marks && !c->cond_parent), st(on_stream ? on_stream : c->stream) {
    if (!on && !graph) return;
    m.phase = phase;
    if (graph) {
      cudaEventCreate(&m.a);
      cudaEventCreate(&m.b);
      cudaEventRecordWithFlags(m.a, st, cudaEventRecordExternal);
      return;
    }
    m.a = take();
    m.b = take();
    cudaEventRecord(m.a, st);
  }
  ~PhaseScope() {
    if (graph) {
      cudaEventRecordWithFlags(m.b, st, cudaEventRecordExternal);
      ctx->capture_marks->push_back(m);
      return;
    }
    if (!on) return;
    cudaEventRecord(m.b, st);
    ctx->marks.push_back(m);
  }
};

enum { PH_PREPROCESS = 0, PH_DEPTH_SORT, PH_DUPLICATE, PH_TILE_SORT, PH_BLEND_FWD, PH_BLEND_BWD, PH_PREPROCESS_BWD,
       PH_UPLOAD, PH_LOSS, PH_ADAM, PH_ALLREDUCE, PH_COVERAGE, PH_GRAD_ZERO };

}  // namespace

struct lgs_map {
  lgs_ctx* ctx = nullptr;
  DevMap dm{};
  float4* pos_opa = nullptr;
  float4* rot = nullptr;
  float4* scale = nullptr;
  float* sh = nullptr;
  float* feat = nullptr;
  bool mapped = false;             // LGS_MEM_HOST_MAPPED: dm.sh and feat_src point into page-locked host memory
  const float* feat_src = nullptr;  // [d][N], device-addressable (features gathered lazily)
  uint64_t version = 0;  // live-map registry key: a new one after lgs_prune (tapes / plans check it)
};

struct lgs_adam {
  lgs_ctx* ctx = nullptr;
  int64_t n = 0;
  int d = 0, dp = 0, K = 1;
  lgs_adam_config cfg{};
  int64_t step = 0;
  // first / second moments in the map's packed layout
  float4 *m_po = nullptr, *m_rot = nullptr, *m_sc = nullptr, *v_po = nullptr, *v_rot = nullptr, *v_sc = nullptr;
  float *m_sh = nullptr, *v_sh = nullptr, *m_ft = nullptr, *v_ft = nullptr;
};

struct lgs_saved {
  lgs_ctx* ctx = nullptr;
  lgs_map* owned_map = nullptr;  // lgs_render convenience path
  uint64_t map_version = 0;      // the map's version at render time (its buffers are the tape's dm)
  float* sh_dev = nullptr;       // host-mapped map rendered in bulk-copy mode: its SH block (dm.sh)
  bool host_rows_in_place = false;  // host-mapped map, zero-copy mode: listed rows were read over PCIe
  DevMap dm{};
  DevCam cam{};
  ViewBufs vb{};
  uint16_t* keys = nullptr;  // sorted tile ids
  uint32_t* vals = nullptr;  // sorted map indices
  uint2* ranges = nullptr;
  uint32_t* order = nullptr;  // tiles by decreasing list length
  int* counter = nullptr;     // persistent-scheduler slot counter
  PixelState ps{};
  float* cot = nullptr;     // loss cotangents [H][W][4 + DP] (fused L1 or lgs_mapping_loss)
  double* loss = nullptr;
  double* loss_sums = nullptr;  // lgs_mapping_loss partial sums [LOSS_COUNT]
  int64_t pairs = 0;
  int64_t vals_count = 0;  // entries allocated in vals (the lists live at the ranges' offsets)
  bool lpt_order = true;    // `order` holds the longest-list-first tile order (else natural order)
  float* gacc = nullptr;    // fused-L1 step (blend_fused.cu): screen-space gradients of the forward
  bool bwd_fused = false;
  const uint32_t* miss = nullptr;  // speculative plan: nonzero -> the chain writes nothing
  int ntiles = 0;
};

namespace {

void ctx_release(lgs_ctx* ctx) {
  if (ctx->refs.fetch_sub(1) == 1) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->comm) {
      if (const NcclApi* nc = nccl_api(nullptr)) nc->CommDestroy(ctx->comm);
    }
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    if (ctx->cond_stream) cudaStreamDestroy(ctx->cond_stream);
    if (ctx->side_stream) cudaStreamDestroy(ctx->side_stream);
    if (ctx->side_fork) cudaEventDestroy(ctx->side_fork);
    if (ctx->side_join) cudaEventDestroy(ctx->side_join);
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
    if (ctx->big_pool) cudaMemPoolDestroy(ctx->big_pool);
    if (ctx->host_u32) cudaFreeHost(ctx->host_u32);
    if (ctx->mh_listed_host) cudaFreeHost(ctx->mh_listed_host);
    if (ctx->mh_listed_dev) cudaFree(ctx->mh_listed_dev);
    if (ctx->delta_stage) cudaFreeHost(ctx->delta_stage);
    if (ctx->mh_event) cudaEventDestroy(ctx->mh_event);
    if (ctx->lp_host) cudaFreeHost(ctx->lp_host);
    if (ctx->lp_dev) cudaFree(ctx->lp_dev);
    if (ctx->lp_ev) cudaEventDestroy(ctx->lp_ev);
    if (ctx->dev_u32) cudaFree(ctx->dev_u32);
    if (ctx->pairs_ready) cudaEventDestroy(ctx->pairs_ready);
    if (ctx->sparse_ovf_dev) cudaFree(ctx->sparse_ovf_dev);
    if (ctx->sparse_ovf_host) cudaFreeHost(ctx->sparse_ovf_host);
    if (ctx->sparse_done) cudaEventDestroy(ctx->sparse_done);
    for (auto& m : ctx->marks) {
      cudaEventDestroy(m.a);
      cudaEventDestroy(m.b);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    delete ctx;
  }
}

constexpr size_t kBigBlock = size_t(256) << 20;

template <typename T>
lgs_status dalloc(lgs_ctx* ctx, T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  if (ctx->capturing)  // captured into a graph memory node (graph-owned memory)
    LGS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(T) * count, ctx->stream));
  else
    LGS_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), sizeof(T) * count,
                                     sizeof(T) * count >= kBigBlock ? ctx->big_pool : ctx->pool, ctx->stream));
  return LGS_OK;
}

template <typename T>
void dfree(lgs_ctx* ctx, T*& p) {
  if (p) cudaFreeAsync(p, ctx->stream);
  p = nullptr;
}

// Camera setup: same double formula as oracle/lgs_oracle.c camera_setup (geometry.hpp:23 Pose
// normalizes q; geometry.cpp:15-20 inverse), then rounded to float.
void quat_to_rot(double w, double x, double y, double z, double r[9]) {
  const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  r[0] = 1 - (tyy + tzz); r[1] = txy - twz;       r[2] = txz + twy;
  r[3] = txy + twz;       r[4] = 1 - (txx + tzz); r[5] = tyz - twx;
  r[6] = txz - twy;       r[7] = tyz + twx;       r[8] = 1 - (txx + tyy);
}

lgs_status make_devcam(const lgs_camera* cam, const lgs_render_config* cfg, DevCam* out) {
  if (!cam) return fail(LGS_EINVAL, "camera is NULL");
  if (cam->width <= 0 || cam->height <= 0 || cam->width > 65535 || cam->height > 65535)
    return fail(LGS_EINVAL, "image size %dx%d out of range [1, 65535]", cam->width, cam->height);
  if (!(cam->fx > 0.0) || !(cam->fy > 0.0)) return fail(LGS_EINVAL, "focal lengths must be positive");
  if (!(cfg->near_plane >= 0.0)) return fail(LGS_EINVAL, "near_plane must be >= 0 (depth keys are f32 bits)");
  double w = cam->q[0], x = cam->q[1], y = cam->q[2], z = cam->q[3];
  const double nrm = std::sqrt(w * w + x * x + y * y + z * z);
  if (!(nrm > 0.0)) return fail(LGS_EINVAL, "camera quaternion has zero norm");
  w /= nrm; x /= nrm; y /= nrm; z /= nrm;
  double rcw[9];
  quat_to_rot(w, -x, -y, -z, rcw);
  for (int i = 0; i < 9; ++i) {
    out->rcw[i] = (float)rcw[i];
    out->rcw_d[i] = rcw[i];
  }
  for (int i = 0; i < 3; ++i) {
    const double tcw = -(rcw[i * 3 + 0] * cam->t[0] + rcw[i * 3 + 1] * cam->t[1] + rcw[i * 3 + 2] * cam->t[2]);
    out->tcw[i] = (float)tcw;
    out->cc[i] = (float)cam->t[i];
    out->tcw_d[i] = tcw;
    out->cc_d[i] = cam->t[i];
  }
  out->fx = (float)cam->fx; out->fy = (float)cam->fy;
  out->fx_d = cam->fx; out->fy_d = cam->fy;
  out->cx = (float)cam->cx; out->cy = (float)cam->cy;
  out->W = cam->width; out->H = cam->height;
  out->tiles_x = (cam->width + kTile - 1) / kTile;
  out->tiles_y = (cam->height + kTile - 1) / kTile;
  if (out->tiles_x * out->tiles_y > 65536) return fail(LGS_EINVAL, "more than 65536 tiles");
  out->near_plane = (float)cfg->near_plane;
  out->dilation = (float)cfg->dilation;
  out->radius_sigma = (float)cfg->radius_sigma;
  out->alpha_clamp = (float)cfg->alpha_clamp;
  out->alpha_skip = (float)cfg->alpha_skip;
  out->t_min = (float)cfg->transmittance_min;
  return LGS_OK;
}

lgs_status copy_in(lgs_ctx* ctx, void* dst, const void* src, size_t bytes, int memory) {
  if (bytes == 0) return LGS_OK;
  if (memory == LGS_MEM_HOST) ctx->bytes_h2d += (int64_t)bytes;
  LGS_CUDA(cudaMemcpyAsync(dst, src, bytes, memory == LGS_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                           ctx->stream));
  return LGS_OK;
}

// device address of page-locked host memory (LGS_MEM_HOST_MAPPED), or an error
lgs_status mapped_ptr(const float* p, const float** dev, const char* what) {
  *dev = nullptr;
  if (!p) return LGS_OK;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess || a.type != cudaMemoryTypeHost || !a.devicePointer) {
    cudaGetLastError();
    return fail(LGS_EINVAL, "LGS_MEM_HOST_MAPPED: %s is not page-locked host memory", what);
  }
  *dev = static_cast<const float*>(a.devicePointer);
  return LGS_OK;
}

lgs_status map_upload(lgs_ctx* ctx, lgs_map* m, const lgs_gaussians* src) {
  const int64_t n = m->dm.n;
  const int d = m->dm.d, K = m->dm.K;
  const bool mapped = src->memory == LGS_MEM_HOST_MAPPED;
  const int mem = mapped ? LGS_MEM_HOST : src->memory;
  if (mapped) {  // read in place: the SH rows of the listed Gaussians, their features gathered lazily
    LGS_TRY(mapped_ptr(src->sh, &m->dm.sh, "sh"));
    LGS_TRY(mapped_ptr(d > 0 ? src->features : nullptr, &m->feat_src, "features"));
  } else {  // the SH block has the same layout on both sides
    LGS_TRY(copy_in(ctx, m->sh, src->sh, sizeof(float) * (size_t)n * K * 3, src->memory));
  }
  const float *pos = src->positions, *rot = src->rotations, *ls = src->log_scales, *op = src->opacity_logits,
              *ft = mapped ? nullptr : src->features;
  float* stage = nullptr;
  if (mem == LGS_MEM_HOST) {
    const size_t tot = (size_t)n * (3 + 4 + 3 + 1 + (mapped ? 0 : d));
    LGS_TRY(dalloc(ctx, &stage, tot));
    float* p = stage;
    LGS_TRY(copy_in(ctx, p, src->positions, sizeof(float) * n * 3, LGS_MEM_HOST)); pos = p; p += n * 3;
    LGS_TRY(copy_in(ctx, p, src->rotations, sizeof(float) * n * 4, LGS_MEM_HOST)); rot = p; p += n * 4;
    LGS_TRY(copy_in(ctx, p, src->log_scales, sizeof(float) * n * 3, LGS_MEM_HOST)); ls = p; p += n * 3;
    LGS_TRY(copy_in(ctx, p, src->opacity_logits, sizeof(float) * n, LGS_MEM_HOST)); op = p; p += n;
    if (d > 0 && !mapped) { LGS_TRY(copy_in(ctx, p, src->features, sizeof(float) * n * d, LGS_MEM_HOST)); ft = p; }
  }
  {
    PhaseScope ph(ctx, PH_UPLOAD);
    launch_pack_map(pos, rot, ls, op, ft, n, d, m->dm.dp, m->pos_opa, m->rot, m->scale, m->feat, ctx->stream);
  }
  ctx->launches++;
  if (stage) dfree(ctx, stage);
  LGS_CUDA(cudaGetLastError());
  return LGS_OK;
}

lgs_status check_gaussians(const lgs_gaussians* src) {
  if (!src) return fail(LGS_EINVAL, "gaussians is NULL");
  if (src->n < 0 || src->n > 0x7fffffffLL) return fail(LGS_EINVAL, "n out of range");
  if (src->feature_dim < 0 || src->feature_dim > LGS_MAX_FEATURE_DIM)
    return fail(LGS_EINVAL, "feature_dim %d out of range [0, %d]", src->feature_dim, LGS_MAX_FEATURE_DIM);
  if (src->sh_degree < 0 || src->sh_degree > LGS_MAX_SH_DEGREE)
    return fail(LGS_EINVAL, "sh_degree %d out of range [0, 3]", src->sh_degree);
  if (src->n > 0 && (!src->positions || !src->rotations || !src->log_scales || !src->opacity_logits || !src->sh ||
                     (src->feature_dim > 0 && !src->features)))
    return fail(LGS_EINVAL, "a map attribute pointer is NULL");
  if (src->memory != LGS_MEM_HOST && src->memory != LGS_MEM_DEVICE && src->memory != LGS_MEM_HOST_MAPPED)
    return fail(LGS_EINVAL, "bad memory kind");
  return LGS_OK;
}

// Registry of live map versions: a tape or plan holds raw pointers into its map's buffers, which
// lgs_prune replaces and lgs_map_destroy frees; both drop the version, and the backward / plan
// entry points refuse a stale one instead of reading freed memory.
std::mutex g_version_mu;
std::unordered_set<uint64_t>& live_versions() {
  static auto* s = new std::unordered_set<uint64_t>();
  return *s;
}
uint64_t g_next_version = 0;
uint64_t version_new() {
  std::lock_guard<std::mutex> lock(g_version_mu);
  const uint64_t v = ++g_next_version;
  live_versions().insert(v);
  return v;
}
void version_drop(uint64_t v) {
  std::lock_guard<std::mutex> lock(g_version_mu);
  live_versions().erase(v);
}
bool version_live(uint64_t v) {
  std::lock_guard<std::mutex> lock(g_version_mu);
  return live_versions().count(v) != 0;
}

void free_map(lgs_map* m) {
  lgs_ctx* ctx = m->ctx;
  version_drop(m->version);
  cudaSetDevice(ctx->device);
  dfree(ctx, m->pos_opa);
  dfree(ctx, m->rot);
  dfree(ctx, m->scale);
  dfree(ctx, m->sh);
  dfree(ctx, m->feat);
  delete m;
  ctx_release(ctx);
}

void free_saved(lgs_saved* t) {
  lgs_ctx* ctx = t->ctx;
  cudaSetDevice(ctx->device);
  dfree(ctx, t->sh_dev);
  dfree(ctx, t->vb.rec0);
  dfree(ctx, t->vb.active);
  dfree(ctx, t->gacc);
  dfree(ctx, t->vb.rec1);
  dfree(ctx, t->vb.rect);
  dfree(ctx, t->vb.color);
  dfree(ctx, t->vb.tiles);
  dfree(ctx, t->vb.dkey);
  dfree(ctx, t->vb.iota);
  dfree(ctx, t->keys);
  dfree(ctx, t->vals);
  dfree(ctx, t->ranges);
  dfree(ctx, t->order);
  dfree(ctx, t->counter);
  dfree(ctx, t->ps.final_t);
  dfree(ctx, t->ps.n_contrib);
  dfree(ctx, t->ps.depth);
  dfree(ctx, t->ps.acc);
  dfree(ctx, t->ps.work);
  dfree(ctx, t->cot);
  dfree(ctx, t->loss);
  dfree(ctx, t->loss_sums);
  if (t->owned_map) free_map(t->owned_map);
  delete t;
  ctx_release(ctx);
}

struct DeviceImages {  // device views of caller images (staged when they are host memory)
  float *rgb = nullptr, *depth = nullptr, *feat = nullptr, *acc = nullptr;
  bool staged = false;
};

}  // namespace

// ===========================================================================================
extern "C" {

LGS_API const char* lgs_version(void) { return "lgs 0.1.0 (sm_100a)"; }

LGS_API const char* lgs_last_error(void) { return g_last_error.c_str(); }

LGS_API lgs_render_config lgs_render_config_default(void) {
  lgs_render_config c;
  c.near_plane = 0.01;
  c.dilation = 0.3;
  c.alpha_clamp = 0.99;
  c.alpha_skip = 1.0 / 255.0;
  c.transmittance_min = 1e-4;
  c.radius_sigma = 3.0;
  return c;
}

LGS_API lgs_status lgs_ctx_create(int32_t device, void* stream, lgs_ctx** out) {
  if (!out) return fail(LGS_EINVAL, "out is NULL");
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return fail(LGS_ENODEV, "no CUDA device");
  if (device < 0 || device >= count) return fail(LGS_EINVAL, "device %d out of range", device);
  cudaDeviceProp prop;
  LGS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(LGS_ENODEV, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major,
                                    prop.minor);
  LGS_CUDA(cudaSetDevice(device));
  lgs_ctx* ctx = new lgs_ctx();
  ctx->device = device;
  if (stream) {
    ctx->stream = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete ctx;
      return fail(LGS_ECUDA, "cudaStreamCreate failed");
    }
    ctx->own_stream = true;
  }
  // A private pool per context: blocks freed on this context's stream are reused only by it, so
  // contexts rendering concurrently on different streams never acquire each other's frees (the
  // shared default pool would insert cross-stream waits and serialize them).  Release threshold
  // raised: steady-state iterations reuse blocks without new cudaMalloc calls.
  {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    if (cudaMemPoolCreate(&ctx->pool, &props) != cudaSuccess) {
      if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
      delete ctx;
      return fail(LGS_ENOMEM, "cudaMemPoolCreate failed");
    }
    if (cudaMemPoolCreate(&ctx->big_pool, &props) != cudaSuccess) {
      cudaMemPoolDestroy(ctx->pool);
      if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
      delete ctx;
      return fail(LGS_ENOMEM, "cudaMemPoolCreate failed");
    }
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &thr);
    cudaMemPoolSetAttribute(ctx->big_pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (cudaMallocHost(&ctx->host_u32, 64) != cudaSuccess || cudaMalloc(&ctx->dev_u32, 64) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->pairs_ready, cudaEventDisableTiming) != cudaSuccess) {
    ctx_release(ctx);
    return fail(LGS_ENOMEM, "context allocation failed");
  }
  *out = ctx;
  return LGS_OK;
}

LGS_API lgs_status lgs_ctx_set_full_tile_lists(lgs_ctx* ctx, int32_t full) {
  if (!ctx) return fail(LGS_EINVAL, "ctx is NULL");
  ctx->full_lists = full != 0;
  return LGS_OK;
}

LGS_API lgs_status lgs_ctx_set_option(lgs_ctx* ctx, int32_t option, int64_t value) {
  if (!ctx) return fail(LGS_EINVAL, "ctx is NULL");
  switch (option) {
    case LGS_OPT_FULL_TILE_LISTS: ctx->full_lists = value != 0; return LGS_OK;
    case LGS_OPT_RADIX_DEPTH_ORDER: ctx->radix_depth = value != 0; return LGS_OK;
    case LGS_OPT_FUSED_EAGER: ctx->fused_eager = value != 0; return LGS_OK;
    case LGS_OPT_SPECULATIVE_PLANS: ctx->no_speculative = value == 0; return LGS_OK;
    case LGS_OPT_HOST_GRAD_DELTA:
      ctx->host_grad_delta = value != 0;
      ctx->delta_n = -1;  // the next backward writes densely
      ctx->delta_rows.clear();
      return LGS_OK;
    default: return fail(LGS_EINVAL, "unknown context option");
  }
}

LGS_API lgs_status lgs_ctx_transfer_bytes(const lgs_ctx* ctx, int64_t* h2d, int64_t* d2h) {
  if (!ctx) return fail(LGS_EINVAL, "ctx is NULL");
  if (h2d) *h2d = ctx->bytes_h2d.load();
  if (d2h) *d2h = ctx->bytes_d2h.load();
  return LGS_OK;
}

LGS_API lgs_status lgs_ctx_destroy(lgs_ctx* ctx) {
  if (!ctx) return LGS_OK;
  ctx_release(ctx);
  return LGS_OK;
}

LGS_API lgs_status lgs_ctx_set_stream(lgs_ctx* ctx, void* stream) {
  if (!ctx) return fail(LGS_EINVAL, "ctx is NULL");
  cudaSetDevice(ctx->device);
  if (ctx->own_stream) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
    ctx->own_stream = false;
  }
  ctx->stream = (cudaStream_t)stream;
  return LGS_OK;
}

LGS_API lgs_status lgs_ctx_synchronize(lgs_ctx* ctx) {
  if (!ctx) return fail(LGS_EINVAL, "ctx is NULL");
  LGS_CUDA(cudaSetDevice(ctx->device));
  LGS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LGS_OK;
}

LGS_API int64_t lgs_ctx_launch_count(const lgs_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

LGS_API int32_t lgs_ctx_layer_div(const lgs_ctx* ctx) { return ctx ? (int32_t)ctx->layer_div : -1; }

LGS_API lgs_status lgs_map_create(lgs_ctx* ctx, const lgs_gaussians* src, lgs_map** out) {
  if (!ctx || !out) return fail(LGS_EINVAL, "ctx/out is NULL");
  *out = nullptr;
  LGS_TRY(check_gaussians(src));
  LGS_CUDA(cudaSetDevice(ctx->device));
  lgs_map* m = new lgs_map();
  m->ctx = ctx;
  ctx->refs++;
  m->dm.n = src->n;
  m->dm.d = src->feature_dim;
  m->dm.dp = pad_dim(src->feature_dim);
  m->dm.deg = src->sh_degree;
  m->dm.K = (src->sh_degree + 1) * (src->sh_degree + 1);
  const size_t n = (size_t)src->n;
  m->mapped = src->memory == LGS_MEM_HOST_MAPPED;
  lgs_status st = LGS_OK;
  if ((st = dalloc(ctx, &m->pos_opa, n)) != LGS_OK || (st = dalloc(ctx, &m->rot, n)) != LGS_OK ||
      (st = dalloc(ctx, &m->scale, n)) != LGS_OK ||
      (!m->mapped && (st = dalloc(ctx, &m->sh, n * m->dm.K * 3)) != LGS_OK) ||
      (st = dalloc(ctx, &m->feat, n * (m->dm.dp > 0 ? m->dm.dp : 1))) != LGS_OK ||
      (st = map_upload(ctx, m, src)) != LGS_OK) {
    free_map(m);
    return st;
  }
  m->dm.pos_opa = m->pos_opa;
  m->dm.rot = m->rot;
  m->dm.scale = m->scale;
  if (!m->mapped) m->dm.sh = m->sh;
  m->dm.feat = m->feat;
  m->version = version_new();
  if (src->memory == LGS_MEM_HOST) LGS_CUDA(cudaStreamSynchronize(ctx->stream));
  *out = m;
  return LGS_OK;
}

LGS_API lgs_status lgs_map_update(lgs_ctx* ctx, lgs_map* map, const lgs_gaussians* src) {
  if (!ctx || !map) return fail(LGS_EINVAL, "ctx/map is NULL");
  LGS_TRY(check_gaussians(src));
  if (src->n != map->dm.n || src->feature_dim != map->dm.d || src->sh_degree != map->dm.deg)
    return fail(LGS_EINVAL, "lgs_map_update: shape differs from the map");
  if (map->mapped != (src->memory == LGS_MEM_HOST_MAPPED))
    return fail(LGS_EINVAL, "lgs_map_update: a host-mapped map is updated from host-mapped memory only");
  LGS_CUDA(cudaSetDevice(ctx->device));
  LGS_TRY(map_upload(ctx, map, src));
  if (src->memory == LGS_MEM_HOST) LGS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LGS_OK;
}

LGS_API lgs_status lgs_map_destroy(lgs_map* map) {
  if (map) free_map(map);
  return LGS_OK;
}

LGS_API int64_t lgs_map_size(const lgs_map* map) { return map ? map->dm.n : -1; }

LGS_API int64_t lgs_grads_flat_size(int64_t n, int32_t feature_dim, int32_t sh_degree) {
  const int64_t K = (int64_t)(sh_degree + 1) * (sh_degree + 1);
  return n * (3 + 4 + 3 + 1 + 3 * K + feature_dim);
}

// -------------------------------------------------------------------------------------------
// forward
// -------------------------------------------------------------------------------------------
}  // extern "C"

namespace {
// Gaussians layer A may hold (the cut's second bound, with the pair cap of layer_a_cap)
int64_t layer_a_gauss_cap(int64_t n, uint32_t div) {
  return std::min<int64_t>(n, std::max<int64_t>(4096, n / (2 * (int64_t)div)));
}

// The layer-A size policy (lgs_ctx::layer_div): reads the counters of the previous uncaptured
// layered render once they have landed (never waits).
void layer_policy_update(lgs_ctx* ctx, int ntiles) {
  if (!ctx->lp_pending || cudaEventQuery(ctx->lp_ev) != cudaSuccess) return;
  ctx->lp_pending = false;
  if (ctx->lp_ntiles != ntiles || ctx->lp_div != ctx->layer_div) return;  // counts of another image / size
  const uint64_t consumed = ctx->lp_host[0], listed = ctx->lp_host[1], unfinished = ctx->lp_host[2];
  uint32_t& div = ctx->layer_div;
  ctx->lp_last_unfinished = unfinished;
  ctx->lp_last_ntiles = ntiles;
  ctx->lp_last_div = div;
  if (unfinished * 20 > (uint64_t)ntiles && div > kLayerDiv) {
    // a layer A shrunk for an earlier view: back towards the default size before judging the
    // layering (a context rendering several views would otherwise switch them all to one pass)
    ctx->layer_bad = std::min(ctx->layer_bad, div);
    div = std::max<uint32_t>(kLayerDiv, div / 4);
    return;
  }
  if (unfinished * 20 > (uint64_t)ntiles && ctx->pairs_cap < kSinglePassPairs) {
    ctx->single_pass = true;
    ctx->sp_cap = ctx->pairs_cap;
    ctx->sp_map = ctx->lp_map;
    ctx->sp_ntiles = ntiles;
  }
  if (unfinished * 4 > (uint64_t)ntiles) {
    ctx->layer_bad = std::min(ctx->layer_bad, div);
    div = std::max<uint32_t>(4, div / 2);
  } else if (unfinished * 50 < (uint64_t)ntiles && listed > 0 && consumed * 4 < listed && div < 1024 &&
             div * 4 < ctx->layer_bad) {
    div *= 4;  // warps consumed < 1/16 of their lists on average (4 warps per tile)
  }
}
}  // namespace

extern "C" {

LGS_API lgs_status lgs_render_forward(lgs_ctx* ctx, const lgs_map* map, const lgs_camera* cam,
                                      const lgs_render_config* cfg_in, const lgs_l1_targets* targets,
                                      lgs_images* out, lgs_saved** tape) {
  if (!ctx || !map) return fail(LGS_EINVAL, "ctx/map is NULL");
  if (tape) *tape = nullptr;
  const lgs_render_config cfg = cfg_in ? *cfg_in : lgs_render_config_default();
  DevCam dc;
  LGS_TRY(make_devcam(cam, &cfg, &dc));
  if (targets && (!targets->rgb || !targets->depth || (map->dm.d > 0 && !targets->feat)))
    return fail(LGS_EINVAL, "L1 targets: rgb/depth/feat must all be given");
  LGS_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const int64_t n = map->dm.n;
  const size_t npix = (size_t)dc.W * dc.H;
  const int ntiles = dc.tiles_x * dc.tiles_y;
  const int dp = map->dm.dp, d = map->dm.d;

  lgs_saved* t = new lgs_saved();
  t->ctx = ctx;
  ctx->refs++;
  t->dm = map->dm;
  t->map_version = map->version;
  t->cam = dc;
  t->ntiles = ntiles;
  auto bail = [&](lgs_status st) {
    free_saved(t);
    return st;
  };
#define TRYB(expr)                      \
  do {                                  \
    lgs_status s2_ = (expr);            \
    if (s2_ != LGS_OK) return bail(s2_); \
  } while (0)
#define CUDAB(call)                                                                                   \
  do {                                                                                                \
    cudaError_t e_ = (call);                                                                          \
    if (e_ != cudaSuccess)                                                                            \
      return bail(fail(e_ == cudaErrorMemoryAllocation ? LGS_ENOMEM : LGS_ECUDA, "%s: %s (%s:%d)", #call, \
                       cudaGetErrorString(e_), __FILE__, __LINE__));                                  \
  } while (0)

  TRYB(dalloc(ctx, &t->vb.rec0, n));
  TRYB(dalloc(ctx, &t->vb.rec1, n));
  TRYB(dalloc(ctx, &t->vb.rect, n));
  TRYB(dalloc(ctx, &t->vb.color, n));
  TRYB(dalloc(ctx, &t->vb.tiles, n));
  TRYB(dalloc(ctx, &t->vb.dkey, n));
  TRYB(dalloc(ctx, &t->vb.iota, n));
  TRYB(dalloc(ctx, &t->ranges, ntiles));
  TRYB(dalloc(ctx, &t->order, ntiles));
  TRYB(dalloc(ctx, &t->counter, 1));
  TRYB(dalloc(ctx, &t->ps.final_t, npix));
  TRYB(dalloc(ctx, &t->ps.n_contrib, npix));
  TRYB(dalloc(ctx, &t->ps.depth, npix));
  TRYB(dalloc(ctx, &t->ps.acc, npix));
  if (ctx->profiling) TRYB(dalloc(ctx, &t->ps.work, npix));  // work counters: profiling renders only

  // LGS_OPT_RADIX_DEPTH_ORDER selects the device radix sort (cross-check of depth_order.cu)
  const bool cub_depth = ctx->radix_depth;
  const bool fast = fast_binning_supported(ntiles);
  // depth-layered binning (binning_fast.cu, depth_order.cu): K1 fills the depth-bucket histogram,
  // the depth order of layer A is built with the binning below, the complete order only when some
  // tile needs the second pass
  // One pass over complete lists instead of the layering, decided from the earlier renders: a view
  // whose pairs all fit a few layer-A minimums (configs[0]: 43k; layer A would take nearly every
  // pair and the second pass most tiles), or a context whose layered renders left more than 1/20 of
  // the tiles to the second pass at up to 16M pairs (lgs_ctx::single_pass; configs[1]).
  if (ctx->single_pass && (ctx->sp_map != (uint64_t)map->dm.n || ctx->sp_ntiles != ntiles ||
                           ctx->pairs_cap > 2 * ctx->sp_cap || ctx->pairs_cap >= kSinglePassPairs))
    ctx->single_pass = false;  // another view: layered renders decide again
  const bool small_view =
      ctx->pairs_cap > 0 && (ctx->pairs_cap < 4 * (int64_t)kLayerMinPairs || ctx->single_pass);
  const bool layered = fast && !ctx->full_lists && n > 0 && !cub_depth && !small_view;
  if (layered && !ctx->capturing) layer_policy_update(ctx, ntiles);
  void* otemp = nullptr;
  const size_t otemp_bytes = cub_depth ? 0 : depth_order_temp_bytes(n);
  if (!cub_depth) TRYB(dalloc(ctx, reinterpret_cast<uint8_t**>(&otemp), otemp_bytes));
  // host-mapped map (LGS_MEM_HOST_MAPPED): the listed Gaussians' SH rows and features are read in
  // place (zero-copy), unless the previous render of this map listed more than 1/64 of it (or
  // every Gaussian may be listed: complete lists) -- then the SH and feature blocks are DMA-copied
  // in bulk for this render (ctx->mh_*).  Uncaptured renders only; plans keep zero-copy.
  const bool mapped = map->mapped && !ctx->capturing;
  bool bulk = false;
  if (mapped) {
    if (!ctx->mh_listed_dev) {
      CUDAB(cudaMalloc(reinterpret_cast<void**>(&ctx->mh_listed_dev), sizeof(uint32_t)));
      CUDAB(cudaHostAlloc(reinterpret_cast<void**>(&ctx->mh_listed_host), sizeof(uint32_t), cudaHostAllocMapped));
      CUDAB(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->mh_listed_hdev), ctx->mh_listed_host, 0));
      CUDAB(cudaEventCreateWithFlags(&ctx->mh_event, cudaEventDisableTiming));
    }
    if (ctx->mh_pending && cudaEventQuery(ctx->mh_event) == cudaSuccess) {  // the last count has landed
      ctx->mh_key = ctx->mh_pending_key;
      ctx->mh_n = ctx->mh_pending_n;
      ctx->mh_listed = *ctx->mh_listed_host;
      ctx->mh_pending = false;
    }
    bulk = !layered || (ctx->mh_key == map->dm.sh && ctx->mh_n == n && ctx->mh_listed > n / 64);
    if (!ctx->mh_pending) CUDAB(cudaMemsetAsync(ctx->mh_listed_dev, 0, sizeof(uint32_t), s));
  }
  t->host_rows_in_place = mapped && !bulk;
  if (bulk) {
    const size_t shn = (size_t)n * map->dm.K * 3;
    TRYB(dalloc(ctx, &t->sh_dev, shn));
    CUDAB(cudaMemcpyAsync(t->sh_dev, map->dm.sh, sizeof(float) * shn, cudaMemcpyDefault, s));
    ctx->bytes_h2d += (int64_t)(sizeof(float) * shn);
    t->dm.sh = t->sh_dev;
    if (d > 0 && map->feat_src) {  // [d][N] block by DMA, packed to [N][dp] on the device
      float* stage = nullptr;
      TRYB(dalloc(ctx, &stage, (size_t)n * d));
      CUDAB(cudaMemcpyAsync(stage, map->feat_src, sizeof(float) * (size_t)n * d, cudaMemcpyDefault, s));
      ctx->bytes_h2d += (int64_t)(sizeof(float) * (size_t)n * d);
      launch_gather_features(stage, map->feat, n, d, dp, s);
      ctx->launches++;
      dfree(ctx, stage);
    }
  }
  const DevMap& dm = t->dm;  // the map's buffers (SH from the bulk copy in bulk mode)
  ColorJob cj;  // layered: colours of just the listed Gaussians, computed where first listed
  if (layered) {
    cj.sh = dm.sh;
    cj.pos_opa = dm.pos_opa;
    for (int a = 0; a < 3; ++a) cj.cc[a] = dc.cc[a];
    cj.deg = dm.deg;
    cj.color = t->vb.color;
    if (mapped && !ctx->mh_pending) cj.listed = ctx->mh_listed_dev;  // count this render (one in flight)
    if (map->mapped && map->feat_src && !bulk) {
      cj.feat_src = map->feat_src;
      cj.feat_dst = map->feat;
      cj.n = n;
      cj.d = dm.d;
      cj.dp = dm.dp;
    }
  }
  if (map->mapped && map->feat_src && !layered && !bulk) {  // every Gaussian may be listed: gather all features
    launch_gather_features(map->feat_src, map->feat, n, dm.d, dm.dp, s);
    ctx->launches++;
  }
  if (layered) {
    launch_depth_prepare(n, dc.near_plane, otemp, &t->vb, s);
    TRYB(dalloc(ctx, &t->vb.active, n));  // tape-owned: the backward reads it
    CUDAB(cudaMemsetAsync(t->vb.active, 0, (size_t)n, s));
  }

  // K1
  const uint32_t* dev_pairs = ctx->dev_u32;
  // with a capacity known before K1 (bin_and_blend's first attempt below), the bucket scan also
  // applies the layer-A cut (no separate cut launch)
  const int64_t cut_cap = (layered && fast && n > 0 && ctx->pairs_cap > 0) ? ctx->pairs_cap : -1;
  const uint32_t cut_div = ctx->layer_div;
  {
    PhaseScope ph(ctx, PH_PREPROCESS);
    launch_preprocess(dm, dc, t->vb, !layered, s);
    // the pair count P = sum of tiles touched sizes the tile lists; it is read back while the GPU
    // is still busy with the depth order queued below, so the host wait never idles the GPU
    // P = visible buckets' pairs; with a known capacity the scan also cuts layer A
    if (layered && cut_cap >= 0) {
      const LayerCut lc{ctx->layer_div, kLayerMinPairs, (uint32_t)layer_a_cap(cut_cap, ntiles, ctx->layer_div),
                        layer_a_gauss_cap(n, ctx->layer_div)};
      launch_depth_scan(n, dc.near_plane, otemp, &lc, &dev_pairs, s);
    } else if (layered) {
      launch_depth_scan(n, dc.near_plane, otemp, nullptr, &dev_pairs, s);
    }
    else launch_sum_tiles(t->vb.tiles, n, ctx->dev_u32, s);
  }
  ctx->launches += 2;
  // side branch of a plan: the gradient buffers' zero rows stream out beside the forward (the
  // backward's chain then writes only the active rows).  Forked right before the first blend,
  // which is issue-bound and leaves HBM to the stores (forking after K1 instead, beside the
  // latency-bound depth order, measured 10-15 us slower per replay).
  // longest-first tile order of the first pass (plans only): with few tiles per CTA slot of the
  // blend (~2 at the headline) the longest tiles' CTAs run alone at the end in natural order.  The
  // tiles are ranked by their measured durations in the previous replay (the view is fixed between
  // replays; list lengths correlate only ~0.3 with them): +2% over ranking by list length.  With
  // many tiles per slot (c2, c4: 3225 tiles) the natural order is faster than either ranking -- it
  // keeps neighbouring tiles, which share most of their Gaussians, on the SMs together
  // (profiles/r2_ab_lpt.log, r2_ab_lpt_cost.log, r2_tile_schedule.md)
  const bool lpt = ctx->capturing && ctx->cap_lpt_cur && ctx->prezero && ntiles < 12 * device_sm_count();
  auto fork_prezero = [&]() -> lgs_status {
    if (!(layered && ctx->capturing && ctx->prezero && !ctx->prezero_forked && n > 0)) return LGS_OK;
    LGS_CUDA(cudaEventRecord(ctx->side_fork, s));
    LGS_CUDA(cudaStreamWaitEvent(ctx->side_stream, ctx->side_fork, 0));
    if (lpt) {  // this replay's order, for the next replay (copied after the join); first on the
                // branch, so its one CTA is resident before the blend fills the SMs
      launch_tile_order_lpt(t->ranges, ctx->cap_tile_cost, ntiles, ctx->cap_lpt_next, ctx->side_stream);
      ctx->lpt_forked = true;
      ctx->launches++;
    }
    {
      PhaseScope ph(ctx, PH_GRAD_ZERO, ctx->side_stream);
      launch_grad_zero(device_grad_out(ctx->prezero, map->dm.d), n, map->dm.K, map->dm.dp > 0 ? map->dm.d : 0,
                       ctx->side_stream);
    }
    LGS_CUDA(cudaEventRecord(ctx->side_join, ctx->side_stream));
    ctx->prezero_forked = true;
    ctx->launches++;
    return LGS_OK;
  };
  if (n > 0) {
    CUDAB(cudaMemcpyAsync(ctx->host_u32, dev_pairs, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    if (!ctx->capturing) CUDAB(cudaEventRecord(ctx->pairs_ready, s));
  }

  // depth sort + scan
  uint32_t *dkey_sorted = nullptr, *idx_sorted = nullptr, *incl = nullptr;
  void* temp = nullptr;
  const int tile_bits = bits_for(ntiles);
  size_t temp_bytes = binning_temp_bytes(n, 0, tile_bits);
  TRYB(dalloc(ctx, &dkey_sorted, n));
  TRYB(dalloc(ctx, &idx_sorted, n));
  TRYB(dalloc(ctx, &incl, n));
  TRYB(dalloc(ctx, reinterpret_cast<uint8_t**>(&temp), temp_bytes));
  if (!layered) {
    PhaseScope ph(ctx, PH_DEPTH_SORT);
    if (cub_depth) {
      launch_depth_sort(t->vb, n, dkey_sorted, idx_sorted, temp, temp_bytes, s);
      launch_scan_tiles(t->vb.tiles, idx_sorted, n, dkey_sorted, incl, temp, temp_bytes, s);
    } else {
      launch_depth_order(t->vb, n, dc.near_plane, otemp, otemp_bytes, idx_sorted, dkey_sorted, s);
      launch_scan_counts(dkey_sorted, n, incl, temp, temp_bytes, s);
    }
    ctx->launches += n > 0 ? (cub_depth ? 6 : 7) : 0;
  }

  // K5 (+ fused L1) buffers
  FwdOut fo{};
  DeviceImages di;
  const bool host_out = out && out->memory == LGS_MEM_HOST;
  if (out) {
    if (host_out) {
      if (out->rgb) TRYB(dalloc(ctx, &di.rgb, npix * 3));
      if (out->depth) TRYB(dalloc(ctx, &di.depth, npix));
      if (out->feat && d > 0) TRYB(dalloc(ctx, &di.feat, npix * d));
      if (out->acc) TRYB(dalloc(ctx, &di.acc, npix));
      di.staged = true;
    } else {
      di.rgb = out->rgb; di.depth = out->depth; di.feat = d > 0 ? out->feat : nullptr; di.acc = out->acc;
    }
  }
  fo.rgb = di.rgb; fo.depth = di.depth; fo.feat = di.feat; fo.acc = di.acc;
  float* tstage = nullptr;
  if (targets) {
    TRYB(dalloc(ctx, &t->cot, npix * (4 + dp)));
    TRYB(dalloc(ctx, &t->loss, 1));
    fo.t_rgb = targets->rgb; fo.t_depth = targets->depth; fo.t_feat = targets->feat;
    if (targets->memory == LGS_MEM_HOST) {
      TRYB(dalloc(ctx, &tstage, npix * (4 + d)));
      ctx->bytes_h2d += (int64_t)(sizeof(float) * npix * (4 + (size_t)(targets->feat ? d : 0)));
      CUDAB(cudaMemcpyAsync(tstage, targets->rgb, sizeof(float) * npix * 3, cudaMemcpyHostToDevice, s));
      CUDAB(cudaMemcpyAsync(tstage + npix * 3, targets->depth, sizeof(float) * npix, cudaMemcpyHostToDevice, s));
      if (d > 0)
        CUDAB(cudaMemcpyAsync(tstage + npix * 4, targets->feat, sizeof(float) * npix * d, cudaMemcpyHostToDevice, s));
      fo.t_rgb = tstage; fo.t_depth = tstage + npix * 3; fo.t_feat = tstage + npix * 4;
    }
    fo.cot = t->cot;
    fo.loss = t->loss;
  }

  // Binning + blend.  With a capacity from earlier renders on this context, everything is enqueued
  // without waiting for the pair count P: the binning reads P on the device, and the host checks it
  // (and an overflow flag) only after the whole forward is queued, when the GPU is far ahead of the
  // check.  P > capacity (or the first render) runs the binning again with buffers of exactly P.
  auto bin_and_blend = [&](int64_t cap, bool exact) -> lgs_status {
    if (!exact && !layered) {  // re-run with exact buffers: the tile counts in depth order again
      launch_scan_tiles(t->vb.tiles, idx_sorted, n, dkey_sorted, incl, temp, temp_bytes, s);
      ctx->launches += n > 0 ? 3 : 0;
    }
    dfree(ctx, t->vals);
    dfree(ctx, t->keys);
    if (layered) {
      // Depth-layered binning.  Pass 1: the depth order of layer A only (the nearest Gaussians
      // owning ~P / kLayerDiv pairs, depth_order.cu), their lists (one warp per tile compacting
      // the depth-ordered candidates) and the forward, which flags every tile it could not
      // saturate.  Those tiles get their complete lists (counting sort restricted to them, at
      // vals + capA) and are blended again: pass 2, a conditional node of a captured plan.
      const uint32_t ldiv = ctx->layer_div;
      const uint32_t capA = (uint32_t)layer_a_cap(cap, ntiles, ldiv);
      const int64_t gcapA = layer_a_gauss_cap(n, ldiv);
      const size_t sat_n = (size_t)(dc.tiles_x + 1) * (dc.tiles_y + 1);
      uint32_t *ra = nullptr, *unfinished = nullptr, *sat = nullptr, *order2 = nullptr, *count2 = nullptr;
      uint32_t* scratch_b = nullptr;
      uint2* cand_rect = nullptr;
      // a speculative plan (captured after a render that saturated every tile) has no pass 2: a
      // replay that leaves a tile unfinished says so through a mapped host word, and lgs_plan_sync
      // re-captures the plan with pass 2 and runs the step again
      uint32_t* const spec = ctx->capturing ? ctx->cap_unfinished_any : nullptr;
      LGS_TRY(dalloc(ctx, &t->vals, (size_t)capA + (spec ? 0 : (size_t)cap)));
      t->vals_count = (int64_t)capA + (spec ? 0 : cap);
      LGS_TRY(dalloc(ctx, &ra, 4 + (size_t)ntiles));  // [0] R_A, [1] list allocator, [4 ..] unfinished flags
      unfinished = ra + 4;
      LGS_TRY(dalloc(ctx, &cand_rect, gcapA));
      if (!spec) {
        LGS_TRY(dalloc(ctx, &sat, sat_n));
        LGS_TRY(dalloc(ctx, &order2, ntiles));
        LGS_TRY(dalloc(ctx, &count2, 2));  // [0] unfinished tiles, [1] pairs of the second pass
        LGS_TRY(dalloc(ctx, reinterpret_cast<uint8_t**>(&scratch_b), fast_binning_scratch_bytes(cap, n, ntiles)));
      }
      LGS_CUDA(cudaMemsetAsync(ra, 0, sizeof(uint32_t) * (4 + (size_t)ntiles), s));
      // captured fused-L1 step: each tile's backward runs right after its forward (blend_fused.cu);
      // the depth order flags the layer-A Gaussians active and zeroes their accumulator rows
      // (LGS_OPT_FUSED_EAGER: the same in uncaptured renders, for profilers that cannot see inside
      // graphs -- the tape then holds the L1 gradients, and a backward with other cotangents is
      // rejected with LGS_EINVAL)
      const bool fuse = (ctx->capturing || ctx->fused_eager) && targets && blend_fused_supported(dp) &&
                        slots_for(dp) == 32;
      if (fuse) {
        dfree(ctx, t->gacc);
        LGS_TRY(dalloc(ctx, &t->gacc, (size_t)n * 32));
        t->bwd_fused = true;
      }
      {
        PhaseScope ph(ctx, PH_DEPTH_SORT);
        launch_depth_order_layer_a(t->vb, n, dc.near_plane, otemp, ldiv, kLayerMinPairs, gcapA, capA,
                                   idx_sorted, cand_rect, ra, t->vb.active, fuse ? t->gacc : nullptr, !exact,
                                   exact && cap == cut_cap && ldiv == cut_div, cj, s);
      }
      {
        PhaseScope ph(ctx, PH_TILE_SORT);
        // (the fused kernel follows directly: the list kernel zeroes its tile counter and the loss)
        launch_layer_tile_lists(cand_rect, idx_sorted, ra, dc.tiles_x, ntiles, ra + 1, t->vals, t->ranges,
                                fuse ? t->counter : nullptr, fuse && targets ? t->loss : nullptr,
                                spec ? ctx->cap_miss : nullptr, s);
      }
      // Layered lists are short and even (every tile stops at its saturation): the blend kernels
      // take tiles in natural order (measured as fast as longest-list-first, one launch less).
      t->lpt_order = false;
      ctx->launches += (exact && cap == cut_cap && ldiv == cut_div) ? 4 : 5;  // (the rank kernel sorts big buckets)
      if (targets && !fuse) LGS_CUDA(cudaMemsetAsync(t->loss, 0, sizeof(double), s));
      FwdOut fo1 = fo;
      fo1.unfinished = unfinished;
      fo1.tile_cost = lpt && fuse ? ctx->cap_tile_cost : nullptr;
      fo1.unfinished_any = spec;
      fo1.miss = spec ? ctx->cap_miss : nullptr;
      t->miss = fo1.miss;
      const bool policy = !ctx->capturing && !ctx->lp_pending;  // count this render for the layer-A policy
      if (policy) {
        if (!ctx->lp_dev) {
          LGS_CUDA(cudaMalloc(reinterpret_cast<void**>(&ctx->lp_dev), 4 * sizeof(uint32_t)));
          LGS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->lp_host), 4 * sizeof(uint32_t), cudaHostAllocMapped));
          LGS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ctx->lp_hdev), ctx->lp_host, 0));
          LGS_CUDA(cudaEventCreateWithFlags(&ctx->lp_ev, cudaEventDisableTiming));
        }
        LGS_CUDA(cudaMemsetAsync(ctx->lp_dev, 0, sizeof(uint32_t), s));
        fo1.consumed = ctx->lp_dev;
      }
      TRYB(fork_prezero());
      {
        PhaseScope ph(ctx, PH_BLEND_FWD);
        if (fuse)
          launch_blend_fused_l1(dm, dc, t->vb, TileLists{t->vals, t->ranges, lpt ? ctx->cap_lpt_cur : nullptr, t->counter},
                                fo1, t->gacc, s, true, ntiles < 2 * device_sm_count());  // few tiles: latency-bound variant
        else
          launch_blend_fwd(dm, dc, t->vb, TileLists{t->vals, t->ranges, nullptr, t->counter}, t->ps, fo1, s);
      }
      ctx->launches++;
      if (spec) {
        dfree(ctx, cand_rect);
        dfree(ctx, ra);
        LGS_CUDA(cudaGetLastError());
        return LGS_OK;
      }
      // pass 2, inside a captured plan as the body of a conditional node (skipped when every tile
      // saturated); eagerly its kernels find no unfinished tile and return at once
      cudaGraphConditionalHandle cond{};
      const bool use_cond = ctx->capturing;
      if (use_cond) LGS_TRY(cond_create(ctx, &cond));
      {
        PhaseScope ph(ctx, PH_TILE_SORT);
        launch_layer_flag(unfinished, ntiles, count2, count2 + 1, use_cond ? &cond : nullptr, s);
      }
      ctx->launches++;
      if (policy) {
        CounterSrc cs{};
        cs.src[0] = ctx->lp_dev;  // consumed
        cs.src[1] = ra + 1;       // layer-A listed pairs
        cs.src[2] = count2;       // unfinished tiles
        cs.n = 3;
        launch_publish_counters(cs, ctx->lp_hdev, s);
        ctx->launches++;
        LGS_CUDA(cudaEventRecord(ctx->lp_ev, s));
        ctx->lp_pending = true;
        ctx->lp_ntiles = ntiles;
        ctx->lp_div = ldiv;
        ctx->lp_map = (uint64_t)map->dm.n;
      }
      if (use_cond) LGS_TRY(cond_begin(ctx, cond));
      lgs_status st2 = LGS_OK;
      {
        cudaStream_t s2 = ctx->stream;  // the conditional body's capture stream inside a plan
        {
          PhaseScope ph(ctx, PH_TILE_SORT);
          launch_layer_prep(unfinished, t->ranges, dc.tiles_x, dc.tiles_y, sat, order2, s2);
          launch_depth_order_rest(t->vb, n, dc.near_plane, otemp, idx_sorted, count2, s2);
          launch_layer_count(t->vb, idx_sorted, n, dc.tiles_x, sat, count2, dkey_sorted, count2 + 1, s2,
                             fuse ? t->gacc : nullptr, cj);
          launch_scan_counts(dkey_sorted, n, incl, temp, temp_bytes, s2);
          const BinPass b{incl, count2 + 1, n, (uint32_t)cap, capA, unfinished, count2};
          launch_fast_binning(t->vb, idx_sorted, n, ntiles, dc.tiles_x, b, scratch_b, t->vals, t->ranges,
                              ctx->dev_u32 + 2, s2);
        }
        FwdOut fo2 = fo;
        {
          PhaseScope ph(ctx, PH_BLEND_FWD);
          if (fuse)
            launch_blend_fused_l1(dm, dc, t->vb, TileLists{t->vals, t->ranges, order2, t->counter, count2}, fo2,
                                  t->gacc, s2, false, true);
          else
            launch_blend_fwd(dm, dc, t->vb, TileLists{t->vals, t->ranges, order2, t->counter, count2}, t->ps,
                             fo2, s2);
        }
        if (cudaGetLastError() != cudaSuccess) st2 = fail(LGS_ECUDA, "layered binning pass 2 launch failed");
      }
      ctx->launches += 13;
      if (use_cond) LGS_TRY(cond_end(ctx));
      LGS_TRY(st2);
      dfree(ctx, scratch_b);
      dfree(ctx, count2);
      dfree(ctx, order2);
      dfree(ctx, sat);
      dfree(ctx, cand_rect);
      dfree(ctx, ra);
      LGS_CUDA(cudaGetLastError());
      return LGS_OK;
    }
    LGS_TRY(dalloc(ctx, &t->vals, cap));
    t->vals_count = cap;
    if (fast) {
      // stable counting sort by tile straight into the final lists (binning_fast.cu)
      uint32_t* scratch = nullptr;
      LGS_TRY(dalloc(ctx, reinterpret_cast<uint8_t**>(&scratch), fast_binning_scratch_bytes(cap, n, ntiles)));
      {
        PhaseScope ph(ctx, PH_TILE_SORT);
        const BinPass all{incl, incl + n - 1, n, (uint32_t)cap, 0u, nullptr};
        launch_fast_binning(t->vb, idx_sorted, n, ntiles, dc.tiles_x, all, scratch, t->vals, t->ranges,
                            ctx->dev_u32 + 1, s);
      }
      ctx->launches += cap > 0 ? 5 : 0;
      dfree(ctx, scratch);
    } else {
      uint16_t* keys_in = nullptr;
      uint32_t* vals_in = nullptr;
      LGS_TRY(dalloc(ctx, &keys_in, cap));
      LGS_TRY(dalloc(ctx, &vals_in, cap));
      LGS_TRY(dalloc(ctx, &t->keys, cap));
      {
        PhaseScope ph(ctx, PH_DUPLICATE);
        launch_duplicate(t->vb, idx_sorted, incl, n, dc.tiles_x, keys_in, vals_in, s);
      }
      const size_t sort_bytes = binning_temp_bytes(0, cap, tile_bits);
      void* stemp = nullptr;
      LGS_TRY(dalloc(ctx, reinterpret_cast<uint8_t**>(&stemp), sort_bytes));
      {
        PhaseScope ph(ctx, PH_TILE_SORT);
        launch_tile_sort(keys_in, t->keys, vals_in, t->vals, cap, tile_bits, stemp, sort_bytes, s);
        launch_ranges(t->keys, cap, ntiles, t->ranges, s);
      }
      ctx->launches += (n > 0 ? 1 : 0) + (cap > 0 ? 5 : 0);
      dfree(ctx, stemp);
      dfree(ctx, keys_in);
      dfree(ctx, vals_in);
    }
    {
      PhaseScope ph(ctx, PH_TILE_SORT);
      launch_tile_order(t->ranges, ntiles, t->order, s);  // longest tile list first
    }
    ctx->launches++;
    if (targets) LGS_CUDA(cudaMemsetAsync(t->loss, 0, sizeof(double), s));
    // complete lists with the fused L1 step (a small view binned in one pass): the fused kernel,
    // with every visible Gaussian's accumulator row zeroed (any may be listed)
    const bool fuse_all = (ctx->capturing || ctx->fused_eager) && targets && blend_fused_supported(dp) &&
                          slots_for(dp) == 32 && n > 0;
    if (fuse_all) {
      dfree(ctx, t->gacc);
      LGS_TRY(dalloc(ctx, &t->gacc, (size_t)n * 32));
      LGS_CUDA(cudaMemsetAsync(t->gacc, 0, sizeof(float) * (size_t)n * 32, s));
      t->bwd_fused = true;
    }
    {
      PhaseScope ph(ctx, PH_BLEND_FWD);
      if (fuse_all)
        launch_blend_fused_l1(dm, dc, t->vb, TileLists{t->vals, t->ranges, t->order, t->counter}, fo, t->gacc, s,
                              false, ntiles < 2 * device_sm_count());
      else
        launch_blend_fwd(dm, dc, t->vb, TileLists{t->vals, t->ranges, t->order, t->counter}, t->ps, fo, s);
    }
    ctx->launches++;
    LGS_CUDA(cudaGetLastError());
    return LGS_OK;
  };

  int64_t P = 0;
  const bool speculate = fast && n > 0 && ctx->pairs_cap > 0;
  if (ctx->capturing) {  // lgs_plan: P is checked after each replay (lgs_plan_sync)
    if (!speculate) return bail(fail(LGS_EINVAL, "plan capture needs the fast binning and a known capacity"));
    TRYB(bin_and_blend(ctx->pairs_cap, true));
    P = ctx->pairs_cap;
  } else if (speculate) {
    TRYB(bin_and_blend(ctx->pairs_cap, true));
    CUDAB(cudaEventSynchronize(ctx->pairs_ready));  // long done: the GPU is busy with the queued forward
    P = ctx->host_u32[0];
    if (P > ctx->pairs_cap) {
      ctx->pairs_cap = P + P / 4;
      TRYB(bin_and_blend(P, false));
    }
  } else {
    if (n > 0) {
      CUDAB(cudaEventSynchronize(ctx->pairs_ready));
      P = ctx->host_u32[0];
    }
    TRYB(bin_and_blend(P, true));
    if (fast) ctx->pairs_cap = std::max<int64_t>(ctx->pairs_cap, P + P / 4);
  }
  t->pairs = P;
  if (otemp) dfree(ctx, otemp);
  dfree(ctx, temp);
  dfree(ctx, dkey_sorted);
  dfree(ctx, idx_sorted);
  dfree(ctx, incl);
  if (tstage) dfree(ctx, tstage);
  if (mapped && !ctx->mh_pending && layered) {
    CounterSrc cs{};
    cs.src[0] = ctx->mh_listed_dev;
    cs.n = 1;
    launch_publish_counters(cs, ctx->mh_listed_hdev, s);
    ctx->launches++;
    CUDAB(cudaEventRecord(ctx->mh_event, s));
    ctx->mh_pending = true;
    ctx->mh_pending_key = map->dm.sh;
    ctx->mh_pending_n = n;
  }
  if (di.staged) {
    if (di.rgb) CUDAB(cudaMemcpyAsync(out->rgb, di.rgb, sizeof(float) * npix * 3, cudaMemcpyDeviceToHost, s));
    if (di.depth) CUDAB(cudaMemcpyAsync(out->depth, di.depth, sizeof(float) * npix, cudaMemcpyDeviceToHost, s));
    if (di.feat) CUDAB(cudaMemcpyAsync(out->feat, di.feat, sizeof(float) * npix * d, cudaMemcpyDeviceToHost, s));
    if (di.acc) CUDAB(cudaMemcpyAsync(out->acc, di.acc, sizeof(float) * npix, cudaMemcpyDeviceToHost, s));
    ctx->bytes_d2h += (int64_t)(sizeof(float) * npix * ((di.rgb ? 3 : 0) + (di.depth ? 1 : 0) + (di.feat ? d : 0) +
                                                       (di.acc ? 1 : 0)));
    dfree(ctx, di.rgb); dfree(ctx, di.depth); dfree(ctx, di.feat); dfree(ctx, di.acc);
    CUDAB(cudaStreamSynchronize(s));
  }
  // the tape no longer needs the sort keys of the depth pass
  dfree(ctx, t->vb.dkey);
  dfree(ctx, t->vb.iota);
  t->vb.dhist = nullptr;  // lived in the depth-order scratch, freed above
  t->vb.dslot = nullptr;
  t->vb.dpart = nullptr;
  if (tape) *tape = t;
  else free_saved(t);
  return LGS_OK;
#undef TRYB
#undef CUDAB
}

LGS_API lgs_status lgs_render(lgs_ctx* ctx, const lgs_gaussians* src, const lgs_camera* cam,
                              const lgs_render_config* cfg, lgs_images* out, lgs_saved** tape) {
  lgs_map* m = nullptr;
  LGS_TRY(lgs_map_create(ctx, src, &m));
  lgs_saved* t = nullptr;
  lgs_status st = lgs_render_forward(ctx, m, cam, cfg, nullptr, out, &t);
  if (st != LGS_OK) {
    free_map(m);
    return st;
  }
  t->owned_map = m;
  if (tape) *tape = t;
  else free_saved(t);
  return LGS_OK;
}

// -------------------------------------------------------------------------------------------
// backward
// -------------------------------------------------------------------------------------------
namespace {

// ---- host-gradient delta mode (LGS_OPT_HOST_GRAD_DELTA) --------------------------------------
// With the depth-layered binning a view's gradient is nonzero on a few thousand of N rows, yet
// the dense MapGradients (renderer.hpp:59-68) of a host caller is N x (11 + 3K + d) floats (150 MB
// at the headline size).  When the caller hands the same host buffers to every backward and leaves
// them alone in between, the rows zero now AND in the previous backward already hold zeros: only
// the rows nonzero now (packed on the device as (index, row) records, sparse_reduce.cu) cross the
// link, and the rows nonzero last time but not now are zeroed on the host.  The buffers hold the
// exact dense gradient after every call.

// rows of the device gradient `src` with a nonzero component -> (index, row) records on the host
// grows the context's page-locked staging block (1.5x headroom: a rare, synchronizing allocation)
lgs_status delta_stage(lgs_ctx* ctx, size_t bytes, void** out) {
  if (bytes > ctx->delta_stage_bytes) {
    if (ctx->delta_stage) cudaFreeHost(ctx->delta_stage);
    ctx->delta_stage = nullptr;
    ctx->delta_stage_bytes = 0;
    const size_t want = bytes + bytes / 2 + 4096;
    LGS_CUDA(cudaHostAlloc(&ctx->delta_stage, want, cudaHostAllocDefault));
    ctx->delta_stage_bytes = want;
  }
  *out = ctx->delta_stage;
  return LGS_OK;
}

// (index, R values) records of the rows with any nonzero value, in the page-locked staging block
lgs_status pack_nonzero_rows(lgs_ctx* ctx, float* const src[6], int64_t n, int K, int d, const float** recs,
                             uint32_t* rows_out) {
  cudaStream_t s = ctx->stream;
  const int width[6] = {3, 4, 3, 1, 3 * K, d};
  const int R = rows_values(width, src);
  uint32_t *list = nullptr, *cnt = nullptr;
  LGS_TRY(dalloc(ctx, &list, (size_t)n));
  LGS_TRY(dalloc(ctx, &cnt, 1));
  launch_rows_scan(src, width, n, list, cnt, s);
  uint32_t* hrows = ctx->host_u32 + 8;  // pinned scalar slot
  LGS_CUDA(cudaMemcpyAsync(hrows, cnt, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  LGS_CUDA(cudaStreamSynchronize(s));
  const uint32_t rows = *hrows;
  ctx->bytes_d2h += (int64_t)sizeof(uint32_t);
  *recs = nullptr;
  if (rows) {
    const size_t bytes = sizeof(float) * (size_t)rows * (R + 1);
    void* stage = nullptr;
    LGS_TRY(delta_stage(ctx, bytes, &stage));
    float* drec = nullptr;
    LGS_TRY(dalloc(ctx, &drec, (size_t)rows * (R + 1)));
    launch_rows_pack(src, width, n, list, cnt, rows, drec, s);
    LGS_CUDA(cudaMemcpyAsync(stage, drec, bytes, cudaMemcpyDeviceToHost, s));
    ctx->bytes_d2h += (int64_t)bytes;
    dfree(ctx, drec);
    *recs = static_cast<const float*>(stage);
  }
  dfree(ctx, list);
  dfree(ctx, cnt);
  LGS_CUDA(cudaStreamSynchronize(s));
  *rows_out = rows;
  return LGS_OK;
}

// write (or zero) row i of the six host arrays in the reference layouts; rec = R values or nullptr
void host_row(float* const dst[6], const int width[6], int64_t n, uint32_t i, const float* rec) {
  int off = 0;
  for (int a = 0; a < 6; ++a) {
    if (!dst[a] || !width[a]) continue;
    for (int j = 0; j < width[a]; ++j) {
      float* e = a == 5 ? dst[5] + (int64_t)j * n + i : dst[a] + (int64_t)i * width[a] + j;
      *e = rec ? rec[off + j] : 0.f;
    }
    off += width[a];
  }
}

lgs_status host_grads_delta(lgs_ctx* ctx, float* const dst[6], float* const src[6], int64_t n, int K, int d) {
  const float* recs = nullptr;
  uint32_t rows = 0;
  LGS_TRY(pack_nonzero_rows(ctx, src, n, K, d, &recs, &rows));
  int width[6] = {3, 4, 3, 1, 3 * K, d};
  for (int a = 0; a < 6; ++a)
    if (!src[a]) width[a] = 0;
  const int R = rows_values(width, src);
  for (uint32_t i : ctx->delta_rows) host_row(dst, width, n, i, nullptr);  // last call's rows -> 0
  ctx->delta_rows.resize(rows);
  for (uint32_t k = 0; k < rows; ++k) {
    const float* r = recs + (size_t)k * (R + 1);
    const uint32_t i = __builtin_bit_cast(uint32_t, r[0]);
    host_row(dst, width, n, i, r + 1);
    ctx->delta_rows[k] = i;
  }
  return LGS_OK;
}

// after a dense write: remember the destination and its nonzero rows for the next delta backward
lgs_status host_grads_note_rows(lgs_ctx* ctx, float* const src[6], int64_t n, int K, int d,
                                const std::array<float*, 6>& key) {
  cudaStream_t s = ctx->stream;
  const int width[6] = {3, 4, 3, 1, 3 * K, d};
  uint32_t *list = nullptr, *cnt = nullptr;
  LGS_TRY(dalloc(ctx, &list, (size_t)n));
  LGS_TRY(dalloc(ctx, &cnt, 1));
  launch_rows_scan(src, width, n, list, cnt, s);
  uint32_t* hrows = ctx->host_u32 + 8;  // pinned scalar slot
  LGS_CUDA(cudaMemcpyAsync(hrows, cnt, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  LGS_CUDA(cudaStreamSynchronize(s));
  const uint32_t rows = *hrows;
  void* stage = nullptr;
  if (rows) {
    LGS_TRY(delta_stage(ctx, sizeof(uint32_t) * rows, &stage));
    LGS_CUDA(cudaMemcpyAsync(stage, list, sizeof(uint32_t) * rows, cudaMemcpyDeviceToHost, s));
  }
  dfree(ctx, list);
  dfree(ctx, cnt);
  LGS_CUDA(cudaStreamSynchronize(s));
  ctx->delta_rows.assign(static_cast<const uint32_t*>(stage), static_cast<const uint32_t*>(stage) + rows);
  ctx->delta_dst = key;
  ctx->delta_n = n;
  return LGS_OK;
}

lgs_status run_backward(lgs_ctx* ctx, const lgs_saved* t, const BwdIn& in_dev, lgs_map_grads* grads, float* pose_grad,
                        bool async_pose = false) {
  if (!version_live(t->map_version))
    return fail(LGS_EINVAL, "the map of this tape was pruned or destroyed after the render");
  cudaStream_t s = ctx->stream;
  const int64_t n = t->dm.n;
  const int d = t->dm.d, K = t->dm.K;
  const int slots = slots_for(t->dm.dp);
  float* gacc = nullptr;
  if (t->bwd_fused) {  // the fused-L1 forward already accumulated the screen-space gradients
    gacc = t->gacc;
  } else {
    LGS_TRY(dalloc(ctx, &gacc, (size_t)n * slots));
    launch_zero_active_rows(t->vb, n, gacc, slots, s);  // rows the blend kernel may add into
  }
  if (!t->bwd_fused) {
    PhaseScope ph(ctx, PH_BLEND_BWD);
    launch_blend_bwd(t->dm, t->cam, t->vb, TileLists{t->vals, t->ranges, t->lpt_order ? t->order : nullptr, t->counter},
                     t->ps, in_dev, gacc, slots, s);
    ctx->launches += 2;
  }

  GradOut go{};
  go.accumulate = grads ? grads->accumulate : 0;
  float* gstage = nullptr;
  const size_t sz_pos = (size_t)n * 3, sz_rot = (size_t)n * 4, sz_ls = (size_t)n * 3, sz_op = (size_t)n,
               sz_sh = (size_t)n * K * 3, sz_ft = (size_t)n * d;
  const bool host = grads && grads->memory == LGS_MEM_HOST;
  if (grads) {
    if (host) {
      LGS_TRY(dalloc(ctx, &gstage, sz_pos + sz_rot + sz_ls + sz_op + sz_sh + sz_ft));
      float* p = gstage;
      float* dst[6] = {grads->position, grads->rotation, grads->log_scale, grads->opacity_logit, grads->sh,
                       grads->feature};
      const size_t szs[6] = {sz_pos, sz_rot, sz_ls, sz_op, sz_sh, sz_ft};
      float** outs[6] = {&go.position, &go.rotation, &go.log_scale, &go.opacity_logit, &go.sh, &go.feature};
      for (int k = 0; k < 6; ++k) {
        if (dst[k] && szs[k]) {
          *outs[k] = p;
          if (go.accumulate) LGS_CUDA(cudaMemcpyAsync(p, dst[k], sizeof(float) * szs[k], cudaMemcpyHostToDevice, s));
        }
        p += szs[k];
      }
    } else {
      go = device_grad_out(grads, d);
    }
  }
  go.skip = t->miss;  // (after device_grad_out above rebuilt go)
  // captured step with the active-row chain: its last CTA writes the pose gradient in place and
  // copies the next tile order (GradOut::done) when the destination is device-accessible
  bool epi = ctx->capturing && t->vb.active && async_pose;
  if (epi && pose_grad) {
    cudaPointerAttributes pa{};
    epi = cudaPointerGetAttributes(&pa, pose_grad) == cudaSuccess && pa.type != cudaMemoryTypeUnregistered &&
          pa.devicePointer != nullptr;
    cudaGetLastError();
  }
  double* dpose = nullptr;
  if (pose_grad || epi) {
    LGS_TRY(dalloc(ctx, &dpose, 8));  // 6 accumulators, [6]: the chain's CTA counter
    LGS_CUDA(cudaMemsetAsync(dpose, 0, sizeof(double) * 8, s));
    if (pose_grad) go.pose = dpose;
  }
  if (epi) {
    go.done = reinterpret_cast<uint32_t*>(dpose + 6);
    if (pose_grad) {
      cudaPointerAttributes pa{};
      cudaPointerGetAttributes(&pa, pose_grad);
      go.pose_out = static_cast<float*>(pa.devicePointer);
    }
  }
  // zero rows already enqueued on the plan's side branch (the forward forked it)?
  bool zeroed = ctx->prezero_forked && grads == ctx->prezero && !host && t->vb.active;
  if (ctx->prezero_forked) {
    LGS_CUDA(cudaStreamWaitEvent(s, ctx->side_join, 0));
    ctx->prezero_forked = false;
    if (ctx->lpt_forked) {  // the next replay's tile order (by the chain's last CTA if it can)
      if (epi) {
        go.copy_src = ctx->cap_lpt_next;
        go.copy_dst = ctx->cap_lpt_cur;
        go.copy_n = t->ntiles;
      } else {
        launch_copy_u32(ctx->cap_lpt_next, t->ntiles, ctx->cap_lpt_cur, s);
        ctx->launches++;
      }
      ctx->lpt_forked = false;
    }
  }
  if (t->vb.active && !zeroed) {  // sparse chain below: the zero rows first (none when accumulating)
    PhaseScope ph(ctx, PH_GRAD_ZERO);
    launch_grad_zero(go, n, K, t->dm.dp > 0 ? d : 0, s);
    if (!go.accumulate) ctx->launches++;
    zeroed = true;
  }
  {
    PhaseScope ph(ctx, PH_PREPROCESS_BWD);
    launch_preprocess_bwd(t->dm, t->cam, t->vb, gacc, slots, go, zeroed, s);
  }
  ctx->launches++;
  LGS_CUDA(cudaGetLastError());
  if (host) {
    float* dst[6] = {grads->position, grads->rotation, grads->log_scale, grads->opacity_logit, grads->sh,
                     grads->feature};
    float* src[6] = {go.position, go.rotation, go.log_scale, go.opacity_logit, go.sh, go.feature};
    const size_t szs[6] = {sz_pos, sz_rot, sz_ls, sz_op, sz_sh, sz_ft};
    const std::array<float*, 6> key = {dst[0], dst[1], dst[2], dst[3], dst[4], dst[5]};
    const bool delta = ctx->host_grad_delta && !go.accumulate && ctx->delta_n == n && ctx->delta_dst == key;
    if (delta) {
      LGS_TRY(host_grads_delta(ctx, dst, src, n, K, d));  // synchronizes
    } else {
      for (int k = 0; k < 6; ++k)
        if (dst[k] && src[k] && szs[k]) {
          LGS_CUDA(cudaMemcpyAsync(dst[k], src[k], sizeof(float) * szs[k], cudaMemcpyDeviceToHost, s));
          ctx->bytes_d2h += (int64_t)(sizeof(float) * szs[k]);
        }
      if (ctx->host_grad_delta && !go.accumulate) LGS_TRY(host_grads_note_rows(ctx, src, n, K, d, key));
    }
  }
  double hpose[6];
  if (pose_grad && async_pose && go.pose_out) {
    // written by the chain's last CTA
  } else if (pose_grad && async_pose) {
    // stream-ordered: fp64 accumulator -> float, copied to pinned-host or device memory
    launch_pose_to_float(dpose, reinterpret_cast<float*>(dpose), s);
    LGS_CUDA(cudaMemcpyAsync(pose_grad, dpose, sizeof(float) * 6, cudaMemcpyDefault, s));
    ctx->launches++;
  } else if (pose_grad) {
    LGS_CUDA(cudaMemcpyAsync(hpose, dpose, sizeof hpose, cudaMemcpyDeviceToHost, s));
  }
  if (!t->bwd_fused) dfree(ctx, gacc);
  dfree(ctx, gstage);
  dfree(ctx, dpose);
  if (host || (pose_grad && !async_pose)) LGS_CUDA(cudaStreamSynchronize(s));
  if (pose_grad && !async_pose)
    for (int a = 0; a < 6; ++a) pose_grad[a] = (float)hpose[a];
  return LGS_OK;
}

lgs_status check_shape(const int32_t shape[3], int H, int W, int C, const char* name) {
  if (shape[0] == 0 && shape[1] == 0 && shape[2] == 0) return LGS_OK;
  if (shape[0] != H || shape[1] != W || shape[2] != C)  // renderer.cpp:174-180
    return fail(LGS_EINVAL, "render_backward: bad shape for %s", name);
  return LGS_OK;
}

}  // namespace

LGS_API lgs_status lgs_render_backward(lgs_ctx* ctx, const lgs_saved* tape, const lgs_cotangents* cot,
                                       lgs_map_grads* grads, float* pose_grad) {
  if (!ctx || !tape) return fail(LGS_EINVAL, "ctx/tape is NULL");
  if (tape->bwd_fused)
    return fail(LGS_EINVAL, "tape of a fused-L1 render (LGS_OPT_FUSED_EAGER): use lgs_render_backward_l1");
  const int H = tape->cam.H, W = tape->cam.W, d = tape->dm.d;
  const size_t npix = (size_t)W * H;
  BwdIn in{};
  float* stage = nullptr;
  if (cot) {
    if (cot->rgb) LGS_TRY(check_shape(cot->rgb_shape, H, W, 3, "grad_rgb"));
    if (cot->depth) LGS_TRY(check_shape(cot->depth_shape, H, W, 1, "grad_depth"));
    if (cot->feat) LGS_TRY(check_shape(cot->feat_shape, H, W, d, "grad_feat"));
  }
  LGS_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  if (cot) {
    in.g_rgb = cot->rgb;
    in.g_depth = cot->depth;
    in.g_feat = d > 0 ? cot->feat : nullptr;
    if (cot->memory == LGS_MEM_HOST) {
      LGS_TRY(dalloc(ctx, &stage, npix * (4 + d)));
      if (cot->rgb) {
        LGS_CUDA(cudaMemcpyAsync(stage, cot->rgb, sizeof(float) * npix * 3, cudaMemcpyHostToDevice, s));
        in.g_rgb = stage;
      }
      if (cot->depth) {
        LGS_CUDA(cudaMemcpyAsync(stage + npix * 3, cot->depth, sizeof(float) * npix, cudaMemcpyHostToDevice, s));
        in.g_depth = stage + npix * 3;
      }
      if (cot->feat && d > 0) {
        LGS_CUDA(cudaMemcpyAsync(stage + npix * 4, cot->feat, sizeof(float) * npix * d, cudaMemcpyHostToDevice, s));
        in.g_feat = stage + npix * 4;
      }
    }
  }
  lgs_status st = run_backward(ctx, tape, in, grads, pose_grad);
  if (stage) dfree(ctx, stage);
  return st;
}

LGS_API lgs_status lgs_render_backward_l1(lgs_ctx* ctx, const lgs_saved* tape, lgs_map_grads* grads,
                                          float* pose_grad) {
  if (!ctx || !tape) return fail(LGS_EINVAL, "ctx/tape is NULL");
  if (!tape->cot) return fail(LGS_EINVAL, "tape has no fused L1 cotangents (forward without targets)");
  LGS_CUDA(cudaSetDevice(ctx->device));
  BwdIn in{};
  in.g_rgb = tape->cot;
  in.cot_stride = 4 + tape->dm.dp;
  return run_backward(ctx, tape, in, grads, pose_grad);
}

LGS_API lgs_status lgs_render_backward_loss(lgs_ctx* ctx, const lgs_saved* tape, lgs_map_grads* grads,
                                            float* pose_grad) {
  return lgs_render_backward_l1(ctx, tape, grads, pose_grad);
}

LGS_API lgs_status lgs_render_backward_loss_async(lgs_ctx* ctx, const lgs_saved* tape, lgs_map_grads* grads,
                                                  float* pose_grad) {
  if (!ctx || !tape) return fail(LGS_EINVAL, "ctx/tape is NULL");
  if (!tape->cot) return fail(LGS_EINVAL, "tape holds no loss cotangents");
  if (grads && grads->memory != LGS_MEM_DEVICE) return fail(LGS_EINVAL, "async backward needs device gradients");
  LGS_CUDA(cudaSetDevice(ctx->device));
  BwdIn in{};
  in.g_rgb = tape->cot;
  in.cot_stride = 4 + tape->dm.dp;
  return run_backward(ctx, tape, in, grads, pose_grad, true);
}

LGS_API lgs_loss_weights lgs_loss_weights_default(void) {
  lgs_loss_weights w;
  w.w_l1 = 0.8;     // SPEC.md:454 rgb mix 0.8 L1 + 0.2 D-SSIM
  w.w_depth = 0.5;
  w.w_feat = 1.0;
  return w;
}

LGS_API lgs_status lgs_mapping_loss(lgs_ctx* ctx, lgs_saved* t, const lgs_images* rendered, const lgs_keyframe* kf,
                                    const lgs_decoder* dec, const lgs_loss_weights* w_in, lgs_loss_breakdown* out) {
  if (!ctx || !t || !rendered || !kf) return fail(LGS_EINVAL, "ctx/tape/rendered/keyframe is NULL");
  if (t->bwd_fused) return fail(LGS_EINVAL, "tape of a fused-L1 render (LGS_OPT_FUSED_EAGER) carries the L1 loss");
  const int H = t->cam.H, W = t->cam.W, d = t->dm.d, dp = t->dm.dp;
  if (H < 11 || W < 11) return fail(LGS_EINVAL, "ssim: image %dx%d smaller than the 11x11 window", W, H);
  if (!rendered->rgb || !kf->rgb || !kf->depth) return fail(LGS_EINVAL, "rendered rgb / keyframe rgb, depth needed");
  if (d > 0) {
    if (!rendered->feat || !kf->feat_gt || !dec) return fail(LGS_EINVAL, "feature loss needs feat, feat_gt, decoder");
    if (dec->low_dim != d) return fail(LGS_EINVAL, "decoder low_dim %d != map feature dim %d", dec->low_dim, d);
    if (!dec->w1 || !dec->b1 || !dec->w2 || !dec->b2) return fail(LGS_EINVAL, "decoder weights missing");
    if (!decoder_supported(dec->hidden, dp, dec->high_dim))
      return fail(LGS_EINVAL, "decoder hidden %d / D %d not supported (hidden 64, D <= 640)", dec->hidden,
                  dec->high_dim);
  }
  const lgs_loss_weights w = w_in ? *w_in : lgs_loss_weights_default();
  LGS_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const size_t npix = (size_t)H * W;
  const int D = d > 0 ? dec->high_dim : 0, hid = d > 0 ? dec->hidden : 0;
  if (!t->cot) LGS_TRY(dalloc(ctx, &t->cot, npix * (4 + dp)));
  if (!t->loss_sums) LGS_TRY(dalloc(ctx, &t->loss_sums, LOSS_COUNT));
  // host inputs are staged (the reference API takes host images); device inputs are used in place
  std::vector<float*> staged;
  auto dev_in = [&](const float* p, size_t count, int memory, const float** outp) -> lgs_status {
    if (memory != LGS_MEM_HOST || !p) {
      *outp = p;
      return LGS_OK;
    }
    float* q = nullptr;
    LGS_TRY(dalloc(ctx, &q, count));
    LGS_CUDA(cudaMemcpyAsync(q, p, sizeof(float) * count, cudaMemcpyHostToDevice, s));
    staged.push_back(q);
    *outp = q;
    return LGS_OK;
  };
  LossArgs a;
  a.H = H; a.W = W; a.d = d; a.dp = dp; a.D = D; a.hidden = hid;
  a.depth = t->ps.depth;
  a.acc = t->ps.acc;
  lgs_status st = LGS_OK;
  auto cleanup = [&]() {
    for (float* q : staged) dfree(ctx, q);
  };
#define LOSS_TRY(expr)          \
  do {                          \
    st = (expr);                \
    if (st != LGS_OK) {         \
      cleanup();                \
      return st;                \
    }                           \
  } while (0)
  LOSS_TRY(dev_in(rendered->rgb, npix * 3, rendered->memory, &a.rgb));
  if (d > 0) LOSS_TRY(dev_in(rendered->feat, npix * d, rendered->memory, &a.feat));
  LOSS_TRY(dev_in(kf->rgb, npix * 3, kf->memory, &a.rgb_gt));
  LOSS_TRY(dev_in(kf->depth, npix, kf->memory, &a.depth_gt));
  if (d > 0) {
    LOSS_TRY(dev_in(kf->feat_gt, npix * D, kf->memory, &a.feat_gt));
    LOSS_TRY(dev_in(dec->w1, (size_t)hid * d, dec->memory, &a.w1));
    LOSS_TRY(dev_in(dec->b1, (size_t)hid, dec->memory, &a.b1));
    LOSS_TRY(dev_in(dec->w2, (size_t)D * hid, dec->memory, &a.w2));
    LOSS_TRY(dev_in(dec->b2, (size_t)D, dec->memory, &a.b2));
  }
  float* abc = nullptr;
  LOSS_TRY(dalloc(ctx, &abc, npix * 9));
  staged.push_back(abc);
  a.abc = abc;
  a.sums = t->loss_sums;
  a.cot = t->cot;
  a.cot_stride = 4 + dp;
  a.w_l1 = w.w_l1; a.w_depth = w.w_depth; a.w_feat = d > 0 ? w.w_feat : 0.0;
  {
    PhaseScope ph(ctx, PH_LOSS);
    if (launch_mapping_loss(a, s) != 0) {
      cleanup();
      return fail(LGS_ECUDA, "mapping loss launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    }
  }
  ctx->launches += 3 + (d > 0 ? 1 : 0);
  LOSS_TRY(cudaGetLastError() == cudaSuccess ? LGS_OK : fail(LGS_ECUDA, "mapping loss kernels failed"));
  cleanup();
#undef LOSS_TRY
  if (out) {
    double h[LOSS_COUNT];
    LGS_CUDA(cudaMemcpyAsync(h, t->loss_sums, sizeof h, cudaMemcpyDeviceToHost, s));
    LGS_CUDA(cudaStreamSynchronize(s));
    const double npos = (double)(H - 10) * (double)(W - 10);
    out->ssim = h[LOSS_SSIM] / (3.0 * npos);
    out->l_rgb = w.w_l1 * h[LOSS_L1_RGB] / (3.0 * (double)npix) + (1.0 - w.w_l1) * (1.0 - out->ssim) / 2.0;
    out->depth_pixels = (int64_t)h[LOSS_DEPTH_CNT];
    out->l_depth = out->depth_pixels ? h[LOSS_DEPTH_ABS] / h[LOSS_DEPTH_CNT] : 0.0;
    out->l_feat = d > 0 ? h[LOSS_FEAT_ABS] / ((double)npix * D) : 0.0;
    out->l_total = out->l_rgb + w.w_depth * out->l_depth + w.w_feat * out->l_feat;
  }
  return LGS_OK;
}

LGS_API lgs_status lgs_debug_cotangents(lgs_ctx* ctx, const lgs_saved* t, float* rgb, float* depth, float* feat) {
  if (!ctx || !t) return fail(LGS_EINVAL, "ctx/tape is NULL");
  if (!t->cot) return fail(LGS_EINVAL, "tape holds no cotangents");
  const size_t npix = (size_t)t->cam.H * t->cam.W;
  const int stride = 4 + t->dm.dp, d = t->dm.d;
  std::vector<float> h(npix * stride);
  LGS_CUDA(cudaSetDevice(ctx->device));
  LGS_CUDA(cudaMemcpyAsync(h.data(), t->cot, sizeof(float) * h.size(), cudaMemcpyDeviceToHost, ctx->stream));
  LGS_CUDA(cudaStreamSynchronize(ctx->stream));
  for (size_t p = 0; p < npix; ++p) {
    const float* c = h.data() + p * stride;
    if (rgb) std::memcpy(rgb + p * 3, c, sizeof(float) * 3);
    if (depth) depth[p] = c[3];
    if (feat && d) std::memcpy(feat + p * d, c + 4, sizeof(float) * d);
  }
  return LGS_OK;
}

LGS_API lgs_status lgs_coverage_mask(lgs_ctx* ctx, const lgs_saved* t, const float* measured_depth, int32_t memory,
                                     uint8_t* mask, int32_t mask_memory, int64_t* count) {
  if (!ctx || !t || !measured_depth || !mask) return fail(LGS_EINVAL, "ctx/tape/depth/mask is NULL");
  LGS_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const size_t npix = (size_t)t->cam.H * t->cam.W;
  const float* md = measured_depth;
  float* stage = nullptr;
  if (memory == LGS_MEM_HOST) {
    LGS_TRY(dalloc(ctx, &stage, npix));
    LGS_CUDA(cudaMemcpyAsync(stage, measured_depth, sizeof(float) * npix, cudaMemcpyHostToDevice, s));
    md = stage;
  }
  uint8_t* dmask = mask;
  if (mask_memory == LGS_MEM_HOST) LGS_TRY(dalloc(ctx, &dmask, npix));
  unsigned long long* dcount = nullptr;
  LGS_TRY(dalloc(ctx, &dcount, 1));
  {
    PhaseScope ph(ctx, PH_COVERAGE);
    launch_coverage(t->ps.acc, t->ps.depth, md, (int64_t)npix, dmask, dcount, s);
  }
  ctx->launches += npix ? 1 : 0;
  unsigned long long hcount = 0;
  if (mask_memory == LGS_MEM_HOST) LGS_CUDA(cudaMemcpyAsync(mask, dmask, npix, cudaMemcpyDeviceToHost, s));
  if (count) LGS_CUDA(cudaMemcpyAsync(&hcount, dcount, sizeof hcount, cudaMemcpyDeviceToHost, s));
  if (mask_memory == LGS_MEM_HOST) dfree(ctx, dmask);
  dfree(ctx, stage);
  dfree(ctx, dcount);
  if (count || mask_memory == LGS_MEM_HOST || memory == LGS_MEM_HOST) LGS_CUDA(cudaStreamSynchronize(s));
  if (count) *count = (int64_t)hcount;
  LGS_CUDA(cudaGetLastError());
  return LGS_OK;
}

LGS_API lgs_status lgs_saved_l1_loss(lgs_ctx* ctx, const lgs_saved* tape, double* loss) {
  if (!ctx || !tape || !loss) return fail(LGS_EINVAL, "NULL argument");
  if (!tape->loss) return fail(LGS_EINVAL, "tape has no fused L1 loss");
  LGS_CUDA(cudaSetDevice(ctx->device));
  LGS_CUDA(cudaMemcpyAsync(loss, tape->loss, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  LGS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LGS_OK;
}

LGS_API lgs_status lgs_saved_stats(const lgs_saved* tape, lgs_render_stats* st) {
  if (!tape || !st) return fail(LGS_EINVAL, "NULL argument");
  lgs_ctx* ctx = tape->ctx;
  LGS_CUDA(cudaSetDevice(ctx->device));
  std::vector<uint32_t> tiles((size_t)tape->dm.n);
  std::vector<uint2> ranges((size_t)tape->ntiles);
  if (tape->dm.n)
    LGS_CUDA(cudaMemcpyAsync(tiles.data(), tape->vb.tiles, sizeof(uint32_t) * tiles.size(), cudaMemcpyDeviceToHost,
                             ctx->stream));
  LGS_CUDA(cudaMemcpyAsync(ranges.data(), tape->ranges, sizeof(uint2) * ranges.size(), cudaMemcpyDeviceToHost,
                           ctx->stream));
  std::vector<uint8_t> act(tape->vb.active ? (size_t)tape->dm.n : 0);
  if (!act.empty())
    LGS_CUDA(cudaMemcpyAsync(act.data(), tape->vb.active, act.size(), cudaMemcpyDeviceToHost, ctx->stream));
  LGS_CUDA(cudaStreamSynchronize(ctx->stream));
  int64_t vis = 0, mx = 0, pairs = 0, listed = 0, active = 0;
  for (uint8_t a : act) active += a != 0;
  for (uint32_t v : tiles) {
    vis += v != 0;
    pairs += v;
  }
  for (const uint2& r : ranges) {
    mx = std::max<int64_t>(mx, (int64_t)r.y - (int64_t)r.x);
    listed += (int64_t)r.y - (int64_t)r.x;
  }
  st->visible = vis;
  st->pairs = pairs;
  st->tiles = tape->ntiles;
  st->max_tile_list = mx;
  st->listed = listed;
  st->active = tape->vb.active ? active : vis;
  st->host_rows = tape->host_rows_in_place ? st->active : 0;
  return LGS_OK;
}

LGS_API lgs_status lgs_saved_work(const lgs_saved* tape, int64_t* evaluated, int64_t* contributed) {
  if (!tape) return fail(LGS_EINVAL, "NULL argument");
  lgs_ctx* ctx = tape->ctx;
  LGS_CUDA(cudaSetDevice(ctx->device));
  if (!tape->ps.work) return fail(LGS_EINVAL, "work counters are collected only while profiling (lgs_ctx_profile)");
  if (tape->bwd_fused) return fail(LGS_EINVAL, "the fused forward+backward kernel does not collect work counters");
  std::vector<uint2> w((size_t)tape->cam.W * tape->cam.H);
  LGS_CUDA(cudaMemcpyAsync(w.data(), tape->ps.work, sizeof(uint2) * w.size(), cudaMemcpyDeviceToHost, ctx->stream));
  LGS_CUDA(cudaStreamSynchronize(ctx->stream));
  int64_t e = 0, c = 0;
  for (const uint2& x : w) {
    e += x.x;
    c += x.y;
  }
  if (evaluated) *evaluated = e;
  if (contributed) *contributed = c;
  return LGS_OK;
}

LGS_API const char* lgs_phase_name(int32_t phase) {
  static const char* names[LGS_PHASE_COUNT] = {"preprocess", "depth_sort_scan", "duplicate_keys", "tile_sort_ranges",
                                               "blend_fwd", "blend_bwd", "preprocess_bwd", "map_upload",
                                               "mapping_loss", "adam", "allreduce", "coverage", "grad_zero"};
  return (phase >= 0 && phase < LGS_PHASE_COUNT) ? names[phase] : "?";
}

LGS_API lgs_status lgs_ctx_profile(lgs_ctx* ctx, int32_t enable) {
  if (!ctx) return fail(LGS_EINVAL, "ctx is NULL");
  ctx->profiling = enable != 0;
  return LGS_OK;
}

LGS_API lgs_status lgs_ctx_phase_times(lgs_ctx* ctx, double* ms, int64_t* counts, int32_t reset) {
  if (!ctx) return fail(LGS_EINVAL, "ctx is NULL");
  LGS_CUDA(cudaSetDevice(ctx->device));
  for (auto& m : ctx->marks) {
    LGS_CUDA(cudaEventSynchronize(m.b));
    float t = 0.f;
    LGS_CUDA(cudaEventElapsedTime(&t, m.a, m.b));
    ctx->phase_ms[m.phase] += t;
    ctx->phase_n[m.phase] += 1;
    ctx->event_pool.push_back(m.a);
    ctx->event_pool.push_back(m.b);
  }
  ctx->marks.clear();
  for (int i = 0; i < LGS_PHASE_COUNT; ++i) {
    if (ms) ms[i] = ctx->phase_ms[i];
    if (counts) counts[i] = ctx->phase_n[i];
    if (reset) {
      ctx->phase_ms[i] = 0.0;
      ctx->phase_n[i] = 0;
    }
  }
  return LGS_OK;
}

LGS_API lgs_status lgs_saved_destroy(lgs_saved* tape) {
  if (tape) free_saved(tape);
  return LGS_OK;
}

// -------------------------------------------------------------------------------------------
// debug / parity exports
// -------------------------------------------------------------------------------------------
LGS_API lgs_status lgs_debug_projected(lgs_ctx* ctx, const lgs_saved* t, uint8_t* visible, float* u, float* v,
                                       float* depth, float* conic, float* radius, int32_t* bbox, float* opacity,
                                       float* color) {
  if (!ctx || !t) return fail(LGS_EINVAL, "NULL argument");
  LGS_CUDA(cudaSetDevice(ctx->device));
  const size_t n = (size_t)t->dm.n;
  std::vector<float4> r0(n), r1(n), col(n);
  std::vector<uint2> rect(n);
  std::vector<uint32_t> tiles(n);
  cudaStream_t s = ctx->stream;
  if (n) {
    if (t->vb.active) launch_colors(t->dm, t->cam, t->vb, s);  // layered: K1 left colours to the listing
    LGS_CUDA(cudaMemcpyAsync(r0.data(), t->vb.rec0, sizeof(float4) * n, cudaMemcpyDeviceToHost, s));
    LGS_CUDA(cudaMemcpyAsync(r1.data(), t->vb.rec1, sizeof(float4) * n, cudaMemcpyDeviceToHost, s));
    LGS_CUDA(cudaMemcpyAsync(col.data(), t->vb.color, sizeof(float4) * n, cudaMemcpyDeviceToHost, s));
    LGS_CUDA(cudaMemcpyAsync(rect.data(), t->vb.rect, sizeof(uint2) * n, cudaMemcpyDeviceToHost, s));
    LGS_CUDA(cudaMemcpyAsync(tiles.data(), t->vb.tiles, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, s));
  }
  LGS_CUDA(cudaStreamSynchronize(s));
  for (size_t i = 0; i < n; ++i) {
    if (tiles[i] == 0) {  // K1 leaves a culled Gaussian's records unwritten: report zeros
      r0[i] = r1[i] = col[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      rect[i] = make_uint2(0u, 0u);
    }
    if (visible) visible[i] = tiles[i] != 0;
    if (u) u[i] = r0[i].x;
    if (v) v[i] = r0[i].y;
    if (depth) depth[i] = r0[i].z;
    if (opacity) opacity[i] = r0[i].w;
    if (conic) { conic[i * 3] = r1[i].x; conic[i * 3 + 1] = r1[i].y; conic[i * 3 + 2] = r1[i].z; }
    if (radius) radius[i] = r1[i].w;
    if (bbox) {
      bbox[i * 4 + 0] = (int32_t)(rect[i].x & 0xffffu);
      bbox[i * 4 + 1] = (int32_t)(rect[i].x >> 16);
      bbox[i * 4 + 2] = (int32_t)(rect[i].y & 0xffffu);
      bbox[i * 4 + 3] = (int32_t)(rect[i].y >> 16);
    }
    if (color) { color[i * 3] = col[i].x; color[i * 3 + 1] = col[i].y; color[i * 3 + 2] = col[i].z; }
  }
  return LGS_OK;
}

LGS_API lgs_status lgs_debug_tile_keys(lgs_ctx* ctx, const lgs_saved* t, uint64_t* keys, uint32_t* vals,
                                       uint32_t* ranges) {
  if (!ctx || !t) return fail(LGS_EINVAL, "NULL argument");
  LGS_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const size_t nv = (size_t)t->vals_count, n = (size_t)t->dm.n;
  std::vector<uint32_t> v32(nv);
  std::vector<float4> r0(n);
  std::vector<uint2> rg((size_t)t->ntiles);
  if (nv) LGS_CUDA(cudaMemcpyAsync(v32.data(), t->vals, sizeof(uint32_t) * nv, cudaMemcpyDeviceToHost, s));
  if (n) LGS_CUDA(cudaMemcpyAsync(r0.data(), t->vb.rec0, sizeof(float4) * n, cudaMemcpyDeviceToHost, s));
  LGS_CUDA(cudaMemcpyAsync(rg.data(), t->ranges, sizeof(uint2) * t->ntiles, cudaMemcpyDeviceToHost, s));
  LGS_CUDA(cudaStreamSynchronize(s));
  // tile lists concatenated in tile order (with the depth-layered binning the lists of saturated
  // tiles are prefixes and the regions of the two passes are not contiguous)
  size_t o = 0;
  for (size_t tt = 0; tt < rg.size(); ++tt) {
    const uint32_t b = (uint32_t)o;
    for (uint32_t i = rg[tt].x; i < rg[tt].y; ++i, ++o) {
      uint32_t db;
      std::memcpy(&db, &r0[v32[i]].z, 4);
      if (keys) keys[o] = ((uint64_t)tt << 32) | db;
      if (vals) vals[o] = v32[i];
    }
    if (ranges) {
      ranges[2 * tt] = b;
      ranges[2 * tt + 1] = (uint32_t)o;
    }
  }
  return LGS_OK;
}

LGS_API lgs_status lgs_debug_pixel_state(lgs_ctx* ctx, const lgs_saved* t, float* final_t, uint32_t* n_contrib) {
  if (!ctx || !t) return fail(LGS_EINVAL, "NULL argument");
  LGS_CUDA(cudaSetDevice(ctx->device));
  const size_t npix = (size_t)t->cam.W * t->cam.H;
  if (final_t)
    LGS_CUDA(cudaMemcpyAsync(final_t, t->ps.final_t, sizeof(float) * npix, cudaMemcpyDeviceToHost, ctx->stream));
  if (n_contrib)
    LGS_CUDA(cudaMemcpyAsync(n_contrib, t->ps.n_contrib, sizeof(uint32_t) * npix, cudaMemcpyDeviceToHost, ctx->stream));
  LGS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LGS_OK;
}


// -------------------------------------------------------------------------------------------
// multi-view mapping batches: NCCL all-reduce of the per-Gaussian gradients
// -------------------------------------------------------------------------------------------
#define LGS_NCCL(call)                                                                     \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess) return fail(LGS_ECUDA, "%s: %s", #call, nc->GetErrorString(r_)); \
  } while (0)

LGS_API lgs_status lgs_comm_unique_id(lgs_comm_id* id) {
  if (!id) return fail(LGS_EINVAL, "id is NULL");
  std::string err;
  const NcclApi* nc = nccl_api(&err);
  if (!nc) return fail(LGS_ENODEV, "%s", err.c_str());
  static_assert(sizeof(ncclUniqueId) == sizeof(id->bytes), "ncclUniqueId size");
  ncclUniqueId u;
  LGS_NCCL(nc->GetUniqueId(&u));
  std::memcpy(id->bytes, &u, sizeof u);
  return LGS_OK;
}

LGS_API lgs_status lgs_comm_init(lgs_ctx* ctx, int32_t world_size, int32_t rank, const lgs_comm_id* id) {
  if (!ctx || !id) return fail(LGS_EINVAL, "ctx/id is NULL");
  if (world_size < 1 || rank < 0 || rank >= world_size) return fail(LGS_EINVAL, "rank %d of %d", rank, world_size);
  if (ctx->comm) return fail(LGS_EINVAL, "context already has a communicator");
  std::string err;
  const NcclApi* nc = nccl_api(&err);
  if (!nc) return fail(LGS_ENODEV, "%s", err.c_str());
  LGS_CUDA(cudaSetDevice(ctx->device));
  ncclUniqueId u;
  std::memcpy(&u, id->bytes, sizeof u);
  LGS_NCCL(nc->CommInitRank(&ctx->comm, world_size, u, rank));
  ctx->comm_world = world_size;
  ctx->comm_rank = rank;
  return LGS_OK;
}

LGS_API lgs_status lgs_comm_destroy(lgs_ctx* ctx) {
  if (!ctx) return fail(LGS_EINVAL, "ctx is NULL");
  if (!ctx->comm) return LGS_OK;
  const NcclApi* nc = nccl_api(nullptr);
  LGS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (nc) LGS_NCCL(nc->CommDestroy(ctx->comm));
  ctx->comm = nullptr;
  ctx->comm_world = ctx->comm_rank = 0;
  ctx->sparse_cap = 0;
  ctx->sparse_pending = false;
  return LGS_OK;
}

LGS_API lgs_status lgs_allreduce_f32(lgs_ctx* ctx, float* buf, int64_t count) {
  if (!ctx || (!buf && count > 0) || count < 0) return fail(LGS_EINVAL, "bad all-reduce arguments");
  if (!ctx->comm) return fail(LGS_EINVAL, "lgs_comm_init was not called on this context");
  if (count == 0) return LGS_OK;
  const NcclApi* nc = nccl_api(nullptr);
  LGS_NCCL(nc->AllReduce(buf, buf, (size_t)count, ncclFloat32, ncclSum, ctx->comm, ctx->stream));
  return LGS_OK;
}

LGS_API lgs_status lgs_allreduce_grads(lgs_ctx* ctx, const lgs_map* map, lgs_map_grads* grads) {
  if (!ctx || !map || !grads) return fail(LGS_EINVAL, "ctx/map/grads is NULL");
  if (grads->memory != LGS_MEM_DEVICE) return fail(LGS_EINVAL, "all-reduce needs device gradient buffers");
  if (!ctx->comm) return fail(LGS_EINVAL, "lgs_comm_init was not called on this context");
  const NcclApi* nc = nccl_api(nullptr);
  const size_t n = (size_t)map->dm.n, K = (size_t)map->dm.K, d = (size_t)map->dm.d;
  float* ptr[6] = {grads->position, grads->rotation, grads->log_scale, grads->opacity_logit, grads->sh,
                   grads->feature};
  const size_t cnt[6] = {n * 3, n * 4, n * 3, n, n * K * 3, n * d};
  // The usual layout (one flat buffer, renderer.py alloc_grads) is reduced in ONE call; otherwise
  // the attribute buffers are grouped into a single NCCL launch.
  bool flat = true;
  size_t total = 0;
  for (int k = 0; k < 6; ++k) {
    if (!ptr[k] || ptr[0] + total != ptr[k]) flat = flat && (cnt[k] == 0);
    total += cnt[k];
  }
  if (flat && ptr[0]) {
    LGS_NCCL(nc->AllReduce(ptr[0], ptr[0], total, ncclFloat32, ncclSum, ctx->comm, ctx->stream));
    return LGS_OK;
  }
  LGS_NCCL(nc->GroupStart());
  for (int k = 0; k < 6; ++k)
    if (ptr[k] && cnt[k]) {
      ncclResult_t r = nc->AllReduce(ptr[k], ptr[k], cnt[k], ncclFloat32, ncclSum, ctx->comm, ctx->stream);
      if (r != ncclSuccess) {
        nc->GroupEnd();
        return fail(LGS_ECUDA, "ncclAllReduce: %s", nc->GetErrorString(r));
      }
    }
  LGS_NCCL(nc->GroupEnd());
  return LGS_OK;
}
}  // extern "C"

namespace {

// Device scratch of one call, released (stream-ordered) on every exit path.
struct Scratch {
  lgs_ctx* ctx;
  std::vector<uint8_t*> bufs;
  explicit Scratch(lgs_ctx* c) : ctx(c) {}
  template <typename T>
  lgs_status get(T** out, size_t count) {
    LGS_TRY(dalloc(ctx, out, count));
    bufs.push_back(reinterpret_cast<uint8_t*>(*out));
    return LGS_OK;
  }
  ~Scratch() {
    for (uint8_t*& b : bufs) dfree(ctx, b);
  }
};

// The all-gather steps of the row-sparse exchange.  NcclGather: one rank per process over the
// context's communicator; SimGather: `world` ranks simulated in one process (device copies), the
// single-GPU test of the same kernels and host logic (lgs_debug_sparse_reduce_simulated).
struct Gather {
  virtual ~Gather() = default;
  // send[r] (bytes each) of every local rank r -> recv[r] = all ranks' sends back to back
  virtual lgs_status all_gather(const void* const* send, void* const* recv, size_t bytes) = 0;
  // host wait for the stream (the counts), bounded and watching for collective failures
  virtual lgs_status wait() = 0;
};

struct NcclGather final : Gather {
  lgs_ctx* ctx;
  const NcclApi* nc;
  cudaEvent_t until = nullptr;  // wait(): for this event (else the whole stream)
  NcclGather(lgs_ctx* c, const NcclApi* n) : ctx(c), nc(n) {}
  lgs_status abort(const char* why) {
    nc->CommAbort(ctx->comm);  // peers blocked in the collective are released with an error
    ctx->comm = nullptr;
    ctx->comm_world = ctx->comm_rank = 0;
    return fail(LGS_ECUDA, "gradient exchange aborted (communicator destroyed): %s", why);
  }
  lgs_status all_gather(const void* const* send, void* const* recv, size_t bytes) override {
    const ncclResult_t r = nc->AllGather(send[0], recv[0], bytes, ncclUint8, ctx->comm, ctx->stream);
    if (r != ncclSuccess) return abort(nc->GetErrorString(r));
    return LGS_OK;
  }
  lgs_status wait() override {
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      const cudaError_t q = until ? cudaEventQuery(until) : cudaStreamQuery(ctx->stream);
      if (q == cudaSuccess) return LGS_OK;
      if (q != cudaErrorNotReady) return fail(LGS_ECUDA, "%s", cudaGetErrorString(q));
      ncclResult_t ae = ncclSuccess;
      nc->CommGetAsyncError(ctx->comm, &ae);
      if (ae != ncclSuccess && ae != ncclInProgress) return abort(nc->GetErrorString(ae));
      const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0);
      if (ms.count() > ctx->comm_timeout_ms) return abort("timed out waiting for the other ranks");
      std::this_thread::yield();
    }
  }
};

struct SimGather final : Gather {
  lgs_ctx* ctx;
  int world;
  SimGather(lgs_ctx* c, int w) : ctx(c), world(w) {}
  lgs_status all_gather(const void* const* send, void* const* recv, size_t bytes) override {
    for (int r = 0; r < world; ++r)
      for (int q = 0; q < world; ++q)
        LGS_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(recv[r]) + (size_t)q * bytes, send[q], bytes,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
    return LGS_OK;
  }
  lgs_status wait() override {
    LGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return LGS_OK;
  }
};

// The exchange for the local ranks' gradient buffers (one in production, `world` when simulated).
// cap == 0: exact -- the counts are read on the host (one wait) and size the record blocks;
// *dense = true when the rows are not sparse enough and nothing was exchanged (the caller then
// runs the dense all-reduce).  cap > 0: capacity-speculative, no host wait -- record blocks of
// `cap` rows; if some rank has more rows nothing is applied (every rank keeps its own gradient)
// and ovf[0] (device) is set; ovf[1] = the largest row count.
lgs_status sparse_exchange(lgs_ctx* ctx, const lgs_map* map, lgs_map_grads* const* grads, int nlocal, int world,
                           Gather& g, int64_t* rows_max, bool* dense, int64_t cap = 0, uint32_t* ovf = nullptr) {
  cudaStream_t s = ctx->stream;
  const int64_t n = map->dm.n;
  const int width[6] = {3, 4, 3, 1, 3 * map->dm.K, map->dm.d};
  *dense = false;
  if (rows_max) *rows_max = 0;
  std::vector<std::array<float*, 6>> ptr((size_t)nlocal);
  for (int r = 0; r < nlocal; ++r)
    ptr[r] = {grads[r]->position, grads[r]->rotation, grads[r]->log_scale, grads[r]->opacity_logit, grads[r]->sh,
              grads[r]->feature};
  const int R = rows_values(width, ptr[0].data());
  if (n == 0 || R == 0) return LGS_OK;
  Scratch sc(ctx);
  std::vector<uint32_t*> list((size_t)nlocal), cnt((size_t)nlocal);
  for (int r = 0; r < nlocal; ++r) {
    LGS_TRY(sc.get(&list[r], (size_t)n));
    LGS_TRY(sc.get(&cnt[r], (size_t)world + 1));  // [0] own count, [1 ..] all ranks'
    launch_rows_scan(ptr[r].data(), width, n, list[r], cnt[r], s);
  }
  {
    std::vector<const void*> snd((size_t)nlocal);
    std::vector<void*> rcv((size_t)nlocal);
    for (int r = 0; r < nlocal; ++r) {
      snd[r] = cnt[r];
      rcv[r] = cnt[r] + 1;
    }
    LGS_TRY(g.all_gather(snd.data(), rcv.data(), sizeof(uint32_t)));
  }
  int64_t maxc = cap;
  if (cap <= 0) {
    std::vector<uint32_t> counts((size_t)world);
    LGS_CUDA(cudaMemcpyAsync(counts.data(), cnt[0] + 1, sizeof(uint32_t) * world, cudaMemcpyDeviceToHost, s));
    LGS_TRY(g.wait());
    maxc = 0;
    for (uint32_t c : counts) maxc = std::max<int64_t>(maxc, c);
    if (rows_max) *rows_max = maxc;
    if (maxc == 0) return LGS_OK;
    if (maxc * (int64_t)world * (R + 1) * 2 >= n * (int64_t)R) {  // not sparse enough: dense sum
      *dense = true;
      if (rows_max) *rows_max = -1;
      return LGS_OK;
    }
  } else if (ovf) {
    launch_rows_overflow(cnt[0] + 1, world, cap, ovf, s);
  }
  std::vector<float*> send((size_t)nlocal), recv((size_t)nlocal);
  for (int r = 0; r < nlocal; ++r) {
    LGS_TRY(sc.get(&send[r], (size_t)maxc * (R + 1)));
    LGS_TRY(sc.get(&recv[r], (size_t)world * maxc * (R + 1)));
    launch_rows_pack(ptr[r].data(), width, n, list[r], cnt[r], maxc, send[r], s);
  }
  {
    std::vector<const void*> snd(send.begin(), send.end());
    std::vector<void*> rcv(recv.begin(), recv.end());
    LGS_TRY(g.all_gather(snd.data(), rcv.data(), sizeof(float) * (size_t)maxc * (R + 1)));
  }
  for (int r = 0; r < nlocal; ++r) launch_rows_apply(ptr[r].data(), width, n, recv[r], cnt[r] + 1, world, maxc, s);
  LGS_CUDA(cudaGetLastError());
  return LGS_OK;
}

}  // namespace

extern "C" {

LGS_API lgs_status lgs_allreduce_grads_sparse(lgs_ctx* ctx, const lgs_map* map, lgs_map_grads* grads,
                                              int64_t* rows_max) {
  if (!ctx || !map || !grads) return fail(LGS_EINVAL, "ctx/map/grads is NULL");
  if (grads->memory != LGS_MEM_DEVICE) return fail(LGS_EINVAL, "all-reduce needs device gradient buffers");
  if (!ctx->comm) return fail(LGS_EINVAL, "lgs_comm_init was not called on this context");
  LGS_CUDA(cudaSetDevice(ctx->device));
  return guarded([&]() -> lgs_status {
    NcclGather g(ctx, nccl_api(nullptr));
    bool dense = false;
    LGS_TRY(sparse_exchange(ctx, map, &grads, 1, ctx->comm_world, g, rows_max, &dense));
    return dense ? lgs_allreduce_grads(ctx, map, grads) : LGS_OK;
  });
}

LGS_API lgs_status lgs_allreduce_grads_sparse_async(lgs_ctx* ctx, const lgs_map* map, lgs_map_grads* grads) {
  if (!ctx || !map || !grads) return fail(LGS_EINVAL, "ctx/map/grads is NULL");
  if (grads->memory != LGS_MEM_DEVICE) return fail(LGS_EINVAL, "all-reduce needs device gradient buffers");
  if (!ctx->comm) return fail(LGS_EINVAL, "lgs_comm_init was not called on this context");
  if (ctx->sparse_pending) return fail(LGS_EINVAL, "a sparse exchange is pending: call lgs_allreduce_grads_sparse_wait");
  LGS_CUDA(cudaSetDevice(ctx->device));
  return guarded([&]() -> lgs_status {
    NcclGather g(ctx, nccl_api(nullptr));
    bool dense = false;
    int64_t rows = 0;
    if (ctx->sparse_cap <= 0) {  // first exchange: exact sizes (one host wait), then the capacity
      LGS_TRY(sparse_exchange(ctx, map, &grads, 1, ctx->comm_world, g, &rows, &dense));
      if (dense) return lgs_allreduce_grads(ctx, map, grads);
      ctx->sparse_cap = std::max<int64_t>(256, rows + rows / 4);
      return LGS_OK;
    }
    if (!ctx->sparse_ovf_dev) {
      LGS_CUDA(cudaMalloc(&ctx->sparse_ovf_dev, 2 * sizeof(uint32_t)));
      LGS_CUDA(cudaMallocHost(&ctx->sparse_ovf_host, 2 * sizeof(uint32_t)));
      LGS_CUDA(cudaEventCreateWithFlags(&ctx->sparse_done, cudaEventDisableTiming));
    }
    LGS_TRY(sparse_exchange(ctx, map, &grads, 1, ctx->comm_world, g, nullptr, &dense, ctx->sparse_cap,
                            ctx->sparse_ovf_dev));
    LGS_CUDA(cudaMemcpyAsync(ctx->sparse_ovf_host, ctx->sparse_ovf_dev, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                             ctx->stream));
    LGS_CUDA(cudaEventRecord(ctx->sparse_done, ctx->stream));
    ctx->sparse_pending = true;
    return LGS_OK;
  });
}

LGS_API lgs_status lgs_allreduce_grads_sparse_wait(lgs_ctx* ctx, const lgs_map* map, lgs_map_grads* grads,
                                                   int64_t* rows_max) {
  if (!ctx || !map || !grads) return fail(LGS_EINVAL, "ctx/map/grads is NULL");
  if (rows_max) *rows_max = 0;
  if (!ctx->sparse_pending) return LGS_OK;
  LGS_CUDA(cudaSetDevice(ctx->device));
  return guarded([&]() -> lgs_status {
    NcclGather g(ctx, nccl_api(nullptr));
    ctx->sparse_pending = false;
    g.until = ctx->sparse_done;
    LGS_TRY(g.wait());  // bounded, aborts the communicator on a peer failure
    g.until = nullptr;
    const int64_t mx = ctx->sparse_ovf_host[1];
    if (rows_max) *rows_max = mx;
    if (ctx->sparse_ovf_host[0] == 0) return LGS_OK;
    // some rank outgrew the capacity: nothing was applied; exact exchange now, larger capacity
    ctx->sparse_cap = std::max<int64_t>(ctx->sparse_cap * 2, mx + mx / 4);
    bool dense = false;
    LGS_TRY(sparse_exchange(ctx, map, &grads, 1, ctx->comm_world, g, rows_max, &dense));
    return dense ? lgs_allreduce_grads(ctx, map, grads) : LGS_OK;
  });
}

LGS_API lgs_status lgs_debug_sparse_reduce_simulated(lgs_ctx* ctx, const lgs_map* map, lgs_map_grads* const* grads,
                                                     int32_t world, int64_t cap, int64_t* rows_max,
                                                     int32_t* overflowed) {
  if (!ctx || !map || !grads || world < 1 || cap < 0) return fail(LGS_EINVAL, "bad simulated exchange arguments");
  for (int r = 0; r < world; ++r)
    if (!grads[r] || grads[r]->memory != LGS_MEM_DEVICE) return fail(LGS_EINVAL, "device gradient buffers needed");
  LGS_CUDA(cudaSetDevice(ctx->device));
  if (overflowed) *overflowed = 0;
  return guarded([&]() -> lgs_status {
    SimGather g(ctx, world);
    bool dense = false;
    uint32_t* ovf = nullptr;
    if (cap > 0) LGS_TRY(dalloc(ctx, &ovf, 2));
    const lgs_status st = sparse_exchange(ctx, map, grads, world, world, g, rows_max, &dense, cap, ovf);
    if (ovf) {
      uint32_t h[2] = {0, 0};
      cudaMemcpyAsync(h, ovf, sizeof h, cudaMemcpyDeviceToHost, ctx->stream);
      cudaStreamSynchronize(ctx->stream);
      dfree(ctx, ovf);
      if (overflowed) *overflowed = (int32_t)h[0];
      if (rows_max) *rows_max = h[1];
    }
    LGS_TRY(st);
    if (dense) return fail(LGS_EINVAL, "rows not sparse: the exchange would take the dense all-reduce");
    return LGS_OK;
  });
}

LGS_API lgs_status lgs_comm_set_timeout(lgs_ctx* ctx, int64_t ms) {
  if (!ctx || ms <= 0) return fail(LGS_EINVAL, "bad timeout");
  ctx->comm_timeout_ms = ms;
  return LGS_OK;
}
#undef LGS_NCCL

}  // extern "C"

// -------------------------------------------------------------------------------------------
// Adam step on the resident map and the map download
// -------------------------------------------------------------------------------------------
namespace {

MapParams map_params(lgs_map* m) {
  MapParams p;
  p.n = m->dm.n; p.d = m->dm.d; p.dp = m->dm.dp; p.K = m->dm.K;
  p.pos_opa = m->pos_opa; p.rot = m->rot; p.scale = m->scale; p.sh = m->sh; p.feat = m->feat;
  return p;
}

void free_adam(lgs_adam* a) {
  lgs_ctx* ctx = a->ctx;
  cudaSetDevice(ctx->device);
  dfree(ctx, a->m_po); dfree(ctx, a->m_rot); dfree(ctx, a->m_sc); dfree(ctx, a->m_sh); dfree(ctx, a->m_ft);
  dfree(ctx, a->v_po); dfree(ctx, a->v_rot); dfree(ctx, a->v_sc); dfree(ctx, a->v_sh); dfree(ctx, a->v_ft);
  delete a;
  ctx_release(ctx);
}

}  // namespace

extern "C" {

LGS_API lgs_adam_config lgs_adam_config_default(void) {
  lgs_adam_config c;
  c.lr_position = 1.6e-4;
  c.lr_rotation = 1e-3;
  c.lr_log_scale = 5e-3;
  c.lr_opacity = 5e-2;
  c.lr_color = 2.5e-3;
  c.lr_sh_rest = 2.5e-3 / 20.0;
  c.lr_feature = 2.5e-3;
  c.beta1 = 0.9;
  c.beta2 = 0.999;
  c.eps = 1e-8;
  return c;
}

LGS_API lgs_status lgs_adam_create(lgs_ctx* ctx, const lgs_map* map, const lgs_adam_config* cfg, lgs_adam** out) {
  if (!ctx || !map || !out) return fail(LGS_EINVAL, "ctx/map/out is NULL");
  if (map->mapped) return fail(LGS_EINVAL, "Adam needs a device map (this one is LGS_MEM_HOST_MAPPED)");
  *out = nullptr;
  const lgs_adam_config c = cfg ? *cfg : lgs_adam_config_default();
  if (!(c.beta1 >= 0.0 && c.beta1 < 1.0 && c.beta2 >= 0.0 && c.beta2 < 1.0 && c.eps > 0.0))
    return fail(LGS_EINVAL, "Adam: need 0 <= beta < 1 and eps > 0");
  LGS_CUDA(cudaSetDevice(ctx->device));
  lgs_adam* a = new lgs_adam();
  a->ctx = ctx;
  ctx->refs++;
  a->n = map->dm.n; a->d = map->dm.d; a->dp = map->dm.dp; a->K = map->dm.K;
  a->cfg = c;
  const size_t n = (size_t)a->n, ks = n * a->K * 3, fs = n * (a->dp > 0 ? a->dp : 1);
  lgs_status st = LGS_OK;
  if ((st = dalloc(ctx, &a->m_po, n)) != LGS_OK || (st = dalloc(ctx, &a->m_rot, n)) != LGS_OK ||
      (st = dalloc(ctx, &a->m_sc, n)) != LGS_OK || (st = dalloc(ctx, &a->m_sh, ks)) != LGS_OK ||
      (st = dalloc(ctx, &a->m_ft, fs)) != LGS_OK || (st = dalloc(ctx, &a->v_po, n)) != LGS_OK ||
      (st = dalloc(ctx, &a->v_rot, n)) != LGS_OK || (st = dalloc(ctx, &a->v_sc, n)) != LGS_OK ||
      (st = dalloc(ctx, &a->v_sh, ks)) != LGS_OK || (st = dalloc(ctx, &a->v_ft, fs)) != LGS_OK) {
    free_adam(a);
    return st;
  }
  cudaStream_t s = ctx->stream;
  cudaMemsetAsync(a->m_po, 0, sizeof(float4) * n, s); cudaMemsetAsync(a->v_po, 0, sizeof(float4) * n, s);
  cudaMemsetAsync(a->m_rot, 0, sizeof(float4) * n, s); cudaMemsetAsync(a->v_rot, 0, sizeof(float4) * n, s);
  cudaMemsetAsync(a->m_sc, 0, sizeof(float4) * n, s); cudaMemsetAsync(a->v_sc, 0, sizeof(float4) * n, s);
  cudaMemsetAsync(a->m_sh, 0, sizeof(float) * ks, s); cudaMemsetAsync(a->v_sh, 0, sizeof(float) * ks, s);
  cudaMemsetAsync(a->m_ft, 0, sizeof(float) * fs, s); cudaMemsetAsync(a->v_ft, 0, sizeof(float) * fs, s);
  LGS_CUDA(cudaGetLastError());
  *out = a;
  return LGS_OK;
}

LGS_API lgs_status lgs_adam_destroy(lgs_adam* adam) {
  if (adam) free_adam(adam);
  return LGS_OK;
}

LGS_API int64_t lgs_adam_steps(const lgs_adam* adam) { return adam ? adam->step : -1; }

LGS_API lgs_status lgs_adam_step(lgs_ctx* ctx, lgs_adam* a, lgs_map* map, const lgs_map_grads* grads) {
  if (!ctx || !a || !map || !grads) return fail(LGS_EINVAL, "ctx/adam/map/grads is NULL");
  if (map->mapped) return fail(LGS_EINVAL, "Adam needs a device map (this one is LGS_MEM_HOST_MAPPED)");
  if (a->n != map->dm.n || a->d != map->dm.d || a->K != map->dm.K)
    return fail(LGS_EINVAL, "Adam state was created for a different map shape");
  if (grads->memory != LGS_MEM_DEVICE) return fail(LGS_EINVAL, "Adam step needs device gradients");
  if (!grads->position || !grads->rotation || !grads->log_scale || !grads->opacity_logit || !grads->sh ||
      (a->d > 0 && !grads->feature))
    return fail(LGS_EINVAL, "Adam step needs every gradient group");
  LGS_CUDA(cudaSetDevice(ctx->device));
  MapParams p = map_params(map), m = p, v = p;
  m.pos_opa = a->m_po; m.rot = a->m_rot; m.scale = a->m_sc; m.sh = a->m_sh; m.feat = a->m_ft;
  v.pos_opa = a->v_po; v.rot = a->v_rot; v.scale = a->v_sc; v.sh = a->v_sh; v.feat = a->v_ft;
  GradIn g;
  g.position = grads->position; g.rotation = grads->rotation; g.log_scale = grads->log_scale;
  g.opacity = grads->opacity_logit; g.sh = grads->sh; g.feature = grads->feature;
  const lgs_adam_config& c = a->cfg;
  AdamLr lr{(float)c.lr_position, (float)c.lr_rotation, (float)c.lr_log_scale, (float)c.lr_opacity,
            (float)c.lr_color, (float)c.lr_sh_rest, (float)c.lr_feature};
  ++a->step;
  {
    PhaseScope ph(ctx, PH_ADAM);
    launch_adam(p, m, v, g, 0, a->n, lr, c.beta1, c.beta2, c.eps, a->step, ctx->stream);
  }
  ctx->launches += a->n > 0 ? 2 : 0;
  LGS_CUDA(cudaGetLastError());
  return LGS_OK;
}

LGS_API lgs_status lgs_map_download(lgs_ctx* ctx, const lgs_map* map, lgs_gaussians* dst) {
  if (!ctx || !map || !dst) return fail(LGS_EINVAL, "ctx/map/dst is NULL");
  if (map->mapped) return fail(LGS_EINVAL, "lgs_map_download: the map is LGS_MEM_HOST_MAPPED (its source is the host copy)");
  if (dst->n != map->dm.n || dst->feature_dim != map->dm.d || dst->sh_degree != map->dm.deg)
    return fail(LGS_EINVAL, "lgs_map_download: destination shape differs from the map");
  LGS_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const size_t n = (size_t)map->dm.n;
  const size_t sz[6] = {n * 3, n * 4, n * 3, n, n * map->dm.K * 3, n * map->dm.d};
  float* outs[6] = {(float*)dst->positions, (float*)dst->rotations, (float*)dst->log_scales,
                    (float*)dst->opacity_logits, (float*)dst->sh, (float*)dst->features};
  float* dev[6] = {};
  const bool host = dst->memory == LGS_MEM_HOST;
  float* stage = nullptr;
  if (host) {
    // staged segments start on 16-byte boundaries (the rotation rows are stored as float4)
    size_t off[7] = {0};
    for (int k = 0; k < 6; ++k) off[k + 1] = off[k] + ((sz[k] + 3) & ~(size_t)3);
    LGS_TRY(dalloc(ctx, &stage, off[6]));
    for (int k = 0; k < 6; ++k) dev[k] = outs[k] ? stage + off[k] : nullptr;
  } else {
    for (int k = 0; k < 6; ++k) dev[k] = outs[k];
  }
  launch_unpack_map(map_params(const_cast<lgs_map*>(map)), dev[0], dev[1], dev[2], dev[3], dev[4],
                    map->dm.d > 0 ? dev[5] : nullptr, s);
  ctx->launches += n > 0 ? 1 : 0;
  if (host) {
    for (int k = 0; k < 6; ++k)
      if (outs[k] && sz[k]) LGS_CUDA(cudaMemcpyAsync(outs[k], dev[k], sizeof(float) * sz[k], cudaMemcpyDeviceToHost, s));
    dfree(ctx, stage);
    LGS_CUDA(cudaStreamSynchronize(s));
  }
  LGS_CUDA(cudaGetLastError());
  return LGS_OK;
}

}  // extern "C"

// -------------------------------------------------------------------------------------------
// LEGOMAP1 files (gaussian_map.cpp:196-259)
// -------------------------------------------------------------------------------------------
namespace {

constexpr char kMapMagic[8] = {'L', 'E', 'G', 'O', 'M', 'A', 'P', '1'};

struct MapFileHeader {
  uint32_t dim = 0;
  uint64_t count = 0;
};

lgs_status read_header(std::ifstream& is, const char* path, MapFileHeader* h) {
  char magic[8];
  is.read(magic, sizeof magic);
  if (!is || std::memcmp(magic, kMapMagic, sizeof magic) != 0) return fail(LGS_EIO, "bad map file magic: %s", path);
  is.read(reinterpret_cast<char*>(&h->dim), sizeof h->dim);
  if (!is) return fail(LGS_EIO, "map file truncated reading feature dim");
  if (h->dim == 0 || h->dim > 4096) return fail(LGS_EIO, "map file declares unreasonable feature dim");
  is.read(reinterpret_cast<char*>(&h->count), sizeof h->count);
  if (!is) return fail(LGS_EIO, "map file truncated reading count");
  return LGS_OK;
}

// The byte size a file of `count` records needs; when the file is shorter, the error the
// record-by-record reader (gaussian_map.cpp:187-192, read_pod) would raise at the first missing
// field -- checked before anything is sized from the header's count.
lgs_status check_map_file_size(std::ifstream& is, const char* path, const MapFileHeader& h) {
  const std::streampos here = is.tellg();
  is.seekg(0, std::ios::end);
  const uint64_t size = (uint64_t)is.tellg();
  is.seekg(here);
  if (!is) return fail(LGS_EIO, "cannot size map file: %s", path);
  const uint64_t rec = 4ull * (14 + h.dim) + 8ull, body = size > 20 ? size - 20 : 0;
  if (h.count <= body / rec) return LGS_OK;
  const uint64_t got = body % rec;  // bytes of the first incomplete record
  const char* what[] = {"position", "rotation", "scale", "opacity", "color", "feature", "anchor"};
  const uint64_t off[] = {0, 12, 28, 40, 44, 56, 56 + 4ull * h.dim};
  int f = 0;
  while (f < 6 && got >= off[f + 1]) ++f;
  return fail(LGS_EIO, "map file truncated reading %s", what[f]);
}

}  // namespace

extern "C" {

LGS_API lgs_status lgs_map_file_info(const char* path, int32_t* feature_dim, int64_t* count) {
  if (!path) return fail(LGS_EINVAL, "path is NULL");
  std::ifstream is(path, std::ios::binary);
  if (!is) return fail(LGS_EIO, "cannot open map file: %s", path);
  MapFileHeader h;
  LGS_TRY(read_header(is, path, &h));
  LGS_TRY(check_map_file_size(is, path, h));
  if (feature_dim) *feature_dim = (int32_t)h.dim;
  if (count) *count = (int64_t)h.count;
  return LGS_OK;
}

LGS_API lgs_status lgs_map_file_read(const char* path, int32_t expected_dim, lgs_gaussians* dst, uint64_t* anchors) {
  return guarded([&]() -> lgs_status {
    if (!path || !dst) return fail(LGS_EINVAL, "path/dst is NULL");
    if (dst->memory != LGS_MEM_HOST) return fail(LGS_EINVAL, "lgs_map_file_read fills host buffers");
    std::ifstream is(path, std::ios::binary);
    if (!is) return fail(LGS_EIO, "cannot open map file: %s", path);
    MapFileHeader h;
    LGS_TRY(read_header(is, path, &h));
    if (expected_dim > 0 && (int32_t)h.dim != expected_dim)
      return fail(LGS_EIO, "map feature dimension mismatch: file has %u, expected %d", h.dim, expected_dim);
    LGS_TRY(check_map_file_size(is, path, h));
    if (dst->n != (int64_t)h.count || dst->feature_dim != (int32_t)h.dim || dst->sh_degree != 0)
      return fail(LGS_EINVAL, "destination must hold %llu Gaussians of dim %u, sh_degree 0",
                  (unsigned long long)h.count, h.dim);
    const uint32_t d = h.dim;
    const size_t rec = sizeof(float) * (3 + 4 + 3 + 1 + 3 + d) + sizeof(uint64_t);
    std::vector<char> buf(rec);
    const char* what[] = {"position", "rotation", "scale", "opacity", "color", "feature", "anchor"};
    const size_t off[] = {0, 12, 28, 40, 44, 56, 56 + 4 * (size_t)d};
    float* pos = (float*)dst->positions;
    float* rot = (float*)dst->rotations;
    float* ls = (float*)dst->log_scales;
    float* op = (float*)dst->opacity_logits;
    float* col = (float*)dst->sh;
    float* ft = (float*)dst->features;
    for (uint64_t i = 0; i < h.count; ++i) {
      is.read(buf.data(), (std::streamsize)rec);
      if (!is) {  // name the first field that ran out, like read_pod (gaussian_map.cpp:187-192)
        const size_t got = (size_t)is.gcount();
        int f = 0;
        while (f < 6 && got >= off[f + 1]) ++f;
        return fail(LGS_EIO, "map file truncated reading %s", what[f]);
      }
      float v[14];
      std::memcpy(v, buf.data(), sizeof v);
      for (int a = 0; a < 3; ++a) pos[i * 3 + a] = v[a];
      // file order w,x,y,z -> Eigen storage x,y,z,w; renormalize only when off-unit (gaussian_map.cpp:21-23)
      double qw = v[3], qx = v[4], qy = v[5], qz = v[6];
      const double nrm = std::sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
      if (std::abs(nrm - 1.0) > 1e-6 && nrm > 0.0) {
        qw /= nrm; qx /= nrm; qy /= nrm; qz /= nrm;
      }
      rot[i * 4 + 0] = (float)qx; rot[i * 4 + 1] = (float)qy; rot[i * 4 + 2] = (float)qz; rot[i * 4 + 3] = (float)qw;
      for (int a = 0; a < 3; ++a) ls[i * 3 + a] = v[7 + a];
      op[i] = v[10];
      for (int a = 0; a < 3; ++a) col[i * 3 + a] = v[11 + a];
      for (uint32_t c = 0; c < d; ++c) {
        float f;
        std::memcpy(&f, buf.data() + 56 + 4 * (size_t)c, 4);
        ft[(size_t)c * h.count + i] = f;  // features [d][N]
      }
      if (anchors) std::memcpy(&anchors[i], buf.data() + off[6], sizeof(uint64_t));
    }
    return LGS_OK;
  });
}

LGS_API lgs_status lgs_map_file_write(const char* path, const lgs_gaussians* src, const uint64_t* anchors) {
  return guarded([&]() -> lgs_status {
    if (!path || !src) return fail(LGS_EINVAL, "path/src is NULL");
    if (src->n < 0 || src->feature_dim <= 0 || src->feature_dim > 4096)
      return fail(LGS_EINVAL, "LEGOMAP1 needs 1 <= feature_dim <= 4096");
    if (src->sh_degree != 0) return fail(LGS_EINVAL, "LEGOMAP1 stores SH degree 0 colour only");
    const size_t n = (size_t)src->n, d = (size_t)src->feature_dim;
    if (n > 0 && (!src->positions || !src->rotations || !src->log_scales || !src->opacity_logits || !src->sh ||
                  !src->features))
      return fail(LGS_EINVAL, "a map attribute pointer is NULL");
    // device sources are copied out first
    std::vector<float> hp, hr, hl, ho, hc, hf;
    const float *pos = (const float*)src->positions, *rot = (const float*)src->rotations,
                *ls = (const float*)src->log_scales, *op = (const float*)src->opacity_logits,
                *col = (const float*)src->sh, *ft = (const float*)src->features;
    if (src->memory == LGS_MEM_DEVICE && n > 0) {
      auto pull = [&](std::vector<float>& v, const float*& p, size_t count) -> lgs_status {
        v.resize(count);
        LGS_CUDA(cudaMemcpy(v.data(), p, sizeof(float) * count, cudaMemcpyDeviceToHost));
        p = v.data();
        return LGS_OK;
      };
      LGS_TRY(pull(hp, pos, n * 3)); LGS_TRY(pull(hr, rot, n * 4)); LGS_TRY(pull(hl, ls, n * 3));
      LGS_TRY(pull(ho, op, n)); LGS_TRY(pull(hc, col, n * 3)); LGS_TRY(pull(hf, ft, n * d));
    }
    std::ofstream os(path, std::ios::binary);
    if (!os) return fail(LGS_EIO, "cannot open map file for writing: %s", path);
    os.write(kMapMagic, sizeof kMapMagic);
    const uint32_t dim = (uint32_t)d;
    const uint64_t count = n;
    os.write(reinterpret_cast<const char*>(&dim), sizeof dim);
    os.write(reinterpret_cast<const char*>(&count), sizeof count);
    std::vector<char> buf(sizeof(float) * (14 + d) + sizeof(uint64_t));
    for (size_t i = 0; i < n; ++i) {
      float v[14];
      for (int a = 0; a < 3; ++a) v[a] = pos[i * 3 + a];
      v[3] = rot[i * 4 + 3]; v[4] = rot[i * 4 + 0]; v[5] = rot[i * 4 + 1]; v[6] = rot[i * 4 + 2];  // w,x,y,z
      for (int a = 0; a < 3; ++a) v[7 + a] = ls[i * 3 + a];
      v[10] = op[i];
      for (int a = 0; a < 3; ++a) v[11 + a] = col[i * 3 + a];
      std::memcpy(buf.data(), v, sizeof v);
      for (size_t c = 0; c < d; ++c) std::memcpy(buf.data() + 56 + 4 * c, &ft[c * n + i], 4);
      const uint64_t an = anchors ? anchors[i] : 0;
      std::memcpy(buf.data() + 56 + 4 * d, &an, sizeof an);
      os.write(buf.data(), (std::streamsize)buf.size());
    }
    if (!os) return fail(LGS_EIO, "failed writing map file: %s", path);
    return LGS_OK;
  });
}

LGS_API lgs_status lgs_map_load(lgs_ctx* ctx, const char* path, int32_t expected_dim, lgs_map** out) {
  return guarded([&]() -> lgs_status {
    if (!ctx || !out) return fail(LGS_EINVAL, "ctx/out is NULL");
    *out = nullptr;
    int32_t dim = 0;
    int64_t count = 0;
    LGS_TRY(lgs_map_file_info(path, &dim, &count));
    if (expected_dim > 0 && dim != expected_dim)
      return fail(LGS_EIO, "map feature dimension mismatch: file has %d, expected %d", dim, expected_dim);
    if (dim > LGS_MAX_FEATURE_DIM)
      return fail(LGS_EINVAL, "feature dim %d exceeds the rasterizer's %d", dim, LGS_MAX_FEATURE_DIM);
    const size_t n = (size_t)count;
    std::vector<float> pos(n * 3), rot(n * 4), ls(n * 3), op(n), col(n * 3), ft(n * dim);
    lgs_gaussians g{};
    g.n = count; g.feature_dim = dim; g.sh_degree = 0;
    g.positions = pos.data(); g.rotations = rot.data(); g.log_scales = ls.data(); g.opacity_logits = op.data();
    g.sh = col.data(); g.features = ft.data(); g.memory = LGS_MEM_HOST;
    LGS_TRY(lgs_map_file_read(path, expected_dim, &g, nullptr));
    return lgs_map_create(ctx, &g, out);  // host source: synchronizes before the vectors go away
  });
}

LGS_API lgs_status lgs_map_save(lgs_ctx* ctx, const lgs_map* map, const char* path, const uint64_t* anchors) {
  return guarded([&]() -> lgs_status {
    if (!ctx || !map) return fail(LGS_EINVAL, "ctx/map is NULL");
    if (map->dm.deg != 0) return fail(LGS_EINVAL, "LEGOMAP1 stores SH degree 0 colour only");
    const size_t n = (size_t)map->dm.n, d = (size_t)map->dm.d;
    std::vector<float> pos(n * 3), rot(n * 4), ls(n * 3), op(n), col(n * 3), ft(n * d);
    lgs_gaussians g{};
    g.n = map->dm.n; g.feature_dim = map->dm.d; g.sh_degree = 0;
    g.positions = pos.data(); g.rotations = rot.data(); g.log_scales = ls.data(); g.opacity_logits = op.data();
    g.sh = col.data(); g.features = ft.data(); g.memory = LGS_MEM_HOST;
    LGS_TRY(lgs_map_download(ctx, map, &g));
    return lgs_map_file_write(path, &g, anchors);
  });
}

// ---- map pruning (csrc/prune.cu) ---------------------------------------------
LGS_API lgs_prune_config lgs_prune_config_default(void) {
  lgs_prune_config c;
  c.k_neighbors = 8;  // SPEC.md:476 defaults
  c.tau_dist = 0.02;
  c.tau_sim = 0.9;
  c.alpha_min = 0.05;
  c.scale_max = 0.5;
  return c;
}

}  // extern "C"

namespace {

lgs_status prune_setup(lgs_ctx* ctx, const lgs_map* map, const lgs_prune_config* cfg_in, int32_t memory,
                       PruneParams* pp, PruneIn* in) {
  if (!ctx || !map) return fail(LGS_EINVAL, "ctx/map is NULL");
  const lgs_prune_config c = cfg_in ? *cfg_in : lgs_prune_config_default();
  if (c.k_neighbors < 1 || c.k_neighbors > 32) return fail(LGS_EINVAL, "k_neighbors %d out of range [1, 32]", c.k_neighbors);
  if (!(c.tau_dist > 0.0) || !std::isfinite(c.tau_dist)) return fail(LGS_EINVAL, "tau_dist must be > 0");
  if (!(c.tau_sim > -1.0 && c.tau_sim <= 1.0)) return fail(LGS_EINVAL, "tau_sim must be in (-1, 1]");
  if (memory != LGS_MEM_HOST && memory != LGS_MEM_DEVICE) return fail(LGS_EINVAL, "bad memory kind for the flags");
  *pp = PruneParams{c.k_neighbors, c.tau_dist, c.tau_sim, c.alpha_min, c.scale_max};
  *in = PruneIn{map->pos_opa, map->scale, map->feat, map->dm.n, map->dm.d, map->dm.dp};
  LGS_CUDA(cudaSetDevice(ctx->device));
  if (map->mapped && map->feat_src && map->dm.n > 0)  // host-mapped: features are gathered lazily
    launch_gather_features(map->feat_src, map->feat, map->dm.n, map->dm.d, map->dm.dp, ctx->stream);
  return LGS_OK;
}

// flags produced on the device, handed out in `memory`
lgs_status flags_out(lgs_ctx* ctx, const uint8_t* dflags, uint8_t* flags, int32_t memory, int64_t n) {
  if (!flags || memory == LGS_MEM_DEVICE || n == 0) return LGS_OK;
  LGS_CUDA(cudaMemcpyAsync(flags, dflags, (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->bytes_d2h += n;
  LGS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LGS_OK;
}

lgs_status language_flags(lgs_ctx* ctx, const PruneIn& in, const PruneParams& pp, uint8_t* dflags, int64_t* count) {
  uint8_t* scratch = nullptr;
  LGS_TRY(dalloc(ctx, &scratch, prune_scratch_bytes(in.n)));
  int64_t cand = 0, rounds = 0;
  const cudaError_t e = run_language_redundant(in, pp, dflags, scratch, count, &cand, &rounds, ctx->stream);
  dfree(ctx, scratch);
  if (e != cudaSuccess) return fail(LGS_ECUDA, "language-redundancy sweep: %s", cudaGetErrorString(e));
  ctx->prune_candidates = cand;
  ctx->prune_rounds = rounds;
  ctx->launches += 6 + 2 * rounds;
  return LGS_OK;
}

lgs_status geometric_flags(lgs_ctx* ctx, const PruneIn& in, const PruneParams& pp, uint8_t* dflags, int64_t* count) {
  uint64_t* scratch = nullptr;
  LGS_TRY(dalloc(ctx, &scratch, 1));
  const cudaError_t e = run_geometric(in, pp, dflags, scratch, count, ctx->stream);
  dfree(ctx, scratch);
  if (e != cudaSuccess) return fail(LGS_ECUDA, "geometric pruning rule: %s", cudaGetErrorString(e));
  ctx->launches++;
  return LGS_OK;
}

// allocate the compacted copy of buffer `p` (rows of `width_floats` floats); swapped in later
struct Swap {
  void** slot;
  void* fresh;
};
template <typename T>
lgs_status compact_alloc(lgs_ctx* ctx, T*& p, int width_floats, int64_t kept, RowCopies& rc, std::vector<Swap>& sw) {
  if (!p) return LGS_OK;
  T* q = nullptr;
  LGS_TRY(dalloc(ctx, &q, (size_t)std::max<int64_t>(kept, 1) * (size_t)width_floats * sizeof(float) / sizeof(T)));
  rc.src[rc.count] = reinterpret_cast<const float*>(p);
  rc.dst[rc.count] = reinterpret_cast<float*>(q);
  rc.width[rc.count] = width_floats;
  rc.count++;
  sw.push_back(Swap{reinterpret_cast<void**>(&p), q});
  return LGS_OK;
}

}  // namespace

extern "C" {

LGS_API lgs_status lgs_find_language_redundant(lgs_ctx* ctx, const lgs_map* map, const lgs_prune_config* cfg,
                                               uint8_t* flags, int32_t memory, int64_t* count) {
  return guarded([&]() -> lgs_status {
    PruneParams pp;
    PruneIn in;
    LGS_TRY(prune_setup(ctx, map, cfg, memory, &pp, &in));
    if (in.n > 0 && !flags) return fail(LGS_EINVAL, "flags is NULL");
    uint8_t* dflags = memory == LGS_MEM_DEVICE ? flags : nullptr;
    if (!dflags) LGS_TRY(dalloc(ctx, &dflags, (size_t)in.n));
    lgs_status st = language_flags(ctx, in, pp, dflags, count);
    if (st == LGS_OK) st = flags_out(ctx, dflags, flags, memory, in.n);
    if (memory != LGS_MEM_DEVICE) dfree(ctx, dflags);
    return st;
  });
}

LGS_API lgs_status lgs_find_geometric(lgs_ctx* ctx, const lgs_map* map, const lgs_prune_config* cfg, uint8_t* flags,
                                      int32_t memory, int64_t* count) {
  return guarded([&]() -> lgs_status {
    PruneParams pp;
    PruneIn in;
    LGS_TRY(prune_setup(ctx, map, cfg, memory, &pp, &in));
    if (in.n > 0 && !flags) return fail(LGS_EINVAL, "flags is NULL");
    uint8_t* dflags = memory == LGS_MEM_DEVICE ? flags : nullptr;
    if (!dflags) LGS_TRY(dalloc(ctx, &dflags, (size_t)in.n));
    lgs_status st = geometric_flags(ctx, in, pp, dflags, count);
    if (st == LGS_OK) st = flags_out(ctx, dflags, flags, memory, in.n);
    if (memory != LGS_MEM_DEVICE) dfree(ctx, dflags);
    return st;
  });
}

LGS_API lgs_status lgs_prune(lgs_ctx* ctx, lgs_map* map, lgs_adam* adam, const lgs_prune_config* cfg,
                             uint8_t* removed_language, uint8_t* removed_geometric, int32_t memory, int64_t* kept) {
  return guarded([&]() -> lgs_status {
    PruneParams pp;
    PruneIn in;
    LGS_TRY(prune_setup(ctx, map, cfg, memory, &pp, &in));
    if (map->mapped) return fail(LGS_EINVAL, "lgs_prune needs a device map (this one is LGS_MEM_HOST_MAPPED)");
    if (adam && (adam->n != map->dm.n || adam->d != map->dm.d || adam->K != map->dm.K))
      return fail(LGS_EINVAL, "Adam state was created for a different map shape");
    const int64_t n = in.n;
    if (kept) *kept = n;
    if (n == 0) return LGS_OK;
    cudaStream_t s = ctx->stream;
    uint8_t *dl = nullptr, *dg = nullptr, *scratch = nullptr;
    LGS_TRY(dalloc(ctx, &dl, (size_t)n));
    LGS_TRY(dalloc(ctx, &dg, (size_t)n));
    lgs_status st = language_flags(ctx, in, pp, dl, nullptr);
    if (st == LGS_OK) st = geometric_flags(ctx, in, pp, dg, nullptr);
    if (st == LGS_OK) st = flags_out(ctx, dl, removed_language, memory, n);
    if (st == LGS_OK) st = flags_out(ctx, dg, removed_geometric, memory, n);
    if (st == LGS_OK && memory == LGS_MEM_DEVICE) {
      if (removed_language) LGS_CUDA(cudaMemcpyAsync(removed_language, dl, (size_t)n, cudaMemcpyDeviceToDevice, s));
      if (removed_geometric) LGS_CUDA(cudaMemcpyAsync(removed_geometric, dg, (size_t)n, cudaMemcpyDeviceToDevice, s));
    }
    int64_t nk = n;
    uint32_t *keep = nullptr, *dst_of = nullptr;
    if (st == LGS_OK) st = dalloc(ctx, &scratch, compact_scratch_bytes(n));
    if (st == LGS_OK) {
      const cudaError_t e = run_compact(dl, dg, n, scratch, &nk, &keep, &dst_of, s);
      if (e != cudaSuccess) st = fail(LGS_ECUDA, "prune compaction: %s", cudaGetErrorString(e));
    }
    if (st == LGS_OK && nk != n) {
      RowCopies rc{};
      std::vector<Swap> sw;
      const int K3 = map->dm.K * 3, fw = map->dm.dp > 0 ? map->dm.dp : 1;
      auto add = [&](auto*& p, int w) {
        if (st == LGS_OK) st = compact_alloc(ctx, p, w, nk, rc, sw);
      };
      add(map->pos_opa, 4); add(map->rot, 4); add(map->scale, 4); add(map->sh, K3); add(map->feat, fw);
      if (adam) {
        add(adam->m_po, 4); add(adam->v_po, 4); add(adam->m_rot, 4); add(adam->v_rot, 4);
        add(adam->m_sc, 4); add(adam->v_sc, 4); add(adam->m_sh, K3); add(adam->v_sh, K3);
        add(adam->m_ft, fw); add(adam->v_ft, fw);
      }
      if (st != LGS_OK) {  // out of memory part way: drop the copies, the map stays as it was
        for (Swap& w : sw) cudaFreeAsync(w.fresh, s);
      } else {
        launch_compact_rows(rc, keep, dst_of, n, s);
        ctx->launches++;
        for (Swap& w : sw) {
          cudaFreeAsync(*w.slot, s);
          *w.slot = w.fresh;
        }
        map->dm.n = nk;
        map->dm.pos_opa = map->pos_opa;
        map->dm.rot = map->rot;
        map->dm.scale = map->scale;
        map->dm.sh = map->sh;
        map->dm.feat = map->feat;
        version_drop(map->version);
        map->version = version_new();
        if (adam) adam->n = nk;
      }
    }
    dfree(ctx, scratch);
    dfree(ctx, dl);
    dfree(ctx, dg);
    if (st != LGS_OK) return st;
    LGS_CUDA(cudaStreamSynchronize(s));
    LGS_CUDA(cudaGetLastError());
    if (kept) *kept = nk;
    return LGS_OK;
  });
}

LGS_API lgs_status lgs_prune_stats(const lgs_ctx* ctx, int64_t* candidates, int64_t* rounds) {
  if (!ctx) return fail(LGS_EINVAL, "ctx is NULL");
  if (candidates) *candidates = ctx->prune_candidates;
  if (rounds) *rounds = ctx->prune_rounds;
  return LGS_OK;
}

}  // extern "C"

// -------------------------------------------------------------------------------------------
// lgs_plan: one fwd (fused L1) + bwd step captured into a CUDA graph and replayed
// -------------------------------------------------------------------------------------------
struct lgs_plan {
  lgs_ctx* ctx = nullptr;
  lgs_map* map = nullptr;
  uint64_t map_version = 0;
  lgs_camera cam{};
  lgs_render_config cfg{};
  lgs_l1_targets targets{};
  lgs_map_grads grads{};
  lgs_images images{};
  bool has_images = false;
  float* pose = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t cap_stream = nullptr;  // private capture stream (the context's may be the legacy one)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<PhaseMark> marks;  // per-phase events recorded inside the graph (profiling plans)
  bool profile = false;
  int64_t cap = 0;
  int64_t launches_per_run = 0;
  int64_t recaptures = 0;
  uint32_t* host_pairs = nullptr;  // pinned: this plan's pair count, written by every replay (each
                                   // plan its own slot: several plans may share a context)
  uint32_t* lpt[3] = {nullptr, nullptr, nullptr};  // tile orders: [0] used by a replay, [1] computed
                                                   // by it; [2] its per-tile durations
  int lpt_n = 0;
  bool speculative = false;       // captured without the layered binning's pass 2
  int64_t spec_misses = 0;        // speculative replays redone with pass 2
  uint32_t* unf_host = nullptr;   // mapped pinned: set by a speculative replay that left a tile unfinished
  uint32_t* unf_dev = nullptr;    // its device address
  uint32_t* miss_dev = nullptr;   // device copy of the flag (the chain of a missed replay adds nothing)
};

namespace {
void plan_free_marks(lgs_plan* p) {
  for (auto& m : p->marks) {
    cudaEventDestroy(m.a);
    cudaEventDestroy(m.b);
  }
  p->marks.clear();
}
}  // namespace

namespace {

lgs_status plan_capture(lgs_plan* p) {
  lgs_ctx* ctx = p->ctx;
  if (p->exec) {
    cudaGraphExecDestroy(p->exec);
    p->exec = nullptr;
  }
  // capture on a private stream (the graph is launched on the context's stream)
  cudaStream_t s = p->cap_stream;
  const cudaStream_t saved = ctx->stream;
  const int64_t l0 = ctx->launches.load();
  if (!ctx->side_stream) {
    LGS_CUDA(cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
    LGS_CUDA(cudaEventCreateWithFlags(&ctx->side_fork, cudaEventDisableTiming));
    LGS_CUDA(cudaEventCreateWithFlags(&ctx->side_join, cudaEventDisableTiming));
  }
  {  // the plan's tile-order buffers (identity before the first replay)
    const int nt = ((p->cam.width + LGS_TILE - 1) / LGS_TILE) * ((p->cam.height + LGS_TILE - 1) / LGS_TILE);
    if (nt != p->lpt_n) {
      for (auto& b : p->lpt)
        if (b) cudaFree(b), b = nullptr;
      std::vector<uint32_t> id((size_t)nt);
      for (int i = 0; i < nt; ++i) id[(size_t)i] = (uint32_t)i;
      for (auto& b : p->lpt) {
        LGS_CUDA(cudaMalloc(reinterpret_cast<void**>(&b), sizeof(uint32_t) * (size_t)std::max(nt, 1)));
        LGS_CUDA(cudaMemcpy(b, id.data(), sizeof(uint32_t) * (size_t)nt, cudaMemcpyHostToDevice));
      }
      LGS_CUDA(cudaMemset(p->lpt[2], 0, sizeof(uint32_t) * (size_t)std::max(nt, 1)));
      p->lpt_n = nt;
    }
  }
  LGS_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  ctx->stream = s;
  ctx->capturing = true;
  ctx->prezero = (p->grads.memory != LGS_MEM_HOST && !p->grads.accumulate) ? &p->grads : nullptr;
  ctx->prezero_forked = false;
  ctx->cap_lpt_cur = p->lpt[0];
  ctx->cap_lpt_next = p->lpt[1];
  ctx->cap_tile_cost = p->lpt[2];
  ctx->lpt_forked = false;
  ctx->cap_unfinished_any = p->speculative ? p->unf_dev : nullptr;
  ctx->cap_miss = p->speculative ? p->miss_dev : nullptr;
  plan_free_marks(p);
  ctx->capture_marks = p->profile ? &p->marks : nullptr;  // event nodes cost ~5 us each per replay
  uint32_t* const saved_host = ctx->host_u32;
  ctx->host_u32 = p->host_pairs;  // the replay's pair-count readback lands in the plan's own slot
  lgs_status st = LGS_OK;
  lgs_saved* tape = nullptr;
  if (cudaEventRecordWithFlags(p->ev0, s, cudaEventRecordExternal) != cudaSuccess)
    st = fail(LGS_ECUDA, "event record in capture failed");
  if (st == LGS_OK)
    st = lgs_render_forward(ctx, p->map, &p->cam, &p->cfg, &p->targets, p->has_images ? &p->images : nullptr, &tape);
  if (st == LGS_OK) {
    BwdIn in{};
    in.g_rgb = tape->cot;
    in.cot_stride = 4 + tape->dm.dp;
    st = run_backward(ctx, tape, in, &p->grads, p->pose, true);
  }
  if (tape) lgs_saved_destroy(tape);  // stream-ordered frees: captured as graph free nodes
  if (st == LGS_OK && cudaEventRecordWithFlags(p->ev1, s, cudaEventRecordExternal) != cudaSuccess)
    st = fail(LGS_ECUDA, "event record in capture failed");
  if (ctx->prezero_forked) {  // forward captured but the backward failed: join the side branch
    cudaStreamWaitEvent(s, ctx->side_join, 0);
    ctx->prezero_forked = false;
  }
  ctx->lpt_forked = false;
  ctx->cap_unfinished_any = nullptr;
  ctx->cap_miss = nullptr;
  ctx->cap_lpt_cur = ctx->cap_lpt_next = ctx->cap_tile_cost = nullptr;
  ctx->prezero = nullptr;
  ctx->capturing = false;
  ctx->capture_marks = nullptr;
  ctx->stream = saved;
  ctx->host_u32 = saved_host;
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(s, &graph);
  if (st != LGS_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (ec != cudaSuccess) return fail(LGS_ECUDA, "stream capture failed: %s", cudaGetErrorString(ec));
  const cudaError_t ei = cudaGraphInstantiate(&p->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) return fail(LGS_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(ei));
  p->cap = ctx->pairs_cap;
  p->launches_per_run = ctx->launches.load() - l0;
  ctx->launches -= p->launches_per_run;  // counted per replay
  return LGS_OK;
}

}  // namespace

extern "C" {

LGS_API lgs_status lgs_plan_create(lgs_ctx* ctx, lgs_map* map, const lgs_camera* cam, const lgs_render_config* cfg,
                                   const lgs_l1_targets* targets, const lgs_images* images, lgs_map_grads* grads,
                                   float* pose_grad, lgs_plan** out) {
  if (!ctx || !map || !cam || !targets || !grads || !out) return fail(LGS_EINVAL, "NULL argument");
  *out = nullptr;
  if (targets->memory != LGS_MEM_DEVICE || grads->memory != LGS_MEM_DEVICE ||
      (images && images->memory != LGS_MEM_DEVICE))
    return fail(LGS_EINVAL, "a plan reads device targets and writes device images / gradients");
  // grads->accumulate: every replay adds its gradients (the later views of a multi-view batch); a
  // replay whose tile lists overflowed adds nothing (empty lists) before lgs_plan_sync re-runs it
  LGS_CUDA(cudaSetDevice(ctx->device));
  lgs_plan* p = new lgs_plan();
  p->ctx = ctx;
  p->map = map;
  p->map_version = map->version;
  p->cam = *cam;
  p->cfg = cfg ? *cfg : lgs_render_config_default();
  p->targets = *targets;
  p->grads = *grads;
  if (images) {
    p->images = *images;
    p->has_images = true;
  }
  p->pose = pose_grad;
  ctx->refs++;
  auto bail = [&](lgs_status st) {
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
    if (p->host_pairs) cudaFreeHost(p->host_pairs);
    if (p->unf_host) cudaFreeHost(p->unf_host);
    if (p->miss_dev) cudaFree(p->miss_dev);
    for (auto& b : p->lpt)
      if (b) cudaFree(b);
    ctx_release(ctx);
    delete p;
    return st;
  };
  if (cudaEventCreate(&p->ev0) != cudaSuccess || cudaEventCreate(&p->ev1) != cudaSuccess ||
      cudaMallocHost(&p->host_pairs, 64) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&p->unf_host), 64, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->unf_dev), p->unf_host, 0) != cudaSuccess ||
      cudaMalloc(reinterpret_cast<void**>(&p->miss_dev), sizeof(uint32_t)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(LGS_ECUDA, "event / stream creation failed"));
  // the layer-A policy starts afresh for the plan's own view (several plans on one context -- the
  // views of a batch -- would otherwise inherit each other's layer-A size or single-pass switch),
  // then forward-only eager renders until it settles (at most 4), then one eager step sizes the
  // tile-list capacity (and runs every one-time kernel setup)
  ctx->layer_div = kLayerDiv;
  ctx->layer_bad = UINT32_MAX;
  ctx->single_pass = false;
  ctx->lp_pending = false;
  for (int it = 0; it < 4; ++it) {
    const uint32_t div0 = ctx->layer_div;
    lgs_status sw = lgs_render_forward(ctx, map, &p->cam, &p->cfg, &p->targets, nullptr, nullptr);
    if (sw != LGS_OK) return bail(sw);
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return bail(fail(LGS_ECUDA, "warm-up render failed"));
    layer_policy_update(ctx, ((p->cam.width + LGS_TILE - 1) / LGS_TILE) * ((p->cam.height + LGS_TILE - 1) / LGS_TILE));
    if (ctx->layer_div == div0 && it > 0) break;
  }
  lgs_saved* tape = nullptr;
  lgs_status st =
      lgs_render_forward(ctx, map, &p->cam, &p->cfg, &p->targets, p->has_images ? &p->images : nullptr, &tape);
  if (st == LGS_OK) st = lgs_render_backward_loss_async(ctx, tape, &p->grads, p->pose);
  if (tape) lgs_saved_destroy(tape);
  if (st != LGS_OK) return bail(st);
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return bail(fail(LGS_ECUDA, "warm-up step failed"));
  {
    // every tile of the last counted render saturated on its layer-A list (the step's pass 2 did
    // nothing): capture pass 1 only; the replays report any unfinished tile (lgs_plan_sync)
    const int nt = ((p->cam.width + LGS_TILE - 1) / LGS_TILE) * ((p->cam.height + LGS_TILE - 1) / LGS_TILE);
    layer_policy_update(ctx, nt);
    p->speculative = !ctx->no_speculative && ctx->lp_last_unfinished == 0 &&
                     ctx->lp_last_ntiles == nt && ctx->lp_last_div == ctx->layer_div;
    *p->unf_host = 0;
  }
  if ((st = plan_capture(p)) != LGS_OK) return bail(st);
  *out = p;
  return LGS_OK;
}

LGS_API lgs_status lgs_plan_run(lgs_ctx* ctx, lgs_plan* p) {
  if (!ctx || !p || ctx != p->ctx) return fail(LGS_EINVAL, "plan / context mismatch");
  if (!version_live(p->map_version)) return fail(LGS_EINVAL, "the plan's map was pruned or destroyed: recreate the plan");
  if (p->speculative) *reinterpret_cast<volatile uint32_t*>(p->unf_host) = 0;
  LGS_CUDA(cudaGraphLaunch(p->exec, ctx->stream));
  ctx->launches += p->launches_per_run;
  return LGS_OK;
}

LGS_API lgs_status lgs_plan_sync(lgs_ctx* ctx, lgs_plan* p, int64_t* pairs) {
  if (!ctx || !p || ctx != p->ctx) return fail(LGS_EINVAL, "plan / context mismatch");
  LGS_CUDA(cudaStreamSynchronize(ctx->stream));
  int64_t P = p->host_pairs[0];
  for (int redo = 0; redo < 3; ++redo) {
    // P > capacity: the replay ran on empty tile lists (grow, re-capture, redo the step); a
    // speculative replay that left a tile unfinished: re-capture with pass 2 and redo the step
    const bool over = P > p->cap;
    const bool unfinished = !over && p->speculative && *reinterpret_cast<volatile uint32_t*>(p->unf_host) != 0;
    if (!over && !unfinished) break;
    if (over) ctx->pairs_cap = std::max<int64_t>(ctx->pairs_cap, P + P / 4);
    if (unfinished) {
      p->speculative = false;
      ++p->spec_misses;
    }
    ++p->recaptures;
    LGS_TRY(plan_capture(p));
    LGS_TRY(lgs_plan_run(ctx, p));
    LGS_CUDA(cudaStreamSynchronize(ctx->stream));
    P = p->host_pairs[0];
  }
  if (pairs) *pairs = P;
  return LGS_OK;
}

LGS_API lgs_status lgs_plan_set_camera(lgs_ctx* ctx, lgs_plan* p, const lgs_camera* cam) {
  if (!ctx || !p || !cam || ctx != p->ctx) return fail(LGS_EINVAL, "bad argument");
  p->cam = *cam;  // the camera is baked into the kernel parameters: re-capture
  return plan_capture(p);
}

LGS_API lgs_status lgs_plan_elapsed_ms(const lgs_plan* p, float* ms) {
  if (!p || !ms) return fail(LGS_EINVAL, "NULL argument");
  LGS_CUDA(cudaEventElapsedTime(ms, p->ev0, p->ev1));
  return LGS_OK;
}

LGS_API int64_t lgs_plan_launches(const lgs_plan* p) { return p ? p->launches_per_run : -1; }

LGS_API lgs_status lgs_plan_set_profiling(lgs_ctx* ctx, lgs_plan* p, int32_t on) {
  if (!ctx || !p || ctx != p->ctx) return fail(LGS_EINVAL, "plan / context mismatch");
  if (p->profile == (on != 0)) return LGS_OK;
  p->profile = on != 0;
  return plan_capture(p);
}

LGS_API lgs_status lgs_plan_phase_times(const lgs_plan* p, double* ms) {
  if (!p || !ms) return fail(LGS_EINVAL, "NULL argument");
  if (!p->profile) return fail(LGS_EINVAL, "plan not profiling (lgs_plan_set_profiling)");
  for (int i = 0; i < LGS_PHASE_COUNT; ++i) ms[i] = 0.0;
  for (const auto& m : p->marks) {
    float t = 0.f;
    LGS_CUDA(cudaEventElapsedTime(&t, m.a, m.b));
    ms[m.phase] += t;
  }
  return LGS_OK;
}

LGS_API lgs_status lgs_plan_destroy(lgs_plan* p) {
  if (!p) return LGS_OK;
  lgs_ctx* ctx = p->ctx;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (p->exec) cudaGraphExecDestroy(p->exec);
  if (p->ev0) cudaEventDestroy(p->ev0);
  plan_free_marks(p);
  if (p->ev1) cudaEventDestroy(p->ev1);
  if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
  if (p->host_pairs) cudaFreeHost(p->host_pairs);
  if (p->unf_host) cudaFreeHost(p->unf_host);
  if (p->miss_dev) cudaFree(p->miss_dev);
  for (auto& b : p->lpt)
    if (b) cudaFree(b);
  delete p;
  ctx_release(ctx);
  return LGS_OK;
}

LGS_API int64_t lgs_plan_recaptures(const lgs_plan* p) { return p ? p->recaptures : -1; }

LGS_API int32_t lgs_plan_speculative(const lgs_plan* p) { return p ? (p->speculative ? 1 : 0) : -1; }

}  // extern "C"
