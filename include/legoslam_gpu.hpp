// legoslam_gpu.hpp -- drop-in C++ shim: the reference's lego::render / lego::render_backward with
// their exact signatures (proj/include/legoslam/renderer.hpp:55-56, 72-74), implemented on liblgs.so.
//
// Compiles inside the reference tree (it needs Eigen and legoslam/renderer.hpp; guarded by
// __has_include).  A maintainer switches the CPU compositor for the B200 rasterizer by calling
// lego::gpu::render / lego::gpu::render_backward (or `namespace lego { using gpu::render; ... }`)
// with the same arguments -- nothing else changes for the callers.  oracle/Makefile builds
// tests/cpp/shim_vs_reference.cpp against the reference's own headers and renderer to prove it.
//
// The reference keeps its backward tape inside RenderOutput (projected + pixel_contribs,
// renderer.hpp:39-41); the GPU tape stays on the device, so the shim keeps it in a per-thread table
// keyed by the RenderOutput's rgb buffer (stable across moves of the RenderOutput) and bounded to
// the kTapes most recent renders of the thread (older ones are released; release(out) frees one
// early).  render_backward of a RenderOutput whose tape is gone throws std::invalid_argument.
#pragma once

#if __has_include(<Eigen/Core>) && __has_include("legoslam/renderer.hpp")
#include <Eigen/Core>

#include <cstddef>
#include <deque>
#include <memory>
#include <stdexcept>
#include <utility>
#include <vector>

#include "legoslam/renderer.hpp"
#include "lgs.h"

namespace lego::gpu {

constexpr std::size_t kTapes = 16;  // renders whose backward tape a thread keeps

inline void check(lgs_status s) {
  if (s == LGS_EINVAL) throw std::invalid_argument(lgs_last_error());
  if (s != LGS_OK) throw std::runtime_error(lgs_last_error());
}

// One context per host thread (the reference allows concurrent renders between map mutations,
// SPEC.md:298-299; a context is one CUDA stream + memory pool).
struct Context {
  lgs_ctx* ctx = nullptr;
  Context() { check(lgs_ctx_create(0, nullptr, &ctx)); }
  ~Context() { lgs_ctx_destroy(ctx); }
};

struct Tape {
  lgs_saved* saved = nullptr;
  Tape() = default;
  Tape(const Tape&) = delete;
  Tape& operator=(const Tape&) = delete;
  ~Tape() { lgs_saved_destroy(saved); }
};

struct State {
  Context context;
  std::deque<std::pair<const double*, std::unique_ptr<Tape>>> tapes;  // most recent last
};

inline State& state() {
  thread_local State s;
  return s;
}

// fp64 Eigen SoA -> fp32 reference layouts (x,y,z,w rotations, [d][N] features)
struct Packed {
  std::vector<float> pos, rot, ls, op, sh, feat;
  lgs_gaussians g{};
  explicit Packed(const GaussianMap& m) {
    const std::size_t n = m.size();
    const int d = m.feature_dim();
    pos.resize(n * 3); rot.resize(n * 4); ls.resize(n * 3); op.resize(n); sh.resize(n * 3);
    feat.resize(n * (std::size_t)d);
    for (std::size_t i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) {
        pos[i * 3 + a] = (float)m.positions()[i][a];
        ls[i * 3 + a] = (float)m.log_scales()[i][a];
        sh[i * 3 + a] = (float)m.colors()[i][a];
      }
      const auto& q = m.rotations()[i].coeffs();  // Eigen storage x, y, z, w
      for (int a = 0; a < 4; ++a) rot[i * 4 + a] = (float)q[a];
      op[i] = (float)m.opacity_logits()[i];
      for (int c = 0; c < d; ++c) feat[(std::size_t)c * n + i] = (float)m.features()((Eigen::Index)i, c);
    }
    g = {(int64_t)n, d, 0, pos.data(), rot.data(), ls.data(), op.data(), sh.data(), feat.data(), LGS_MEM_HOST};
  }
};

inline lgs_camera camera(const Pose& p, const CameraIntrinsics& k) {
  lgs_camera c{};
  c.q[0] = p.rotation.w(); c.q[1] = p.rotation.x(); c.q[2] = p.rotation.y(); c.q[3] = p.rotation.z();
  for (int a = 0; a < 3; ++a) c.t[a] = p.translation[a];
  c.fx = k.fx; c.fy = k.fy; c.cx = k.cx; c.cy = k.cy; c.width = k.width; c.height = k.height;
  return c;
}

// Drops the device tape of `out` (optional: the table forgets old renders by itself).
inline void release(const RenderOutput& out) {
  auto& t = state().tapes;
  for (auto it = t.begin(); it != t.end(); ++it)
    if (it->first == out.rgb.data.data()) {
      t.erase(it);
      return;
    }
}

// lego::render (renderer.hpp:55-56)
inline RenderOutput render(const GaussianMap& map, const Pose& cam_pose, const CameraIntrinsics& k,
                           const RenderConfig& cfg = {}) {
  State& st = state();
  Packed pk(map);
  const lgs_camera cam = camera(cam_pose, k);
  const lgs_render_config rc{cfg.near_plane, cfg.dilation, cfg.alpha_clamp, cfg.alpha_skip, cfg.transmittance_min,
                             cfg.radius_sigma};
  const int d = map.feature_dim();
  const std::size_t npix = (std::size_t)k.width * k.height;
  std::vector<float> rgb(npix * 3), depth(npix), feat(npix * (std::size_t)d), acc(npix);
  lgs_images img{rgb.data(), depth.data(), d ? feat.data() : nullptr, acc.data(), LGS_MEM_HOST};
  auto tape = std::make_unique<Tape>();
  check(lgs_render(st.context.ctx, &pk.g, &cam, &rc, &img, &tape->saved));
  RenderOutput o;
  o.cam_pose = cam_pose;
  o.intrinsics = k;
  o.config = cfg;
  o.rgb = ImageD(k.height, k.width, 3);
  o.depth = ImageD(k.height, k.width, 1);
  o.feat = ImageD(k.height, k.width, d);
  o.acc = ImageD(k.height, k.width, 1);
  for (std::size_t i = 0; i < npix * 3; ++i) o.rgb.data[i] = rgb[i];
  for (std::size_t i = 0; i < npix; ++i) {
    o.depth.data[i] = depth[i];
    o.acc.data[i] = acc[i];
  }
  for (std::size_t i = 0; i < npix * (std::size_t)d; ++i) o.feat.data[i] = feat[i];
  st.tapes.emplace_back(o.rgb.data.data(), std::move(tape));
  while (st.tapes.size() > kTapes) st.tapes.pop_front();
  return o;
}

// lego::render_backward (renderer.hpp:72-74): an empty cotangent means zero; a shape mismatch
// throws std::invalid_argument (renderer.cpp:176-178); gradients are dense over the map.
inline MapGradients render_backward(const GaussianMap& map, const RenderOutput& out, const ImageD& grad_rgb,
                                    const ImageD& grad_depth, const ImageD& grad_feat) {
  State& st = state();
  const Tape* tape = nullptr;
  for (const auto& e : st.tapes)
    if (e.first == out.rgb.data.data()) tape = e.second.get();
  if (!tape) throw std::invalid_argument("render_backward: no GPU tape for this RenderOutput (released or too old)");
  const int d = map.feature_dim();
  const std::size_t n = map.size();
  auto to_f32 = [](const ImageD& im) { return std::vector<float>(im.data.begin(), im.data.end()); };
  std::vector<float> gr = to_f32(grad_rgb), gd = to_f32(grad_depth), gf = to_f32(grad_feat);
  lgs_cotangents cot{};
  cot.rgb = grad_rgb.empty() ? nullptr : gr.data();
  cot.depth = grad_depth.empty() ? nullptr : gd.data();
  cot.feat = grad_feat.empty() ? nullptr : gf.data();
  cot.memory = LGS_MEM_HOST;
  cot.rgb_shape[0] = grad_rgb.height; cot.rgb_shape[1] = grad_rgb.width; cot.rgb_shape[2] = grad_rgb.channels;
  cot.depth_shape[0] = grad_depth.height; cot.depth_shape[1] = grad_depth.width; cot.depth_shape[2] = grad_depth.channels;
  cot.feat_shape[0] = grad_feat.height; cot.feat_shape[1] = grad_feat.width; cot.feat_shape[2] = grad_feat.channels;
  std::vector<float> pos(n * 3), rot(n * 4), ls(n * 3), op(n), col(n * 3), feat(n * (std::size_t)d);
  lgs_map_grads g{pos.data(), rot.data(), ls.data(), op.data(), col.data(), d ? feat.data() : nullptr, LGS_MEM_HOST, 0};
  check(lgs_render_backward(st.context.ctx, tape->saved, &cot, &g, nullptr));
  MapGradients mg;
  mg.resize(n, d);
  for (std::size_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) {
      mg.position[i][a] = pos[i * 3 + a];
      mg.log_scale[i][a] = ls[i * 3 + a];
      mg.color[i][a] = col[i * 3 + a];
    }
    for (int a = 0; a < 4; ++a) mg.rotation[i][a] = rot[i * 4 + a];  // (w, x, y, z)
    mg.opacity_logit[i] = op[i];
    for (int c = 0; c < d; ++c) mg.feature((Eigen::Index)i, c) = feat[(std::size_t)c * n + i];
  }
  return mg;
}

}  // namespace lego::gpu
#endif
