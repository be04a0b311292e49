// legoslam_gpu.hpp -- drop-in C++ shim: the reference's lego::render / lego::render_backward
// signatures (proj/include/legoslam/renderer.hpp:55-56, 72-74) implemented on liblgs.so.
//
// Only compiles inside the reference tree (needs Eigen and legoslam/renderer.hpp); it is the glue a
// maintainer adds to switch the CPU compositor for the B200 rasterizer without touching callers.
// Usage: #include "legoslam_gpu.hpp" and call lego::gpu::render(...) / lego::gpu::render_backward(...)
// with the same arguments as lego::render / lego::render_backward (or alias them in renderer.hpp).
#pragma once

#if __has_include(<Eigen/Core>) && __has_include("legoslam/renderer.hpp")
#include <Eigen/Core>

#include <memory>
#include <stdexcept>
#include <vector>

#include "legoslam/renderer.hpp"
#include "lgs.h"

namespace lego::gpu {

// The backward tape of one GPU render (the GPU counterpart of RenderOutput.projected +
// pixel_contribs, renderer.hpp:39-41).
struct Tape {
  lgs_saved* saved = nullptr;
  ~Tape() { lgs_saved_destroy(saved); }
};

inline lgs_ctx* context() {
  static lgs_ctx* ctx = [] {
    lgs_ctx* c = nullptr;
    if (lgs_ctx_create(0, nullptr, &c) != LGS_OK) throw std::runtime_error(lgs_last_error());
    return c;
  }();
  return ctx;
}

inline void check(lgs_status s) {
  if (s == LGS_EINVAL) throw std::invalid_argument(lgs_last_error());
  if (s != LGS_OK) throw std::runtime_error(lgs_last_error());
}

// fp64 Eigen SoA -> fp32 reference layouts (x,y,z,w rotations, [d][N] features)
struct Packed {
  std::vector<float> pos, rot, ls, op, sh, feat;
  lgs_gaussians g{};
  explicit Packed(const GaussianMap& m) {
    const size_t n = m.size();
    const int d = m.feature_dim();
    pos.resize(n * 3); rot.resize(n * 4); ls.resize(n * 3); op.resize(n); sh.resize(n * 3); feat.resize(n * d);
    for (size_t i = 0; i < n; ++i) {
      for (int a = 0; a < 3; ++a) {
        pos[i * 3 + a] = (float)m.positions()[i][a];
        ls[i * 3 + a] = (float)m.log_scales()[i][a];
        sh[i * 3 + a] = (float)m.colors()[i][a];
      }
      const auto& q = m.rotations()[i].coeffs();  // Eigen storage x, y, z, w
      for (int a = 0; a < 4; ++a) rot[i * 4 + a] = (float)q[a];
      op[i] = (float)m.opacity_logits()[i];
      for (int c = 0; c < d; ++c) feat[(size_t)c * n + i] = (float)m.features()(i, c);
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

// lego::render (renderer.hpp:55-56).  The returned RenderOutput carries images, pose, intrinsics
// and config; `tape` keeps what render_backward needs on the device.
inline RenderOutput render(const GaussianMap& map, const Pose& cam_pose, const CameraIntrinsics& k,
                           const RenderConfig& cfg, std::shared_ptr<Tape>& tape) {
  Packed pk(map);
  const lgs_camera cam = camera(cam_pose, k);
  const lgs_render_config rc{cfg.near_plane, cfg.dilation, cfg.alpha_clamp, cfg.alpha_skip, cfg.transmittance_min,
                             cfg.radius_sigma};
  const int d = map.feature_dim();
  const size_t npix = (size_t)k.width * k.height;
  std::vector<float> rgb(npix * 3), depth(npix), feat(npix * d), acc(npix);
  lgs_images out{rgb.data(), depth.data(), feat.data(), acc.data(), LGS_MEM_HOST};
  tape = std::make_shared<Tape>();
  check(lgs_render(context(), &pk.g, &cam, &rc, &out, &tape->saved));
  RenderOutput o;
  o.cam_pose = cam_pose;
  o.intrinsics = k;
  o.config = cfg;
  o.rgb = ImageD(k.height, k.width, 3);
  o.depth = ImageD(k.height, k.width, 1);
  o.feat = ImageD(k.height, k.width, d);
  o.acc = ImageD(k.height, k.width, 1);
  for (size_t i = 0; i < npix * 3; ++i) o.rgb.data[i] = rgb[i];
  for (size_t i = 0; i < npix; ++i) { o.depth.data[i] = depth[i]; o.acc.data[i] = acc[i]; }
  for (size_t i = 0; i < npix * d; ++i) o.feat.data[i] = feat[i];
  return o;
}

// lego::render_backward (renderer.hpp:72-74): same empty-means-zero and std::invalid_argument rules.
inline MapGradients render_backward(const GaussianMap& map, const RenderOutput& out, const Tape& tape,
                                    const ImageD& grad_rgb, const ImageD& grad_depth, const ImageD& grad_feat) {
  const int d = map.feature_dim();
  const size_t n = map.size();
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
  std::vector<float> pos(n * 3), rot(n * 4), ls(n * 3), op(n), col(n * 3), feat(n * d);
  lgs_map_grads g{pos.data(), rot.data(), ls.data(), op.data(), col.data(), feat.data(), LGS_MEM_HOST, 0};
  check(lgs_render_backward(context(), tape.saved, &cot, &g, nullptr));
  MapGradients mg;
  mg.resize(n, d);
  for (size_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) {
      mg.position[i][a] = pos[i * 3 + a];
      mg.log_scale[i][a] = ls[i * 3 + a];
      mg.color[i][a] = col[i * 3 + a];
    }
    for (int a = 0; a < 4; ++a) mg.rotation[i][a] = rot[i * 4 + a];  // (w, x, y, z)
    mg.opacity_logit[i] = op[i];
    for (int c = 0; c < d; ++c) mg.feature(i, c) = feat[(size_t)c * n + i];
  }
  (void)out;
  return mg;
}

}  // namespace lego::gpu
#endif
