// TEST INFRASTRUCTURE ONLY -- C ABI over the reference renderer compiled from its own sources.
//
// oracle/Makefile builds this file together with the UNMODIFIED reference translation units
// /root/reference/proj/src/renderer.cpp and geometry.cpp (and includes the reference headers and
// proj/tests/gradcheck.hpp from /root/reference) into oracle/_ref/liblgs_ref.so, using the
// self-written Eigen subset in oracle/eigen_shim (the reference needs Eigen3, absent here).  The
// library is the checker of oracle A (tests/test_reference_build.py) and the CPU arm of bench.py
// --impl reference; the product never loads it.
//
// Flat layouts are oracle A's (lgs_oracle.c orc_map / orc_camera / orc_config): positions [N][3],
// rotations [N][4] (x,y,z,w), log-scales [N][3], opacity logits [N], colours [N][3] (SH degree 0:
// the reference has no higher bands), features [d][N]; images HWC; gradient rotations (w,x,y,z).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "gradcheck.hpp"
#include "legoslam/gaussian_map.hpp"
#include "legoslam/kdtree.hpp"
#include "legoslam/renderer.hpp"

namespace lego {
// GaussianMap::insert lives in gaussian_map.cpp (:19-37), a translation unit that also holds the
// keyframe insertion (Eigen's eigen solver + the codec) and the map I/O; rather than compiling
// that, the member is restated here: append every attribute, renormalise a rotation whose norm is
// off unit by more than 1e-6, hand out the next id.
std::uint64_t GaussianMap::insert(const LanguageGaussian& g, std::uint64_t anchor_kf) {
  positions_.push_back(g.position);
  Quat q = g.rotation;
  if (std::abs(q.norm() - 1.0) > 1e-6) q.normalize();
  rotations_.push_back(q);
  log_scales_.push_back(g.log_scale);
  opacity_logits_.push_back(g.opacity_logit);
  colors_.push_back(g.color);
  const auto n = static_cast<Eigen::Index>(positions_.size());
  features_.conservativeResize(n, feature_dim_);
  features_.row(n - 1) = g.feature.transpose();
  ids_.push_back(next_id_++);
  anchors_.push_back(anchor_kf);
  known_anchors_.insert(anchor_kf);
  return ids_.back();
}
}  // namespace lego

namespace {

struct RefMap {
  int64_t n;
  int32_t d;
  int32_t sh_degree;
  const double* pos;
  const double* rot;
  const double* log_s;
  const double* opac;
  const double* sh;
  const double* feat;
};
struct RefConfig {
  double near_plane, dilation, alpha_clamp, alpha_skip, transmittance_min, radius_sigma;
};
struct RefCamera {
  double q[4];
  double t[3];
  double fx, fy, cx, cy;
  int32_t width, height;
};

// The map through its mutable SoA accessors (gaussian_map.hpp:57-68).  GaussianMap::insert would
// conservativeResize the feature matrix once per Gaussian (quadratic in N); render and
// render_backward read only these arrays.  Rotations are stored as given (already unit).
lego::GaussianMap build_map(const RefMap* m) {
  lego::GaussianMap map(m->d);
  const auto n = static_cast<std::size_t>(m->n);
  const int K = (m->sh_degree + 1) * (m->sh_degree + 1);
  map.positions().reserve(n);
  map.rotations().reserve(n);
  map.log_scales().reserve(n);
  map.opacity_logits().reserve(n);
  map.colors().reserve(n);
  for (std::size_t i = 0; i < n; ++i) {
    map.positions().push_back(lego::Vec3(m->pos[i * 3], m->pos[i * 3 + 1], m->pos[i * 3 + 2]));
    map.rotations().push_back(lego::Quat(m->rot[i * 4 + 3], m->rot[i * 4], m->rot[i * 4 + 1], m->rot[i * 4 + 2]));
    map.log_scales().push_back(lego::Vec3(m->log_s[i * 3], m->log_s[i * 3 + 1], m->log_s[i * 3 + 2]));
    map.opacity_logits().push_back(m->opac[i]);
    map.colors().push_back(lego::Vec3(m->sh[i * K * 3], m->sh[i * K * 3 + 1], m->sh[i * K * 3 + 2]));
  }
  Eigen::MatrixXd f(static_cast<Eigen::Index>(n), m->d);
  for (int c = 0; c < m->d; ++c)
    for (std::size_t i = 0; i < n; ++i) f(static_cast<Eigen::Index>(i), c) = m->feat[(std::size_t)c * n + i];
  map.features() = f;
  return map;
}

lego::Pose to_pose(const RefCamera* c) {
  return lego::Pose(lego::Quat(c->q[0], c->q[1], c->q[2], c->q[3]), lego::Vec3(c->t[0], c->t[1], c->t[2]));
}
lego::CameraIntrinsics to_k(const RefCamera* c) {
  lego::CameraIntrinsics k;
  k.fx = c->fx;
  k.fy = c->fy;
  k.cx = c->cx;
  k.cy = c->cy;
  k.width = c->width;
  k.height = c->height;
  return k;
}
lego::RenderConfig to_cfg(const RefConfig* c) {
  lego::RenderConfig r;
  r.near_plane = c->near_plane;
  r.dilation = c->dilation;
  r.alpha_clamp = c->alpha_clamp;
  r.alpha_skip = c->alpha_skip;
  r.transmittance_min = c->transmittance_min;
  r.radius_sigma = c->radius_sigma;
  return r;
}

struct Handle {
  lego::GaussianMap map{0};
  lego::RenderOutput out;
};

lego::ImageD image_from(const double* p, int h, int w, int c) {
  if (!p) return lego::ImageD{};
  lego::ImageD im(h, w, c);
  std::memcpy(im.data.data(), p, sizeof(double) * im.data.size());
  return im;
}

void grads_out(const lego::MapGradients& g, int64_t n, int d, double* o_pos, double* o_rot, double* o_logs,
               double* o_opac, double* o_color, double* o_feat) {
  for (int64_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) {
      if (o_pos) o_pos[i * 3 + a] = g.position[i][a];
      if (o_logs) o_logs[i * 3 + a] = g.log_scale[i][a];
      if (o_color) o_color[i * 3 + a] = g.color[i][a];
    }
    for (int a = 0; a < 4; ++a)
      if (o_rot) o_rot[i * 4 + a] = g.rotation[i][a];
    if (o_opac) o_opac[i] = g.opacity_logit[i];
    for (int c = 0; c < d; ++c)
      if (o_feat) o_feat[c * n + i] = g.feature(i, c);
  }
}

// L1 cotangents of L = mean|rgb - T| + mean|depth - T| + mean|feat - T| (the bench loss)
void l1_cot(const lego::RenderOutput& o, const double* trgb, const double* tdepth, const double* tfeat,
            lego::ImageD& g_rgb, lego::ImageD& g_depth, lego::ImageD& g_feat) {
  auto sgn = [](double x) { return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); };
  g_rgb = lego::ImageD(o.rgb.height, o.rgb.width, 3);
  g_depth = lego::ImageD(o.depth.height, o.depth.width, 1);
  g_feat = lego::ImageD(o.feat.height, o.feat.width, o.feat.channels);
  for (std::size_t i = 0; i < g_rgb.data.size(); ++i) g_rgb.data[i] = sgn(o.rgb.data[i] - trgb[i]) / g_rgb.data.size();
  for (std::size_t i = 0; i < g_depth.data.size(); ++i)
    g_depth.data[i] = sgn(o.depth.data[i] - tdepth[i]) / g_depth.data.size();
  for (std::size_t i = 0; i < g_feat.data.size(); ++i)
    g_feat.data[i] = sgn(o.feat.data[i] - tfeat[i]) / g_feat.data.size();
}

}  // namespace

#define REF_API extern "C" __attribute__((visibility("default")))

REF_API void* ref_render(const RefMap* m, const RefCamera* cam, const RefConfig* cfg, double* rgb, double* depth,
                         double* feat, double* acc) {
  auto* h = new Handle;
  h->map = build_map(m);
  h->out = lego::render(h->map, to_pose(cam), to_k(cam), to_cfg(cfg));
  std::memcpy(rgb, h->out.rgb.data.data(), sizeof(double) * h->out.rgb.data.size());
  std::memcpy(depth, h->out.depth.data.data(), sizeof(double) * h->out.depth.data.size());
  if (feat && !h->out.feat.data.empty())
    std::memcpy(feat, h->out.feat.data.data(), sizeof(double) * h->out.feat.data.size());
  std::memcpy(acc, h->out.acc.data.data(), sizeof(double) * h->out.acc.data.size());
  return h;
}

REF_API int64_t ref_num_projected(void* hp) { return (int64_t) static_cast<Handle*>(hp)->out.projected.size(); }

REF_API void ref_sorted_indices(void* hp, int64_t* out) {
  const auto& p = static_cast<Handle*>(hp)->out.projected;
  for (std::size_t i = 0; i < p.size(); ++i) out[i] = p[i].index;
}

REF_API void ref_contrib_counts(void* hp, int32_t* out) {
  const auto& c = static_cast<Handle*>(hp)->out.pixel_contribs;
  for (std::size_t i = 0; i < c.size(); ++i) out[i] = (int32_t)c[i].size();
}

// 0 ok, 1 std::invalid_argument (cotangent shape mismatch, renderer.cpp:176-178)
REF_API int ref_render_backward(void* hp, const double* g_rgb, const int32_t* rgb_shape, const double* g_depth,
                                const int32_t* depth_shape, const double* g_feat, const int32_t* feat_shape,
                                double* o_pos, double* o_rot, double* o_logs, double* o_opac, double* o_color,
                                double* o_feat) {
  auto* h = static_cast<Handle*>(hp);
  const auto& k = h->out.intrinsics;
  auto img = [&](const double* p, const int32_t* s, int c) {
    if (!p) return lego::ImageD{};
    return s ? image_from(p, s[0], s[1], s[2]) : image_from(p, k.height, k.width, c);
  };
  try {
    const auto g = lego::render_backward(h->map, h->out, img(g_rgb, rgb_shape, 3), img(g_depth, depth_shape, 1),
                                         img(g_feat, feat_shape, h->map.feature_dim()));
    grads_out(g, (int64_t)h->map.size(), h->map.feature_dim(), o_pos, o_rot, o_logs, o_opac, o_color, o_feat);
  } catch (const std::invalid_argument&) {
    return 1;
  }
  return 0;
}

REF_API void ref_render_free(void* hp) { delete static_cast<Handle*>(hp); }

REF_API int ref_project_gaussian(const RefMap* m, int64_t index, const RefCamera* cam, const RefConfig* cfg,
                                 double* uvdr, double* cov, double* conic) {
  const auto map = build_map(m);
  const auto p = lego::project_gaussian(map, (std::size_t)index, to_pose(cam), to_k(cam), to_cfg(cfg));
  if (!p) return 0;
  uvdr[0] = p->u;
  uvdr[1] = p->v;
  uvdr[2] = p->depth;
  uvdr[3] = p->radius;
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c) {
      cov[r * 2 + c] = p->cov2d(r, c);
      conic[r * 2 + c] = p->conic(r, c);
    }
  return 1;
}

// The reference's own seeded gradcheck scene (gradcheck.hpp:31-78), as built by THIS compiler
// (constructor-argument evaluation order is the compiler's): map arrays (n, d given), camera,
// config, and the weight images w_rgb [S][S][3], w_depth [S][S], w_feat [S][S][d].
REF_API void ref_grad_scene(int n, int size, int d, uint64_t seed, double* pos, double* rot, double* log_s,
                            double* opac, double* color, double* feat, RefCamera* cam, RefConfig* cfg, double* w_rgb,
                            double* w_depth, double* w_feat) {
  const auto s = legotest::make_grad_scene(n, size, d, seed);
  for (int i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) {
      pos[i * 3 + a] = s.map.positions()[i][a];
      log_s[i * 3 + a] = s.map.log_scales()[i][a];
      color[i * 3 + a] = s.map.colors()[i][a];
    }
    const auto& q = s.map.rotations()[i];
    rot[i * 4 + 0] = q.x();
    rot[i * 4 + 1] = q.y();
    rot[i * 4 + 2] = q.z();
    rot[i * 4 + 3] = q.w();
    opac[i] = s.map.opacity_logits()[i];
    for (int c = 0; c < d; ++c) feat[c * n + i] = s.map.features()(i, c);
  }
  cam->q[0] = s.cam_pose.rotation.w();
  cam->q[1] = s.cam_pose.rotation.x();
  cam->q[2] = s.cam_pose.rotation.y();
  cam->q[3] = s.cam_pose.rotation.z();
  for (int a = 0; a < 3; ++a) cam->t[a] = s.cam_pose.translation[a];
  cam->fx = s.intrinsics.fx;
  cam->fy = s.intrinsics.fy;
  cam->cx = s.intrinsics.cx;
  cam->cy = s.intrinsics.cy;
  cam->width = s.intrinsics.width;
  cam->height = s.intrinsics.height;
  *cfg = RefConfig{s.config.near_plane, s.config.dilation,          s.config.alpha_clamp,
                   s.config.alpha_skip, s.config.transmittance_min, s.config.radius_sigma};
  std::memcpy(w_rgb, s.w_rgb.data.data(), sizeof(double) * s.w_rgb.data.size());
  std::memcpy(w_depth, s.w_depth.data.data(), sizeof(double) * s.w_depth.data.size());
  std::memcpy(w_feat, s.w_feat.data.data(), sizeof(double) * s.w_feat.data.size());
}

// legotest::gradcheck_scene on the seeded scene: max relative error (gradcheck.hpp:105-148).
REF_API double ref_gradcheck(int n, int size, int d, uint64_t seed) {
  auto s = legotest::make_grad_scene(n, size, d, seed);
  return legotest::gradcheck_scene(s).max_rel_error;
}

// CPU arm of bench.py --impl reference: `threads` host threads each run `iters` full steps of the
// reference path -- lego::render, the L1 cotangents against the targets, lego::render_backward --
// on one shared const map (render is pure w.r.t. the map).  Returns wall seconds of
// the whole batch; *loss = the last step's L1 loss.
REF_API double ref_bench(const RefMap* m, const RefCamera* cam, const RefConfig* cfg, const double* trgb,
                         const double* tdepth, const double* tfeat, int threads, int iters, double* loss) {
  const auto map = build_map(m);
  const auto pose = to_pose(cam);
  const auto k = to_k(cam);
  const auto rc = to_cfg(cfg);
  std::vector<double> losses(threads > 0 ? threads : 1, 0.0);
  const auto t0 = std::chrono::steady_clock::now();
  auto work = [&](int t) {
    for (int it = 0; it < iters; ++it) {
      const auto out = lego::render(map, pose, k, rc);
      lego::ImageD gr, gd, gf;
      l1_cot(out, trgb, tdepth, tfeat, gr, gd, gf);
      const auto g = lego::render_backward(map, out, gr, gd, gf);
      double l = 0;
      for (std::size_t i = 0; i < out.rgb.data.size(); ++i) l += std::abs(out.rgb.data[i] - trgb[i]) / out.rgb.data.size();
      losses[t] = l + g.opacity_logit.size() * 0.0;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (loss) *loss = losses[0];
  return sec;
}

// CPU arm with all host threads: one step = the full image's fwd + bwd split into `threads` row
// bands, each thread running the reference's own lego::render + lego::render_backward on its band
// (the band camera is the full camera with cy shifted and the band's height: the reference culls
// against the band, keeps the global (depth, index) order, and its pixels are exactly the full
// image's rows; gradients are sums over pixels, so the bands' gradients sum to the full one).
// This is the per-pixel data parallelism SPEC.md:298-299 allows.  Returns wall seconds per step;
// *loss = the image's L1 loss of the last step.
REF_API double ref_bench_bands(const RefMap* m, const RefCamera* cam, const RefConfig* cfg, const double* trgb,
                               const double* tdepth, const double* tfeat, int threads, int iters, double* loss) {
  const auto map = build_map(m);
  const auto pose = to_pose(cam);
  const auto rc = to_cfg(cfg);
  const int H = cam->height, W = cam->width, d = m->d;
  threads = std::max(1, std::min(threads, H));
  std::vector<double> band_loss((size_t)threads, 0.0);
  const double inv_rgb = 1.0 / (3.0 * W * H), inv_d = 1.0 / ((double)W * H), inv_f = d ? 1.0 / ((double)d * W * H) : 0;
  auto sgn = [](double x) { return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); };
  auto band = [&](int t) {
    const int y0 = (int)((int64_t)H * t / threads), y1 = (int)((int64_t)H * (t + 1) / threads);
    lego::CameraIntrinsics k = to_k(cam);
    k.cy = cam->cy - y0;
    k.height = y1 - y0;
    if (k.height <= 0) return;
    const auto out = lego::render(map, pose, k, rc);
    lego::ImageD gr(k.height, W, 3), gd(k.height, W, 1), gf(k.height, W, d);
    double l = 0.0;
    const size_t off = (size_t)y0 * W;
    for (size_t i = 0; i < gr.data.size(); ++i) {
      const double df = out.rgb.data[i] - trgb[off * 3 + i];
      gr.data[i] = sgn(df) * inv_rgb;
      l += std::abs(df) * inv_rgb;
    }
    for (size_t i = 0; i < gd.data.size(); ++i) {
      const double df = out.depth.data[i] - tdepth[off + i];
      gd.data[i] = sgn(df) * inv_d;
      l += std::abs(df) * inv_d;
    }
    for (size_t i = 0; i < gf.data.size(); ++i) {
      const double df = out.feat.data[i] - tfeat[off * d + i];
      gf.data[i] = sgn(df) * inv_f;
      l += std::abs(df) * inv_f;
    }
    const auto g = lego::render_backward(map, out, gr, gd, gf);
    band_loss[(size_t)t] = l + 0.0 * g.opacity_logit.size();
  };
  const auto t0 = std::chrono::steady_clock::now();
  for (int it = 0; it < iters; ++it) {
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(band, t);
    band(0);
    for (auto& th : pool) th.join();
  }
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (loss) {
    double s = 0.0;
    for (double v : band_loss) s += v;
    *loss = s;
  }
  return sec / std::max(1, iters);
}

// ---- map pruning (Eq. 4; the reference's pruning.cpp is a placeholder) ----------
// The greedy ascending-index sweep of the SPEC run on the reference's own KD-tree
// (kdtree.hpp: KdTree3::knn_if, exact k nearest among the accepted points, ties by index), with
// the live filter and self-exclusion as the predicate.  d2 is KdTree3's (p - q).squaredNorm();
// the cosine is restated as in oracle/prune_oracle.c.  pos [n][3], feat [d][n].
REF_API int64_t ref_find_language_redundant(int64_t n, int32_t d, const double* pos, const double* feat, int32_t k,
                                            double tau_dist, double tau_sim, uint8_t* flags) {
  std::fill(flags, flags + n, uint8_t(0));
  if (n < 2 || d <= 0 || k <= 0) return 0;
  std::vector<lego::Vec3> pts((size_t)n);
  for (int64_t i = 0; i < n; ++i) pts[(size_t)i] = lego::Vec3(pos[i * 3 + 0], pos[i * 3 + 1], pos[i * 3 + 2]);
  const lego::KdTree3 tree(pts);
  std::vector<double> norm((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int32_t c = 0; c < d; ++c) s += feat[(int64_t)c * n + i] * feat[(int64_t)c * n + i];
    norm[(size_t)i] = std::sqrt(s);
  }
  const double tau2 = tau_dist * tau_dist;
  std::vector<lego::KdTree3::Neighbor> nn;
  int64_t marked = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (flags[i]) continue;
    const auto live_other = [&](int j) { return j != (int)i && !flags[j]; };
    tree.knn_if(pts[(size_t)i], k, live_other, nn);
    for (const auto& nb : nn) {
      const int64_t j = nb.index;
      if (!(nb.dist_sq < tau2)) continue;
      if (!(norm[(size_t)i] > 0.0) || !(norm[(size_t)j] > 0.0)) continue;
      double dot = 0.0;
      for (int32_t c = 0; c < d; ++c) dot += feat[(int64_t)c * n + i] * feat[(int64_t)c * n + j];
      if (dot / (norm[(size_t)i] * norm[(size_t)j]) > tau_sim) {
        flags[j] = 1;
        ++marked;
      }
    }
  }
  return marked;
}
