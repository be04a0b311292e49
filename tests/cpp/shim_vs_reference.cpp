// The C++ drop-in (include/legoslam_gpu.hpp) against the reference itself, in one program.
//
// Built by oracle/Makefile (needs /root/reference: the reference headers, renderer.cpp and
// geometry.cpp, unmodified, against oracle/eigen_shim) and linked with liblgs.so; run on a GPU by
// tests/test_gpu_c_abi.py::test_cpp_drop_in_against_the_reference.  lego::gpu::render /
// render_backward are called with exactly the
// arguments lego::render / lego::render_backward take (renderer.hpp:55-56, 72-74) on:
//   * the reference's own gradcheck scene (gradcheck.hpp:31-78, seed 101; no thresholds active):
//     every image value within 1e-4 rel / 1e-5 abs, every gradient within 1e-3 (rel. to the
//     component, 1e-2 of the group's RMS floor) -- same bar as tests/parity.py;
//   * scenes of proj/tests/test_renderer.cpp (single opaque splat, coincident splats);
//   * a seeded 64x64 scene of 400 Gaussians with the default thresholds: images within tolerance
//     except pixels where a threshold decision flips between fp32 and fp64 (at most 0.5%);
//   * the error convention: a mismatched cotangent shape throws std::invalid_argument.
// Exit code 0 when everything holds; one line per check.
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "gradcheck.hpp"
#include "legoslam_gpu.hpp"
#include "legoslam/random.hpp"

using namespace lego;

namespace {

int failures = 0;

void report(bool ok, const std::string& what) {
  std::printf("[%s] %s\n", ok ? "pass" : "FAIL", what.c_str());
  if (!ok) ++failures;
}

// pixels (any channel) outside |gpu - ref| <= 1e-5 + 1e-4 |ref|
long outside(const ImageD& g, const ImageD& r, double* max_err) {
  long bad = 0;
  *max_err = 0.0;
  const int C = r.channels;
  for (std::size_t p = 0; p < r.data.size() / (std::size_t)C; ++p) {
    bool b = false;
    for (int c = 0; c < C; ++c) {
      const double e = std::abs(g.data[p * C + c] - r.data[p * C + c]);
      *max_err = std::max(*max_err, e);
      b = b || e > 1e-5 + 1e-4 * std::abs(r.data[p * C + c]);
    }
    bad += b;
  }
  return bad;
}

// components outside |gpu - ref| <= 1e-3 (|ref| + 1e-2 rms(group))
long grad_outside(const std::vector<double>& g, const std::vector<double>& r) {
  double ss = 0.0;
  for (double v : r) ss += v * v;
  const double floor = 1e-2 * std::sqrt(ss / std::max<std::size_t>(r.size(), 1));
  long bad = 0;
  for (std::size_t i = 0; i < r.size(); ++i) bad += std::abs(g[i] - r[i]) > 1e-3 * (std::abs(r[i]) + floor) + 1e-30;
  return bad;
}

std::vector<std::vector<double>> groups(const MapGradients& m) {
  std::vector<std::vector<double>> out(6);
  for (std::size_t i = 0; i < m.position.size(); ++i) {
    for (int a = 0; a < 3; ++a) {
      out[0].push_back(m.position[i][a]);
      out[2].push_back(m.log_scale[i][a]);
      out[4].push_back(m.color[i][a]);
    }
    for (int a = 0; a < 4; ++a) out[1].push_back(m.rotation[i][a]);
    out[3].push_back(m.opacity_logit[i]);
    for (int c = 0; c < m.feature.cols(); ++c) out[5].push_back(m.feature((Eigen::Index)i, c));
  }
  return out;
}

void compare(const char* name, const GaussianMap& map, const Pose& pose, const CameraIntrinsics& k,
             const RenderConfig& cfg, const ImageD& wr, const ImageD& wd, const ImageD& wf, double max_flip_frac) {
  const RenderOutput ro = render(map, pose, k, cfg);
  const RenderOutput go = gpu::render(map, pose, k, cfg);
  const long npix = (long)k.width * k.height;
  long worst = 0;
  double mx = 0.0, e = 0.0;
  for (auto im : {std::make_pair(&go.rgb, &ro.rgb), std::make_pair(&go.depth, &ro.depth),
                  std::make_pair(&go.feat, &ro.feat), std::make_pair(&go.acc, &ro.acc)}) {
    worst = std::max(worst, outside(*im.first, *im.second, &e));
    mx = std::max(mx, e);
  }
  char buf[256];
  std::snprintf(buf, sizeof buf, "%s: images, %ld of %ld pixels outside 1e-4/1e-5 (max err %.2e)", name, worst, npix,
                mx);
  report(worst <= (long)(max_flip_frac * npix), buf);
  const auto gr = groups(render_backward(map, ro, wr, wd, wf));
  const auto gg = groups(gpu::render_backward(map, go, wr, wd, wf));
  long gbad = 0, total = 0;
  for (int gi = 0; gi < 6; ++gi) {
    gbad += grad_outside(gg[gi], gr[gi]);
    total += (long)gr[gi].size();
  }
  std::snprintf(buf, sizeof buf, "%s: gradients, %ld of %ld components outside 1e-3", name, gbad, total);
  report(max_flip_frac == 0.0 ? gbad == 0 : gbad <= (long)(0.01 * total), buf);
}

LanguageGaussian splat_at(const Vec3& p, double scale, double opacity_logit, const Vec3& color, int d) {
  LanguageGaussian g;  // test_renderer.cpp:22-32
  g.position = p;
  g.rotation = Quat::Identity();
  g.log_scale = Vec3::Constant(std::log(scale));
  g.opacity_logit = opacity_logit;
  g.color = color;
  g.feature = Eigen::VectorXd::Zero(d);
  return g;
}

}  // namespace

int main() {
  try {
    // the reference's gradcheck scene and its weight images
    auto s = legotest::make_grad_scene(12, 16, 8, 101);
    compare("gradcheck scene (seed 101)", s.map, s.cam_pose, s.intrinsics, s.config, s.w_rgb, s.w_depth, s.w_feat,
            0.0);

    CameraIntrinsics k;  // test_renderer.cpp:14-20
    k.fx = k.fy = 100;
    k.cx = k.cy = 31.5;
    k.width = k.height = 64;
    Rng rng(7);
    auto weights = [&](int c) {
      ImageD w(k.height, k.width, c);
      for (auto& v : w.data) v = rng.uniform(-1, 1);
      return w;
    };
    {
      GaussianMap map(4);  // test_renderer.cpp:82-93
      map.insert(splat_at(Vec3(0, 0, 1.0), 0.2, std::log(0.99 / 0.01), Vec3(1, 0, 0), 4), 0);
      const RenderOutput o = gpu::render(map, Pose::identity(), k);
      report(std::abs(o.rgb.at(31, 31, 0) - 0.99) < 1e-3 && std::abs(o.depth.at(31, 31) - 1.0) < 1e-6,
             "single opaque splat: centre rgb 0.99, depth 1");
    }
    {
      GaussianMap map(4);  // test_renderer.cpp:95-106
      map.insert(splat_at(Vec3(0, 0, 1.0), 0.5, 0.0, Vec3(1, 0, 0), 4), 0);
      map.insert(splat_at(Vec3(0, 0, 1.0001), 0.5, 0.0, Vec3(0, 1, 0), 4), 0);
      const RenderOutput o = gpu::render(map, Pose::identity(), k);
      report(std::abs(o.rgb.at(31, 31, 0) - 0.5) < 1e-3 && std::abs(o.rgb.at(31, 31, 1) - 0.25) < 1e-3,
             "two coincident splats: 0.5 / 0.25 front to back");
    }
    {
      GaussianMap map(8);  // seeded scene, default thresholds
      for (int i = 0; i < 400; ++i) {
        LanguageGaussian g = splat_at(Vec3(rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), rng.uniform(0.8, 3.0)),
                                      rng.uniform(0.02, 0.09), rng.uniform(-1, 3),
                                      Vec3(rng.uniform(0, 1), rng.uniform(0, 1), rng.uniform(0, 1)), 8);
        Quat q(rng.normal(), rng.normal(), rng.normal(), rng.normal());
        g.rotation = q.normalized();
        g.log_scale = Vec3(std::log(rng.uniform(0.01, 0.08)), std::log(rng.uniform(0.01, 0.08)),
                           std::log(rng.uniform(0.01, 0.08)));
        for (int c = 0; c < 8; ++c) g.feature[c] = rng.normal();
        map.insert(g, 0);
      }
      const ImageD wr = weights(3), wd = weights(1), wf = weights(8);
      compare("seeded 400-Gaussian scene", map, Pose::identity(), k, RenderConfig{}, wr, wd, wf, 0.005);
      const RenderOutput o = gpu::render(map, Pose::identity(), k);
      bool threw = false;
      try {
        gpu::render_backward(map, o, ImageD(8, 8, 3), ImageD{}, ImageD{});
      } catch (const std::invalid_argument&) {
        threw = true;
      }
      report(threw, "mismatched cotangent shape throws std::invalid_argument");
    }
  } catch (const std::exception& e) {
    std::printf("[FAIL] exception: %s\n", e.what());
    ++failures;
  }
  std::printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
