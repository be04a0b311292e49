/* lgs_c_demo.c -- a plain C99 program against the C ABI (include/lgs.h), linked with liblgs.so.
 *
 * Built by __graft_entry__.build() (gcc), run on a GPU by tests/test_gpu_c_abi.py.  Restates three
 * renderer tests of the reference (proj/tests/test_renderer.cpp) through the ABI a C / cgo / FFI
 * caller would use:
 *   - test_renderer.cpp:95-106  two coincident splats composite front to back (0.5, 0.25);
 *   - test_renderer.cpp:175-187 d rgb(centre) / d colour = acc(centre) for a single splat;
 *   - test_renderer.cpp:189-196 a mismatched cotangent shape is LGS_EINVAL (std::invalid_argument).
 * Exit code 0 when all hold. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lgs.h"

#define W 64
#define H 64
#define D 4

static int failures = 0;

static void expect(int ok, const char* what) {
  printf("[%s] %s\n", ok ? "pass" : "FAIL", what);
  if (!ok) ++failures;
}

static int check(lgs_status s, const char* call) {
  if (s != LGS_OK) printf("%s -> %d (%s)\n", call, (int)s, lgs_last_error());
  return s == LGS_OK;
}

/* n splats at (0, 0, z[i]) with the given isotropic scale, logit and colour (test_renderer.cpp:22-32) */
static lgs_gaussians splats(int n, const double* z, double scale, const double* logit, const double (*col)[3],
                            float* buf) {
  float* pos = buf;
  float* rot = pos + 3 * n;
  float* ls = rot + 4 * n;
  float* op = ls + 3 * n;
  float* sh = op + n;
  float* feat = sh + 3 * n;
  for (int i = 0; i < n; ++i) {
    pos[3 * i] = 0.f; pos[3 * i + 1] = 0.f; pos[3 * i + 2] = (float)z[i];
    rot[4 * i] = rot[4 * i + 1] = rot[4 * i + 2] = 0.f; rot[4 * i + 3] = 1.f; /* x, y, z, w */
    for (int a = 0; a < 3; ++a) { ls[3 * i + a] = (float)log(scale); sh[3 * i + a] = (float)col[i][a]; }
    op[i] = (float)logit[i];
    for (int c = 0; c < D; ++c) feat[c * n + i] = 0.f;
  }
  lgs_gaussians g;
  memset(&g, 0, sizeof g);
  g.n = n; g.feature_dim = D; g.sh_degree = 0;
  g.positions = pos; g.rotations = rot; g.log_scales = ls; g.opacity_logits = op; g.sh = sh; g.features = feat;
  g.memory = LGS_MEM_HOST;
  return g;
}

int main(void) {
  lgs_ctx* ctx = NULL;
  if (!check(lgs_ctx_create(0, NULL, &ctx), "lgs_ctx_create")) return 2;
  printf("%s\n", lgs_version());
  lgs_camera cam;  /* test_renderer.cpp:14-20: fx = fy = 100, c = 31.5, 64 x 64, identity pose */
  memset(&cam, 0, sizeof cam);
  cam.q[0] = 1.0;
  cam.fx = cam.fy = 100.0; cam.cx = cam.cy = 31.5; cam.width = W; cam.height = H;
  const lgs_render_config cfg = lgs_render_config_default();
  static float rgb[H * W * 3], depth[H * W], feat[H * W * D], acc[H * W];
  lgs_images img = {rgb, depth, feat, acc, LGS_MEM_HOST};
  float* buf = (float*)calloc(2 * (14 + D), sizeof(float));

  { /* two coincident splats, opacity 0.5 each, red in front of green */
    const double z[2] = {1.0, 1.0001}, logit[2] = {0.0, 0.0}, col[2][3] = {{1, 0, 0}, {0, 1, 0}};
    lgs_gaussians g = splats(2, z, 0.5, logit, col, buf);
    lgs_saved* tape = NULL;
    if (check(lgs_render(ctx, &g, &cam, &cfg, &img, &tape), "lgs_render")) {
      const float* p = rgb + (31 * W + 31) * 3;
      expect(fabs(p[0] - 0.5) < 1e-3 && fabs(p[1] - 0.25) < 1e-3, "two coincident splats: 0.5 / 0.25");
    } else {
      ++failures;
    }
    lgs_saved_destroy(tape);
  }
  { /* single splat: d rgb(centre, r) / d colour_r = acc(centre) */
    const double z[1] = {1.0}, logit[1] = {log(0.8 / 0.2)}, col[1][3] = {{0.3, 0.3, 0.3}};
    lgs_gaussians g = splats(1, z, 0.2, logit, col, buf);
    lgs_saved* tape = NULL;
    if (check(lgs_render(ctx, &g, &cam, &cfg, &img, &tape), "lgs_render")) {
      static float grgb[H * W * 3];
      memset(grgb, 0, sizeof grgb);
      grgb[(31 * W + 31) * 3] = 1.f;
      float gpos[3], grot[4], gls[3], gop[1], gcol[3], gfeat[D];
      lgs_map_grads mg = {gpos, grot, gls, gop, gcol, gfeat, LGS_MEM_HOST, 0};
      lgs_cotangents cot;
      memset(&cot, 0, sizeof cot);
      cot.rgb = grgb;
      cot.memory = LGS_MEM_HOST;
      cot.rgb_shape[0] = H; cot.rgb_shape[1] = W; cot.rgb_shape[2] = 3;
      if (check(lgs_render_backward(ctx, tape, &cot, &mg, NULL), "lgs_render_backward")) {
        const float a = acc[31 * W + 31];
        expect(fabs(gcol[0] - a) <= 1e-6 * fabs(a) && gcol[1] == 0.f, "colour gradient = acc at the centre");
      } else {
        ++failures;
      }
      cot.rgb_shape[0] = 8; cot.rgb_shape[1] = 8;  /* the reference's ImageD(8, 8, 3) */
      expect(lgs_render_backward(ctx, tape, &cot, &mg, NULL) == LGS_EINVAL, "mismatched cotangent -> LGS_EINVAL");
    } else {
      ++failures;
    }
    lgs_saved_destroy(tape);
  }
  free(buf);
  lgs_ctx_destroy(ctx);
  printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
