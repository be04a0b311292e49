/*
 * lgs_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A plain-C restatement of the LEGO-SLAM reference CPU renderer so that the
 * CUDA rasterizer in paper_2511_16144_b200/ can be checked against it.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.
 *
 * Three parts:
 *
 *  (A) "oracle A": fp64, global (depth, index) sort, per-pixel contributor
 *      lists -- the reference algorithm of proj/src/renderer.cpp:11-356,
 *      restated without Eigen.  Every function cites the lines it follows.
 *      Extensions the reference does not have (SH degree 1..3 colour, the
 *      6-DoF camera-pose gradient, a pixel window for the sharded CPU
 *      baseline, injection of fp32 projected records) are marked EXT and are
 *      pinned by finite differences (tests/test_oracle_*.py), not by the
 *      reference.
 *
 *  (B) "oracle B": the fp32 twin of the product's preprocess kernel (same
 *      operation order, explicit fmaf, no contraction: build with
 *      -ffp-contract=off) plus tile-key duplication, stable sort and per-tile
 *      ranges.  Bit-exact parity target for the GPU key lists / order / ranges.
 *      Its projected records can be injected into (A) so the fp64 blend runs
 *      on exactly the Gaussians/pixel-rects the GPU used.
 *
 *  (C) Rng: std::mt19937_64 + the reference's own uniform/normal transforms
 *      (proj/include/legoslam/random.hpp:12-50), to rebuild the reference
 *      tests' seeded scenes bit-for-bit.
 *
 * Parity pinning: (A) is checked against the reference ITSELF -- its unmodified
 * renderer.cpp / geometry.cpp compiled by oracle/Makefile into oracle/_ref
 * (against the self-written Eigen subset in eigen_shim/) -- to fp64 rounding on
 * images, gradients, depth order and contributor counts
 * (tests/test_reference_build.py), and against the reference's own renderer
 * tests (proj/tests/test_renderer.cpp:38-204, also run unmodified against that
 * build), including the seed-101 finite-difference gradcheck
 * (gradcheck.hpp:31-148).  Part (D), map pruning, is in prune_oracle.c.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Types (plain C layouts, mirrored by oracle/oracle.py via ctypes)          */
/* ------------------------------------------------------------------------ */

/* renderer.hpp:15-22 (RenderConfig) */
typedef struct {
  double near_plane, dilation, alpha_clamp, alpha_skip, transmittance_min, radius_sigma;
} orc_config;

/* geometry.hpp:18-29 (Pose, world<-camera, q = w,x,y,z) + geometry.hpp:43-52 */
typedef struct {
  double q[4];
  double t[3];
  double fx, fy, cx, cy;
  int32_t width, height;
} orc_camera;

/* gaussian_map.hpp:57-93: SoA map.  rot is Eigen storage order (x,y,z,w);
 * feat is the column-major N x d Eigen matrix, i.e. [d][N]; sh is [N][K][3]
 * with K = (sh_degree+1)^2 (K = 1 is the reference `colors`). */
typedef struct {
  int64_t n;
  int32_t d;
  int32_t sh_degree;
  const double* pos;
  const double* rot;
  const double* log_s;
  const double* opac;
  const double* sh;
  const double* feat;
} orc_map;

/* EXT: fp32 projected records (from oracle B or the GPU) injected into (A). */
typedef struct {
  const uint8_t* visible;
  const float* u;
  const float* v;
  const float* conic; /* [N][3]: A, B, C with q = A dx^2 + 2B dx dy + C dy^2 */
  const float* depth;
  const int32_t* bbox; /* [N][4]: x0, x1, y0, y1 (inclusive pixel rect) */
  const float* opacity;
  const float* color; /* [N][3] */
} orc_inject;

/* renderer.hpp:24-31 (ProjectedGaussian) + cached opacity/colour/pixel rect */
typedef struct {
  double u, v;
  double cov[4];
  double conic[4];
  double depth;
  double radius;
  int64_t index;
  int32_t x0, x1, y0, y1;
  double opacity;
  double color[3];
} orc_proj;

typedef struct {
  int32_t* idx;
  int32_t n, cap;
} orc_list;

/* renderer.hpp:33-45 (RenderOutput) */
typedef struct {
  orc_map map;
  orc_camera cam;
  orc_config cfg;
  int32_t win[4]; /* x_lo, y_lo, x_hi, y_hi (half-open) */
  int32_t injected;
  int64_t np;
  orc_proj* proj; /* depth-sorted */
  orc_list* contrib;
  double* acc;
  double* depth;
  double rcw[9], tcw[3], cc[3];
  int64_t evaluated; /* (pixel, gaussian) pairs that reached the alpha test */
  int64_t contributions;
  /* EXT (injected records only): fp32 decision twin.  pix_flag [H*W]: bit 0 an alpha-skip
   * decision (renderer.cpp:147), bit 1 a transmittance decision (:140), bit 2 a backward clamp
   * decision (:274) differs between fp64 and the kernel's fp32 arithmetic, or the fp32 value lies
   * within its rounding band of the threshold.  g_flag [N] (map index): bit 0 the Gaussian took
   * part in such a decision, bit 1 it contributes at a pixel with bit 0|1 set (its gradient sees
   * the flipped compositing chain), bit 2 its clamp decision was marginal at some pixel. */
  uint8_t* pix_flag;
  uint8_t* g_flag;
} orc_render;

/* ------------------------------------------------------------------------ */
/* Small fp64 linear algebra (replaces the Eigen call sites of the path)     */
/* ------------------------------------------------------------------------ */

/* Eigen Quaternion::toRotationMatrix for a unit quaternion (w,x,y,z). */
static void quat_to_rot(double w, double x, double y, double z, double r[9]) {
  const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  r[0] = 1 - (tyy + tzz); r[1] = txy - twz;       r[2] = txz + twy;
  r[3] = txy + twz;       r[4] = 1 - (txx + tzz); r[5] = tyz - twx;
  r[6] = txz - twy;       r[7] = tyz + twx;       r[8] = 1 - (txx + tyy);
}

static void mat3_mul(const double a[9], const double b[9], double c[9]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      c[i * 3 + j] = a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j] + a[i * 3 + 2] * b[2 * 3 + j];
}

static void mat3_mul_bt(const double a[9], const double b[9], double c[9]) { /* a * b^T */
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      c[i * 3 + j] = a[i * 3 + 0] * b[j * 3 + 0] + a[i * 3 + 1] * b[j * 3 + 1] + a[i * 3 + 2] * b[j * 3 + 2];
}

static void mat3_mul_at(const double a[9], const double b[9], double c[9]) { /* a^T * b */
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      c[i * 3 + j] = a[0 * 3 + i] * b[0 * 3 + j] + a[1 * 3 + i] * b[1 * 3 + j] + a[2 * 3 + i] * b[2 * 3 + j];
}

/* Camera setup: geometry.hpp:23 (Pose normalizes q), geometry.cpp:15-20
 * (inverse: conjugate rotation, t' = -(q* t)).  The product host code
 * (csrc/lgs_host.cpp lgs_camera_setup) uses this same double formula. */
static void camera_setup(const orc_camera* cam, double rcw[9], double tcw[3], double cc[3]) {
  double w = cam->q[0], x = cam->q[1], y = cam->q[2], z = cam->q[3];
  const double nrm = sqrt(w * w + x * x + y * y + z * z);
  w /= nrm; x /= nrm; y /= nrm; z /= nrm;
  quat_to_rot(w, -x, -y, -z, rcw);
  for (int i = 0; i < 3; ++i)
    tcw[i] = -(rcw[i * 3 + 0] * cam->t[0] + rcw[i * 3 + 1] * cam->t[1] + rcw[i * 3 + 2] * cam->t[2]);
  for (int i = 0; i < 3; ++i) cc[i] = cam->t[i];
}

/* renderer.cpp:11 */
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

/* ------------------------------------------------------------------------ */
/* EXT: real spherical harmonics, degree <= 3.  Colour convention (unpinned  */
/* by the reference, which is SH0 only): colour = DC +          */
/* sum_{l>=1} Y_lm(dir) * coef, no C0 factor, no +0.5, no clamp, so SH0      */
/* reproduces the reference colour exactly.  dir = normalize(p - cam centre). */
/* ------------------------------------------------------------------------ */
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

static void sh_basis(int deg, double x, double y, double z, double b[16], double db[16][3]) {
  for (int k = 0; k < 16; ++k) { b[k] = 0; db[k][0] = db[k][1] = db[k][2] = 0; }
  b[0] = 1.0;
  if (deg < 1) return;
  b[1] = -SH_C1 * y; db[1][1] = -SH_C1;
  b[2] = SH_C1 * z;  db[2][2] = SH_C1;
  b[3] = -SH_C1 * x; db[3][0] = -SH_C1;
  if (deg < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  b[4] = SH_C2[0] * x * y;                db[4][0] = SH_C2[0] * y; db[4][1] = SH_C2[0] * x;
  b[5] = SH_C2[1] * y * z;                db[5][1] = SH_C2[1] * z; db[5][2] = SH_C2[1] * y;
  b[6] = SH_C2[2] * (2 * zz - xx - yy);   db[6][0] = -2 * SH_C2[2] * x; db[6][1] = -2 * SH_C2[2] * y; db[6][2] = 4 * SH_C2[2] * z;
  b[7] = SH_C2[3] * x * z;                db[7][0] = SH_C2[3] * z; db[7][2] = SH_C2[3] * x;
  b[8] = SH_C2[4] * (xx - yy);            db[8][0] = 2 * SH_C2[4] * x; db[8][1] = -2 * SH_C2[4] * y;
  if (deg < 3) return;
  b[9] = SH_C3[0] * y * (3 * xx - yy);
  db[9][0] = SH_C3[0] * 6 * x * y; db[9][1] = SH_C3[0] * (3 * xx - 3 * yy);
  b[10] = SH_C3[1] * x * y * z;
  db[10][0] = SH_C3[1] * y * z; db[10][1] = SH_C3[1] * x * z; db[10][2] = SH_C3[1] * x * y;
  b[11] = SH_C3[2] * y * (4 * zz - xx - yy);
  db[11][0] = SH_C3[2] * (-2 * x * y); db[11][1] = SH_C3[2] * (4 * zz - xx - 3 * yy); db[11][2] = SH_C3[2] * 8 * y * z;
  b[12] = SH_C3[3] * z * (2 * zz - 3 * xx - 3 * yy);
  db[12][0] = SH_C3[3] * (-6 * x * z); db[12][1] = SH_C3[3] * (-6 * y * z); db[12][2] = SH_C3[3] * (6 * zz - 3 * xx - 3 * yy);
  b[13] = SH_C3[4] * x * (4 * zz - xx - yy);
  db[13][0] = SH_C3[4] * (4 * zz - 3 * xx - yy); db[13][1] = SH_C3[4] * (-2 * x * y); db[13][2] = SH_C3[4] * 8 * x * z;
  b[14] = SH_C3[5] * z * (xx - yy);
  db[14][0] = SH_C3[5] * 2 * x * z; db[14][1] = SH_C3[5] * (-2 * y * z); db[14][2] = SH_C3[5] * (xx - yy);
  b[15] = SH_C3[6] * x * (xx - 3 * yy);
  db[15][0] = SH_C3[6] * (3 * xx - 3 * yy); db[15][1] = SH_C3[6] * (-6 * x * y);
}

static int sh_coeffs(int deg) { return (deg + 1) * (deg + 1); }

/* colour of Gaussian i for camera centre cc (renderer.cpp:128 for K = 1) */
static void eval_color(const orc_map* m, int64_t i, const double cc[3], double out[3]) {
  const int K = sh_coeffs(m->sh_degree);
  const double* c = m->sh + i * K * 3;
  if (K == 1) { out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; return; }
  double dx = m->pos[i * 3 + 0] - cc[0], dy = m->pos[i * 3 + 1] - cc[1], dz = m->pos[i * 3 + 2] - cc[2];
  const double n = sqrt(dx * dx + dy * dy + dz * dz);
  if (n > 0) { dx /= n; dy /= n; dz /= n; }
  double b[16], db[16][3];
  sh_basis(m->sh_degree, dx, dy, dz, b, db);
  for (int ch = 0; ch < 3; ++ch) {
    double s = 0;
    for (int k = 0; k < K; ++k) s += b[k] * c[k * 3 + ch];
    out[ch] = s;
  }
}

/* ------------------------------------------------------------------------ */
/* (A) project_gaussian  -- renderer.cpp:53-92 (+ proj_jacobian :14-21)      */
/* ------------------------------------------------------------------------ */
static int project_one(const orc_map* m, int64_t i, const orc_camera* k, const orc_config* cfg,
                       const double rcw[9], const double tcw[3], orc_proj* p) {
  const double* P = m->pos + i * 3;
  double t[3];
  for (int r = 0; r < 3; ++r) t[r] = rcw[r * 3 + 0] * P[0] + rcw[r * 3 + 1] * P[1] + rcw[r * 3 + 2] * P[2] + tcw[r];
  if (t[2] <= cfg->near_plane) return 0; /* :60 */

  /* :63 rotations are stored x,y,z,w; normalized() then toRotationMatrix() */
  const double* q = m->rot + i * 4;
  const double qn = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  double rg[9];
  quat_to_rot(q[3] / qn, q[0] / qn, q[1] / qn, q[2] / qn, rg);
  double s2[3];
  for (int a = 0; a < 3; ++a) s2[a] = exp(2.0 * m->log_s[i * 3 + a]); /* :64 */
  double rs[9], sigma3[9], tmp[9], sigmac[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) rs[r * 3 + c] = rg[r * 3 + c] * s2[c];
  mat3_mul_bt(rs, rg, sigma3);   /* :65 R S^2 R^T */
  mat3_mul(rcw, sigma3, tmp);
  mat3_mul_bt(tmp, rcw, sigmac); /* :66 */

  /* :68-71 J sigma_c J^T + dilation */
  const double z = t[2];
  const double j[6] = {k->fx / z, 0.0, -k->fx * t[0] / (z * z), 0.0, k->fy / z, -k->fy * t[1] / (z * z)};
  double js[6];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c)
      js[r * 3 + c] = j[r * 3 + 0] * sigmac[0 * 3 + c] + j[r * 3 + 1] * sigmac[1 * 3 + c] + j[r * 3 + 2] * sigmac[2 * 3 + c];
  double cov[4];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c)
      cov[r * 2 + c] = js[r * 3 + 0] * j[c * 3 + 0] + js[r * 3 + 1] * j[c * 3 + 1] + js[r * 3 + 2] * j[c * 3 + 2];
  cov[0] += cfg->dilation;
  cov[3] += cfg->dilation;

  /* :74-76 */
  const double mid = 0.5 * (cov[0] + cov[3]);
  const double det = cov[0] * cov[3] - cov[1] * cov[2];
  const double lam = mid + sqrt(fmax(mid * mid - det, 0.0));

  p->u = k->fx * t[0] / t[2] + k->cx; /* :79-81 */
  p->v = k->fy * t[1] / t[2] + k->cy;
  p->depth = t[2];
  memcpy(p->cov, cov, sizeof cov);
  p->radius = cfg->radius_sigma * sqrt(lam); /* :83 */
  p->index = i;
  /* :86-89 */
  if (p->u + p->radius < -0.5 || p->u - p->radius > k->width - 0.5 || p->v + p->radius < -0.5 ||
      p->v - p->radius > k->height - 0.5)
    return 0;
  /* :90 Eigen 2x2 inverse (adjugate / determinant) */
  const double d2 = cov[0] * cov[3] - cov[1] * cov[2];
  p->conic[0] = cov[3] / d2;
  p->conic[1] = -cov[1] / d2;
  p->conic[2] = -cov[2] / d2;
  p->conic[3] = cov[0] / d2;
  /* :131-134 pixel rect.  The float clamp before the int conversion only
   * matters past 2^31 (the reference would be UB there). */
  const double fx0 = fmax(0.0, floor(p->u - p->radius));
  const double fx1 = fmin((double)(k->width - 1), ceil(p->u + p->radius));
  const double fy0 = fmax(0.0, floor(p->v - p->radius));
  const double fy1 = fmin((double)(k->height - 1), ceil(p->v + p->radius));
  p->x0 = (int32_t)fx0; p->x1 = (int32_t)fx1; p->y0 = (int32_t)fy0; p->y1 = (int32_t)fy1;
  return 1;
}

ORC_API int orc_project_gaussian(const orc_map* m, int64_t i, const orc_camera* cam, const orc_config* cfg,
                                 double out_uv_depth_radius[4], double out_cov[4], double out_conic[4]) {
  double rcw[9], tcw[3], cc[3];
  camera_setup(cam, rcw, tcw, cc);
  orc_proj p;
  if (!project_one(m, i, cam, cfg, rcw, tcw, &p)) return 0;
  out_uv_depth_radius[0] = p.u; out_uv_depth_radius[1] = p.v;
  out_uv_depth_radius[2] = p.depth; out_uv_depth_radius[3] = p.radius;
  memcpy(out_cov, p.cov, sizeof p.cov);
  memcpy(out_conic, p.conic, sizeof p.conic);
  return 1;
}

/* renderer.cpp:114-117: (depth asc, map index asc) */
static int cmp_proj(const void* a, const void* b) {
  const orc_proj* x = (const orc_proj*)a;
  const orc_proj* y = (const orc_proj*)b;
  if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
  return (x->index > y->index) - (x->index < y->index);
}

static void list_push(orc_list* l, int32_t v) {
  if (l->n == l->cap) {
    l->cap = l->cap ? l->cap * 2 : 8;
    l->idx = (int32_t*)realloc(l->idx, sizeof(int32_t) * (size_t)l->cap);
  }
  l->idx[l->n++] = v;
}

/* EXT fp32 decision twin: the kernels' per-(tile, entry) conic frame (blend_common.cuh
 * stage_frame), the same IEEE fp64 operations in the same order (-ffp-contract=off), rounded to
 * fp32: out = S0, T0, ux, uy, wx, wy, dxc, dyc. */
static void twin_frame(float u, float v, float A, float B, float C, float xc, float yc, float out[8]) {
  const double a = A, b = B, c = C, k = 0.72134752044448170368;
  const double h = 0.5 * (a - c);
  const double r = sqrt(fma(h, h, b * b));
  const double l1 = 0.5 * (a + c) + r;
  double l2 = fma(a, c, -(b * b)) / l1;
  if (!(l2 > 0.0)) l2 = 0.0;
  double ex, ey;
  if (h >= 0.0) { ex = h + r; ey = b; } else { ex = b; ey = r - h; }
  const double nrm = sqrt(fma(ex, ex, ey * ey));
  double cx = 1.0, cy = 0.0;
  if (nrm > 0.0) { cx = ex / nrm; cy = ey / nrm; }
  const double a1 = sqrt(k * l1), a2 = sqrt(k * l2);
  const double dxc = (double)xc - (double)u, dyc = (double)yc - (double)v;
  out[0] = (float)(a1 * fma(cx, dxc, cy * dyc));
  out[1] = (float)(a2 * fma(cx, dyc, -(cy * dxc)));
  out[2] = (float)(a1 * cx);
  out[3] = (float)(a1 * cy);
  out[4] = (float)(-(a2 * cy));
  out[5] = (float)(a2 * cx);
  out[6] = (float)dxc;
  out[7] = (float)dyc;
}

/* ------------------------------------------------------------------------ */
/* (A) render -- renderer.cpp:94-167                                          */
/* rgb [H][W][3], depth [H][W], feat [H][W][d], acc [H][W] (HWC, image.hpp).  */
/* win: NULL = whole image (EXT: half-open pixel window x_lo,y_lo,x_hi,y_hi). */
/* ------------------------------------------------------------------------ */
ORC_API orc_render* orc_render_forward(const orc_map* m, const orc_camera* cam, const orc_config* cfg,
                                       const orc_inject* inj, const int32_t* win, double* rgb,
                                       double* depth, double* feat, double* acc) {
  orc_render* R = (orc_render*)calloc(1, sizeof(orc_render));
  R->map = *m;
  R->cam = *cam;
  R->cfg = *cfg;
  const int W = cam->width, H = cam->height, d = m->d;
  if (win) memcpy(R->win, win, sizeof R->win);
  else { R->win[0] = 0; R->win[1] = 0; R->win[2] = W; R->win[3] = H; }
  R->injected = inj != NULL;
  camera_setup(cam, R->rcw, R->tcw, R->cc);

  const size_t npix = (size_t)W * H;
  memset(rgb, 0, sizeof(double) * npix * 3);
  memset(depth, 0, sizeof(double) * npix);
  if (d > 0) memset(feat, 0, sizeof(double) * npix * (size_t)d);
  memset(acc, 0, sizeof(double) * npix);
  R->contrib = (orc_list*)calloc(npix, sizeof(orc_list));
  R->acc = acc;
  R->depth = depth;

  /* :106-111 project */
  R->proj = (orc_proj*)malloc(sizeof(orc_proj) * (size_t)(m->n > 0 ? m->n : 1));
  int64_t np = 0;
  for (int64_t i = 0; i < m->n; ++i) {
    orc_proj* p = &R->proj[np];
    if (inj) {
      if (!inj->visible[i]) continue;
      memset(p, 0, sizeof *p);
      p->u = inj->u[i]; p->v = inj->v[i]; p->depth = inj->depth[i];
      p->conic[0] = inj->conic[i * 3 + 0];
      p->conic[1] = p->conic[2] = inj->conic[i * 3 + 1];
      p->conic[3] = inj->conic[i * 3 + 2];
      p->index = i;
      p->x0 = inj->bbox[i * 4 + 0]; p->x1 = inj->bbox[i * 4 + 1];
      p->y0 = inj->bbox[i * 4 + 2]; p->y1 = inj->bbox[i * 4 + 3];
      p->opacity = inj->opacity[i];
      for (int c = 0; c < 3; ++c) p->color[c] = inj->color[i * 3 + c];
    } else {
      if (!project_one(m, i, cam, cfg, R->rcw, R->tcw, p)) continue;
      p->opacity = sigmoid(m->opac[i]);       /* :127 */
      eval_color(m, i, R->cc, p->color);      /* :128 (+ EXT SH) */
    }
    ++np;
  }
  R->np = np;
  qsort(R->proj, (size_t)np, sizeof(orc_proj), cmp_proj); /* :114-117 */

  double* trans = (double*)malloc(sizeof(double) * npix); /* :120-123 */
  double* draw = (double*)calloc(npix, sizeof(double));
  for (size_t i = 0; i < npix; ++i) trans[i] = 1.0;

  const int wx0 = R->win[0], wy0 = R->win[1], wx1 = R->win[2] - 1, wy1 = R->win[3] - 1;
  int64_t evaluated = 0, contributions = 0;
  /* EXT fp32 decision twin (see orc_render.pix_flag): the kernel's per-pair arithmetic
   * (blend_common.cuh splat_alpha: conic pre-scaled by -log2(e)/2, _rn products, exp2) */
  float* t32 = NULL;
  const float skip_f = (float)cfg->alpha_skip, tmin_f = (float)cfg->transmittance_min;
  const float clamp_f = (float)cfg->alpha_clamp;
  if (inj) {
    t32 = (float*)malloc(sizeof(float) * npix);
    for (size_t i = 0; i < npix; ++i) t32[i] = 1.0f;
    R->pix_flag = (uint8_t*)calloc(npix, 1);
    R->g_flag = (uint8_t*)calloc((size_t)(m->n > 0 ? m->n : 1), 1);
  }
  for (int64_t gi = 0; gi < np; ++gi) { /* :125-161 */
    const orc_proj* g = &R->proj[gi];
    const double opacity = g->opacity;
    const double* color = g->color;
    const int64_t mi = g->index;
    const int x0 = g->x0 > wx0 ? g->x0 : wx0, x1 = g->x1 < wx1 ? g->x1 : wx1;
    const int y0 = g->y0 > wy0 ? g->y0 : wy0, y1 = g->y1 < wy1 ? g->y1 : wy1;
    const double cs = g->conic[1] + g->conic[2];
    int frame_tile = -1; /* EXT fp32 twin: conic frame of the current tile */
    float frame[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int y = y0; y <= y1; ++y) {
      for (int x = x0; x <= x1; ++x) {
        const size_t pix = (size_t)y * W + x;
        double* t_pix = &trans[pix];
        float a32 = 0.0f;
        int skip32 = 1;
        if (t32) { /* EXT fp32 twin of the decisions at this pair */
          const int tskip32 = t32[pix] < tmin_f;
          if (tskip32 != (*t_pix < cfg->transmittance_min)) {
            R->pix_flag[pix] |= 2;
            R->g_flag[mi] |= 1;
          }
          if (!tskip32) {
            /* the kernels' conic frame of this (tile, Gaussian), blend_common.cuh stage_frame */
            const int tid_ = (y / 16) * 65536 + (x / 16);
            if (tid_ != frame_tile) {
              frame_tile = tid_;
              twin_frame((float)g->u, (float)g->v, (float)g->conic[0], (float)g->conic[1], (float)g->conic[3],
                         (float)((x / 16) * 16) + 7.5f, (float)((y / 16) * 16) + 7.5f, frame);
            }
            const float fex = (float)(x % 16) - 7.5f, fey = (float)(y % 16) - 7.5f;
            const float S = fmaf(frame[2], fex, fmaf(frame[3], fey, frame[0]));
            const float Tt = fmaf(frame[4], fex, fmaf(frame[5], fey, frame[1]));
            const float p = -fmaf(S, S, Tt * Tt);
            a32 = (float)opacity * exp2f(p);
            skip32 = !(a32 >= skip_f);
            const double qq = g->conic[0] * (x - g->u) * (x - g->u) + cs * (x - g->u) * (y - g->v) +
                              g->conic[3] * (y - g->v) * (y - g->v);
            const double a64 = opacity * exp(-0.5 * qq);
            if (*t_pix >= cfg->transmittance_min &&
                (skip32 != !(a64 >= cfg->alpha_skip) || fabsf(a32 - skip_f) <= 4e-6f * skip_f)) {
              R->pix_flag[pix] |= 1;
              R->g_flag[mi] |= 1;
            }
            if (!skip32) {
              const double g64 = exp(-0.5 * qq);
              if (((opacity * g64 > cfg->alpha_clamp) != (a32 > clamp_f)) || fabsf(a32 - clamp_f) <= 4e-6f * clamp_f) {
                R->pix_flag[pix] |= 4;
                R->g_flag[mi] |= 4;
              }
              t32[pix] = t32[pix] * (1.0f - fminf(a32, clamp_f));
              if (fabsf(t32[pix] - tmin_f) <= 2e-5f * tmin_f) {
                R->pix_flag[pix] |= 2;
                R->g_flag[mi] |= 1;
              }
            }
          }
        }
        if (*t_pix < cfg->transmittance_min) continue; /* :140 */
        ++evaluated;
        const double dx = x - g->u, dy = y - g->v;
        const double q = g->conic[0] * dx * dx + cs * dx * dy + g->conic[3] * dy * dy;
        double alpha = opacity * exp(-0.5 * q);
        if (!(alpha >= cfg->alpha_skip)) continue; /* :147 */
        if (alpha > cfg->alpha_clamp) alpha = cfg->alpha_clamp;
        const double w = alpha * *t_pix;
        double* px = rgb + pix * 3;
        for (int c = 0; c < 3; ++c) px[c] += w * color[c];
        double* ft = feat + pix * (size_t)d;
        for (int c = 0; c < d; ++c) ft[c] += w * m->feat[(int64_t)c * m->n + mi];
        draw[pix] += w * g->depth;
        acc[pix] += w;
        list_push(&R->contrib[pix], (int32_t)gi);
        ++contributions;
        *t_pix *= 1.0 - alpha;
      }
    }
  }
  for (size_t pix = 0; pix < npix; ++pix) /* :163-165 */
    depth[pix] = draw[pix] / fmax(acc[pix], 1e-6);
  if (t32) { /* EXT: every contributor of a pixel whose compositing chain may differ */
    for (size_t pix = 0; pix < npix; ++pix) {
      if (!(R->pix_flag[pix] & 3)) continue;
      const orc_list* cl = &R->contrib[pix];
      for (int32_t ci = 0; ci < cl->n; ++ci) R->g_flag[R->proj[cl->idx[ci]].index] |= 2;
    }
    free(t32);
  }
  free(trans);
  free(draw);
  R->evaluated = evaluated;
  R->contributions = contributions;
  return R;
}

ORC_API int64_t orc_render_num_projected(const orc_render* R) { return R->np; }
ORC_API int64_t orc_render_num_evaluated(const orc_render* R) { return R->evaluated; }
ORC_API int64_t orc_render_num_contributions(const orc_render* R) { return R->contributions; }

/* per pixel contributor count (for the GPU's per-pixel last-index parity) */
ORC_API void orc_render_contrib_counts(const orc_render* R, int32_t* out) {
  const size_t npix = (size_t)R->cam.width * R->cam.height;
  for (size_t i = 0; i < npix; ++i) out[i] = R->contrib[i].n;
}

/* EXT: fp32 decision-twin flags (injected renders only; returns 0 when absent) */
ORC_API int orc_render_flags(const orc_render* R, uint8_t* pix_flag, uint8_t* g_flag) {
  if (!R->pix_flag) return 0;
  const size_t npix = (size_t)R->cam.width * R->cam.height;
  if (pix_flag) memcpy(pix_flag, R->pix_flag, npix);
  if (g_flag) memcpy(g_flag, R->g_flag, (size_t)R->map.n);
  return 1;
}

/* sorted projected map indices */
ORC_API void orc_render_sorted_indices(const orc_render* R, int64_t* out) {
  for (int64_t i = 0; i < R->np; ++i) out[i] = R->proj[i].index;
}

ORC_API void orc_render_free(orc_render* R) {
  if (!R) return;
  const size_t npix = (size_t)R->cam.width * R->cam.height;
  for (size_t i = 0; i < npix; ++i) free(R->contrib[i].idx);
  free(R->contrib);
  free(R->proj);
  free(R->pix_flag);
  free(R->g_flag);
  free(R);
}

/* ------------------------------------------------------------------------ */
/* (A) render_backward -- renderer.cpp:169-356                                */
/* Cotangents may be NULL (= the reference's empty image, hpp:70-71).         */
/* Outputs are dense over the map (renderer.cpp:185-186):                     */
/*   g_pos [N][3], g_rot [N][4] in (w,x,y,z) (renderer.hpp:61), g_log_s       */
/*   [N][3], g_opac [N], g_sh [N][K][3], g_feat [d][N] (column-major N x d).  */
/* EXT: g_pose6 (nullable) = dL/dxi at xi = 0 for cam_pose <- compose(       */
/* se3_exp(xi), cam_pose), xi = (omega, nu) (geometry.hpp:13-14).             */
/* The depth/acc images the caller got from orc_render_forward must still be */
/* alive (the reference reads out.acc / out.depth, renderer.cpp:204-206).     */
/* ------------------------------------------------------------------------ */
ORC_API int orc_render_backward(const orc_render* R, const double* g_rgb, const double* g_depth,
                                const double* g_feat, double* o_pos, double* o_rot, double* o_logs,
                                double* o_opac, double* o_sh, double* o_feat, double* g_pose6) {
  const orc_map* m = &R->map;
  const orc_camera* k = &R->cam;
  const int W = k->width, d = m->d;
  const int K = sh_coeffs(m->sh_degree);
  const int64_t n = m->n, np = R->np;
  memset(o_pos, 0, sizeof(double) * (size_t)n * 3); /* :44-51 */
  memset(o_rot, 0, sizeof(double) * (size_t)n * 4);
  memset(o_logs, 0, sizeof(double) * (size_t)n * 3);
  memset(o_opac, 0, sizeof(double) * (size_t)n);
  memset(o_sh, 0, sizeof(double) * (size_t)n * K * 3);
  if (d > 0) memset(o_feat, 0, sizeof(double) * (size_t)n * d);
  if (g_pose6) memset(g_pose6, 0, sizeof(double) * 6);

  /* :188-192 per projected screen-space accumulators (+ colour for SH) */
  double* g_mu = (double*)calloc((size_t)np * 2 + 1, sizeof(double));
  double* g_con = (double*)calloc((size_t)np * 4 + 1, sizeof(double));
  double* g_cz = (double*)calloc((size_t)np + 1, sizeof(double));
  double* g_col = (double*)calloc((size_t)np * 3 + 1, sizeof(double));
  size_t cap = 64;
  double* alphas = (double*)malloc(sizeof(double) * cap);
  double* ts = (double*)malloc(sizeof(double) * cap);
  double* dldw = (double*)malloc(sizeof(double) * cap);

  for (int y = R->win[1]; y < R->win[3]; ++y) { /* :198-291 */
    for (int x = R->win[0]; x < R->win[2]; ++x) {
      const size_t pix = (size_t)y * W + x;
      const orc_list* cl = &R->contrib[pix];
      if (cl->n == 0) continue;
      const double acc = R->acc[pix];
      const double mm = fmax(acc, 1e-6);
      const double depth_norm = R->depth[pix];
      const double* grp = g_rgb ? g_rgb + pix * 3 : NULL;
      const double* gfp = (g_feat && d > 0) ? g_feat + pix * (size_t)d : NULL;
      const double g_d = g_depth ? g_depth[pix] : 0.0;
      const double g_draw = g_d / mm;                               /* :211 */
      const double g_acc = acc > 1e-6 ? -g_d * depth_norm / mm : 0.0; /* :212 */
      const size_t nc = (size_t)cl->n;
      if (nc > cap) {
        while (cap < nc) cap *= 2;
        alphas = (double*)realloc(alphas, sizeof(double) * cap);
        ts = (double*)realloc(ts, sizeof(double) * cap);
        dldw = (double*)realloc(dldw, sizeof(double) * cap);
      }
      double t_pix = 1.0; /* :219-231 */
      for (size_t ci = 0; ci < nc; ++ci) {
        const orc_proj* g = &R->proj[cl->idx[ci]];
        const double dx = x - g->u, dy = y - g->v;
        const double q = g->conic[0] * dx * dx + (g->conic[1] + g->conic[2]) * dx * dy + g->conic[3] * dy * dy;
        double a = g->opacity * exp(-0.5 * q);
        alphas[ci] = a < R->cfg.alpha_clamp ? a : R->cfg.alpha_clamp;
        ts[ci] = t_pix;
        t_pix *= 1.0 - alphas[ci];
      }
      for (size_t ci = 0; ci < nc; ++ci) { /* :233-246 */
        const orc_proj* g = &R->proj[cl->idx[ci]];
        double v = g_draw * g->depth + g_acc;
        if (grp) v += grp[0] * g->color[0] + grp[1] * g->color[1] + grp[2] * g->color[2];
        if (gfp)
          for (int c = 0; c < d; ++c) v += gfp[c] * m->feat[(int64_t)c * n + g->index];
        dldw[ci] = v;
      }
      double accum = 0.0; /* :248-289 */
      for (size_t r = nc; r-- > 0;) {
        const int32_t pj = cl->idx[r];
        const orc_proj* g = &R->proj[pj];
        const int64_t mi = g->index;
        const double alpha = alphas[r];
        const double w = alpha * ts[r];
        const double dl_dalpha = ts[r] * dldw[r] - accum / (1.0 - alpha);
        accum += dldw[r] * w;
        if (grp)
          for (int c = 0; c < 3; ++c) g_col[(size_t)pj * 3 + c] += grp[c] * w;
        if (gfp)
          for (int c = 0; c < d; ++c) o_feat[(int64_t)c * n + mi] += gfp[c] * w;
        g_cz[pj] += g_draw * w;
        const double opacity = g->opacity;
        const double dx = x - g->u, dy = y - g->v;
        const double cs = g->conic[1] + g->conic[2];
        const double q = g->conic[0] * dx * dx + cs * dx * dy + g->conic[3] * dy * dy;
        const double gauss = exp(-0.5 * q);
        if (opacity * gauss > R->cfg.alpha_clamp) continue; /* :274 */
        o_opac[mi] += dl_dalpha * gauss * opacity * (1.0 - opacity);
        const double dl_dg = dl_dalpha * opacity;
        const double dg_dq = -0.5 * gauss;
        const double dq_ddx = 2.0 * (g->conic[0] * dx) + cs * dy;
        const double dq_ddy = 2.0 * (g->conic[3] * dy) + cs * dx;
        g_mu[(size_t)pj * 2 + 0] += dl_dg * dg_dq * -dq_ddx;
        g_mu[(size_t)pj * 2 + 1] += dl_dg * dg_dq * -dq_ddy;
        g_con[(size_t)pj * 4 + 0] += dl_dg * dg_dq * dx * dx;
        g_con[(size_t)pj * 4 + 1] += dl_dg * dg_dq * dx * dy;
        g_con[(size_t)pj * 4 + 2] += dl_dg * dg_dq * dx * dy;
        g_con[(size_t)pj * 4 + 3] += dl_dg * dg_dq * dy * dy;
      }
    }
  }
  free(alphas); free(ts); free(dldw);

  /* :293-354 chain screen-space gradients to the 3D attributes */
  const double* rcw = R->rcw;
  const double* tcw = R->tcw;
  double pose[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t pj = 0; pj < np; ++pj) {
    const orc_proj* g = &R->proj[pj];
    const int64_t mi = g->index;
    const double* P = m->pos + mi * 3;
    double gpos_world[3] = {0, 0, 0}; /* everything that reaches the position */

    /* colour -> SH coefficients (K = 1: the reference's colour gradient) */
    const double* gc = g_col + (size_t)pj * 3;
    if (gc[0] != 0.0 || gc[1] != 0.0 || gc[2] != 0.0) {
      double* osh = o_sh + mi * K * 3;
      if (K == 1) {
        for (int c = 0; c < 3; ++c) osh[c] += gc[c];
      } else { /* EXT */
        double dr[3] = {P[0] - R->cc[0], P[1] - R->cc[1], P[2] - R->cc[2]};
        const double nr = sqrt(dr[0] * dr[0] + dr[1] * dr[1] + dr[2] * dr[2]);
        double dn[3] = {dr[0] / nr, dr[1] / nr, dr[2] / nr};
        double b[16], db[16][3];
        sh_basis(m->sh_degree, dn[0], dn[1], dn[2], b, db);
        const double* coef = m->sh + mi * K * 3;
        double gdn[3] = {0, 0, 0};
        for (int kk = 0; kk < K; ++kk) {
          double s = 0;
          for (int c = 0; c < 3; ++c) {
            osh[kk * 3 + c] += b[kk] * gc[c];
            s += coef[kk * 3 + c] * gc[c];
          }
          for (int a = 0; a < 3; ++a) gdn[a] += db[kk][a] * s;
        }
        const double dd = dn[0] * gdn[0] + dn[1] * gdn[1] + dn[2] * gdn[2];
        double gdir[3];
        for (int a = 0; a < 3; ++a) gdir[a] = (gdn[a] - dn[a] * dd) / nr;
        for (int a = 0; a < 3; ++a) gpos_world[a] += gdir[a];
        if (g_pose6) { /* dir = p - c, c' = c + omega x c + nu */
          const double* c = R->cc;
          pose[0] += gdir[1] * c[2] - gdir[2] * c[1];
          pose[1] += gdir[2] * c[0] - gdir[0] * c[2];
          pose[2] += gdir[0] * c[1] - gdir[1] * c[0];
          for (int a = 0; a < 3; ++a) pose[3 + a] -= gdir[a];
        }
      }
    }

    const double* gm = g_mu + (size_t)pj * 2;
    const double* gC = g_con + (size_t)pj * 4;
    if (!(gm[0] == 0.0 && gm[1] == 0.0 && gC[0] == 0.0 && gC[1] == 0.0 && gC[2] == 0.0 && gC[3] == 0.0 &&
          g_cz[pj] == 0.0)) { /* :299 */
      double t[3];
      for (int r = 0; r < 3; ++r) t[r] = rcw[r * 3 + 0] * P[0] + rcw[r * 3 + 1] * P[1] + rcw[r * 3 + 2] * P[2] + tcw[r];
      const double z = t[2];
      const double* qr = m->rot + mi * 4; /* x,y,z,w */
      const double qv[4] = {qr[3], qr[0], qr[1], qr[2]}; /* w,x,y,z */
      const double norm = sqrt(qv[0] * qv[0] + qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3]);
      const double qh[4] = {qv[0] / norm, qv[1] / norm, qv[2] / norm, qv[3] / norm};
      double rg[9];
      quat_to_rot(qh[0], qh[1], qh[2], qh[3], rg);
      double s2[3];
      for (int a = 0; a < 3; ++a) s2[a] = exp(2.0 * m->log_s[mi * 3 + a]);
      double rs[9], sigma3[9], tmp[9], sigmac[9];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) rs[r * 3 + c] = rg[r * 3 + c] * s2[c];
      mat3_mul_bt(rs, rg, sigma3);
      mat3_mul(rcw, sigma3, tmp);
      mat3_mul_bt(tmp, rcw, sigmac);
      const double j[6] = {k->fx / z, 0.0, -k->fx * t[0] / (z * z), 0.0, k->fy / z, -k->fy * t[1] / (z * z)};

      /* :315 g_sigma2 = -C gC C */
      const double* C = g->conic;
      double cg[4], gs2[4];
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) cg[r * 2 + c] = C[r * 2 + 0] * gC[0 * 2 + c] + C[r * 2 + 1] * gC[1 * 2 + c];
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) gs2[r * 2 + c] = -(cg[r * 2 + 0] * C[0 * 2 + c] + cg[r * 2 + 1] * C[1 * 2 + c]);
      /* :316 g_sigma_c = J^T gs2 J */
      double gsc[9];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
          double s = 0;
          for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) s += j[a * 3 + r] * gs2[a * 2 + b] * j[b * 3 + c];
          gsc[r * 3 + c] = s;
        }
      /* :317-318 g_J = (gs2 + gs2^T) J sigma_c */
      double sym2[4] = {gs2[0] + gs2[0], gs2[1] + gs2[2], gs2[2] + gs2[1], gs2[3] + gs2[3]};
      double jsc[6], gj[6];
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c)
          jsc[r * 3 + c] = j[r * 3 + 0] * sigmac[0 * 3 + c] + j[r * 3 + 1] * sigmac[1 * 3 + c] + j[r * 3 + 2] * sigmac[2 * 3 + c];
      for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 3; ++c) gj[r * 3 + c] = sym2[r * 2 + 0] * jsc[0 * 3 + c] + sym2[r * 2 + 1] * jsc[1 * 3 + c];
      /* :320-327 */
      double gt[3];
      for (int a = 0; a < 3; ++a) gt[a] = j[0 * 3 + a] * gm[0] + j[1 * 3 + a] * gm[1];
      const double z2 = z * z, z3 = z2 * z;
      gt[0] += gj[0 * 3 + 2] * (-k->fx / z2);
      gt[1] += gj[1 * 3 + 2] * (-k->fy / z2);
      gt[2] += gj[0 * 3 + 0] * (-k->fx / z2) + gj[0 * 3 + 2] * (2.0 * k->fx * t[0] / z3) +
               gj[1 * 3 + 1] * (-k->fy / z2) + gj[1 * 3 + 2] * (2.0 * k->fy * t[1] / z3);
      gt[2] += g_cz[pj];
      /* :329 */
      double gw[3];
      for (int a = 0; a < 3; ++a) gw[a] = rcw[0 * 3 + a] * gt[0] + rcw[1 * 3 + a] * gt[1] + rcw[2 * 3 + a] * gt[2];
      for (int a = 0; a < 3; ++a) gpos_world[a] += gw[a];
      /* :331-338 */
      double g3[9], tmp2[9];
      mat3_mul_at(rcw, gsc, tmp2);
      mat3_mul(tmp2, rcw, g3);
      double symm[9], grot[9], rts[9];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) symm[r * 3 + c] = g3[r * 3 + c] + g3[c * 3 + r];
      double rgs[9];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) rgs[r * 3 + c] = rg[r * 3 + c] * s2[c];
      mat3_mul(symm, rgs, grot);
      double rtg[9];
      mat3_mul_at(rg, g3, rtg);
      mat3_mul(rtg, rg, rts);
      for (int a = 0; a < 3; ++a) o_logs[mi * 3 + a] += rts[a * 3 + a] * 2.0 * s2[a];
      /* :340-345 with rotation_derivatives :28-40 */
      const double w = qh[0], x = qh[1], y = qh[2], zq = qh[3];
      const double dw[9] = {0, -zq, y, zq, 0, -x, -y, x, 0};
      const double dx[9] = {0, y, zq, y, -2 * x, -w, zq, w, -2 * x};
      const double dy[9] = {-2 * y, x, w, x, 0, zq, -w, zq, -2 * y};
      const double dz[9] = {-2 * zq, -w, x, w, -2 * zq, y, x, y, 0};
      double gq[4] = {0, 0, 0, 0};
      for (int e = 0; e < 9; ++e) {
        gq[0] += grot[e] * 2.0 * dw[e];
        gq[1] += grot[e] * 2.0 * dx[e];
        gq[2] += grot[e] * 2.0 * dy[e];
        gq[3] += grot[e] * 2.0 * dz[e];
      }
      /* :347-353 chain through normalization */
      const double dot = qh[0] * gq[0] + qh[1] * gq[1] + qh[2] * gq[2] + qh[3] * gq[3];
      for (int a = 0; a < 4; ++a) o_rot[mi * 4 + a] += (gq[a] - qh[a] * dot) / norm;

      if (g_pose6) { /* EXT pose: t' = R_cw (p - omega x p - nu) + t_cw, Sigma' = (I-W) S3 (I+W) */
        pose[0] += gw[1] * P[2] - gw[2] * P[1];
        pose[1] += gw[2] * P[0] - gw[0] * P[2];
        pose[2] += gw[0] * P[1] - gw[1] * P[0];
        for (int a = 0; a < 3; ++a) pose[3 + a] -= gw[a];
        double a1[9], a2[9];
        mat3_mul(sigma3, g3, a1);
        mat3_mul(g3, sigma3, a2);
        double A[9];
        for (int e = 0; e < 9; ++e) A[e] = a1[e] - a2[e];
        pose[0] += A[7] - A[5];
        pose[1] += A[2] - A[6];
        pose[2] += A[3] - A[1];
      }
    }
    for (int a = 0; a < 3; ++a) o_pos[mi * 3 + a] += gpos_world[a];
  }
  if (g_pose6) memcpy(g_pose6, pose, sizeof pose);
  free(g_mu); free(g_con); free(g_cz); free(g_col);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* EXT: geometry helpers for the pose finite-difference check                 */
/* geometry.cpp:8-13 (compose) and :22-41 (se3_exp)                           */
/* ------------------------------------------------------------------------ */
static void rot_to_quat(const double m[9], double q[4]) { /* Eigen Quaternion(Matrix3) */
  const double tr = m[0] + m[4] + m[8];
  if (tr > 0) {
    double t = sqrt(tr + 1.0);
    q[0] = 0.5 * t;
    t = 0.5 / t;
    q[1] = (m[7] - m[5]) * t; q[2] = (m[2] - m[6]) * t; q[3] = (m[3] - m[1]) * t;
  } else {
    int i = 0;
    if (m[4] > m[0]) i = 1;
    if (m[8] > m[i * 3 + i]) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    double t = sqrt(m[i * 3 + i] - m[j * 3 + j] - m[k * 3 + k] + 1.0);
    double v[3];
    v[i] = 0.5 * t;
    t = 0.5 / t;
    q[0] = (m[k * 3 + j] - m[j * 3 + k]) * t;
    v[j] = (m[j * 3 + i] + m[i * 3 + j]) * t;
    v[k] = (m[k * 3 + i] + m[i * 3 + k]) * t;
    q[1] = v[0]; q[2] = v[1]; q[3] = v[2];
  }
}

static void quat_mul(const double a[4], const double b[4], double c[4]) {
  c[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  c[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  c[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
  c[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
}

/* out = compose(se3_exp(xi), pose) */
ORC_API void orc_perturb_pose(const double xi[6], const double q_in[4], const double t_in[3], double q_out[4],
                              double t_out[3]) {
  const double* om = xi;
  const double* nu = xi + 3;
  const double th = sqrt(om[0] * om[0] + om[1] * om[1] + om[2] * om[2]);
  const double W[9] = {0, -om[2], om[1], om[2], 0, -om[0], -om[1], om[0], 0};
  double W2[9];
  mat3_mul(W, W, W2);
  double rot[9], V[9];
  double a, b, c;
  if (th < 1e-10) { a = 1.0; b = 0.5; c = 1.0 / 6.0; }
  else {
    const double t2 = th * th;
    a = sin(th) / th; b = (1.0 - cos(th)) / t2; c = (th - sin(th)) / (t2 * th);
  }
  for (int e = 0; e < 9; ++e) {
    const double I = (e % 4 == 0) ? 1.0 : 0.0;
    rot[e] = I + a * W[e] + b * W2[e];
    V[e] = I + b * W[e] + c * W2[e];
  }
  double qe[4];
  rot_to_quat(rot, qe);
  double n = sqrt(qe[0] * qe[0] + qe[1] * qe[1] + qe[2] * qe[2] + qe[3] * qe[3]);
  for (int i = 0; i < 4; ++i) qe[i] /= n;
  double te[3];
  for (int r = 0; r < 3; ++r) te[r] = V[r * 3 + 0] * nu[0] + V[r * 3 + 1] * nu[1] + V[r * 3 + 2] * nu[2];
  double qb[4] = {q_in[0], q_in[1], q_in[2], q_in[3]};
  n = sqrt(qb[0] * qb[0] + qb[1] * qb[1] + qb[2] * qb[2] + qb[3] * qb[3]);
  for (int i = 0; i < 4; ++i) qb[i] /= n;
  quat_mul(qe, qb, q_out);
  n = sqrt(q_out[0] * q_out[0] + q_out[1] * q_out[1] + q_out[2] * q_out[2] + q_out[3] * q_out[3]);
  for (int i = 0; i < 4; ++i) q_out[i] /= n;
  double re[9];
  quat_to_rot(qe[0], qe[1], qe[2], qe[3], re);
  for (int r = 0; r < 3; ++r)
    t_out[r] = re[r * 3 + 0] * t_in[0] + re[r * 3 + 1] * t_in[1] + re[r * 3 + 2] * t_in[2] + te[r];
}

/* ------------------------------------------------------------------------ */
/* EXT: all-cores CPU baseline.  The reference is single threaded; SPEC.md:   */
/* 298-299 permits per-pixel data parallelism.  Each thread runs the full     */
/* reference algorithm (project, global sort, composite, backward) on a       */
/* horizontal band of the image; per-thread gradients are summed.             */
/* ------------------------------------------------------------------------ */
typedef struct {
  const orc_map* m;
  const orc_camera* cam;
  const orc_config* cfg;
  int32_t win[4];
  double *rgb, *depth, *feat, *acc;
  const double *g_rgb, *g_depth, *g_feat;
  const double *t_rgb, *t_depth, *t_feat; /* EXT: L1 targets (cotangents computed per band) */
  double *o_pos, *o_rot, *o_logs, *o_opac, *o_sh, *o_feat, pose[6];
  double loss;
} band_job;

static void* band_worker(void* arg) {
  band_job* j = (band_job*)arg;
  orc_render* R = orc_render_forward(j->m, j->cam, j->cfg, NULL, j->win, j->rgb, j->depth, j->feat, j->acc);
  const double *g_rgb = j->g_rgb, *g_depth = j->g_depth, *g_feat = j->g_feat;
  double* cot = NULL;
  if (j->t_rgb) {
    /* EXT (SURVEY.md §8d loss): L = mean|rgb-T| + mean|depth-T| + mean|feat-T|, cotangent
     * sign(diff)/count, computed per pixel of this band from its own forward output. */
    const int W = j->cam->width, H = j->cam->height, d = j->m->d;
    const size_t npix = (size_t)W * H;
    cot = (double*)calloc(npix * (size_t)(4 + d), sizeof(double));
    double* cr = cot;
    double* cd = cot + npix * 3;
    double* cf = cot + npix * 4;
    const double nr = 3.0 * (double)npix, nd = (double)npix, nf = (double)d * (double)npix;
    double loss = 0.0;
    for (int y = j->win[1]; y < j->win[3]; ++y)
      for (int x = j->win[0]; x < j->win[2]; ++x) {
        const size_t p = (size_t)y * W + x;
        for (int c = 0; c < 3; ++c) {
          const double df = j->rgb[p * 3 + c] - j->t_rgb[p * 3 + c];
          cr[p * 3 + c] = df > 0 ? 1.0 / nr : (df < 0 ? -1.0 / nr : 0.0);
          loss += fabs(df) / nr;
        }
        const double dd = j->depth[p] - j->t_depth[p];
        cd[p] = dd > 0 ? 1.0 / nd : (dd < 0 ? -1.0 / nd : 0.0);
        loss += fabs(dd) / nd;
        for (int c = 0; c < d; ++c) {
          const double df = j->feat[p * d + c] - j->t_feat[p * d + c];
          cf[p * d + c] = df > 0 ? 1.0 / nf : (df < 0 ? -1.0 / nf : 0.0);
          loss += fabs(df) / nf;
        }
      }
    (void)H;
    j->loss = loss;
    g_rgb = cr; g_depth = cd; g_feat = d > 0 ? cf : NULL;
  }
  orc_render_backward(R, g_rgb, g_depth, g_feat, j->o_pos, j->o_rot, j->o_logs, j->o_opac, j->o_sh, j->o_feat,
                      j->pose);
  orc_render_free(R);
  free(cot);
  return NULL;
}

/* One fwd+bwd of rows [row_lo, row_hi) split into `threads` bands.  Images
 * are written for those rows; gradients are summed over bands. */
ORC_API int orc_fwd_bwd_bands(const orc_map* m, const orc_camera* cam, const orc_config* cfg, int32_t row_lo,
                              int32_t row_hi, int32_t threads, const double* g_rgb, const double* g_depth,
                              const double* g_feat, double* rgb, double* depth, double* feat, double* acc,
                              double* o_pos, double* o_rot, double* o_logs, double* o_opac, double* o_sh,
                              double* o_feat, double* pose6, const double* t_rgb, const double* t_depth,
                              const double* t_feat, double* loss) {
  if (threads < 1) threads = 1;
  const int W = cam->width, H = cam->height, d = m->d;
  const int K = sh_coeffs(m->sh_degree);
  const int64_t n = m->n;
  const size_t npix = (size_t)W * H;
  band_job* jobs = (band_job*)calloc((size_t)threads, sizeof(band_job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  const int rows = row_hi - row_lo;
  for (int t = 0; t < threads; ++t) {
    band_job* j = &jobs[t];
    j->m = m; j->cam = cam; j->cfg = cfg;
    j->win[0] = 0; j->win[2] = W;
    j->win[1] = row_lo + (int)((int64_t)rows * t / threads);
    j->win[3] = row_lo + (int)((int64_t)rows * (t + 1) / threads);
    j->rgb = (double*)malloc(sizeof(double) * npix * 3);
    j->depth = (double*)malloc(sizeof(double) * npix);
    j->feat = (double*)malloc(sizeof(double) * npix * (size_t)(d > 0 ? d : 1));
    j->acc = (double*)malloc(sizeof(double) * npix);
    j->g_rgb = g_rgb; j->g_depth = g_depth; j->g_feat = g_feat;
    j->t_rgb = t_rgb; j->t_depth = t_depth; j->t_feat = t_feat;
    j->o_pos = (double*)malloc(sizeof(double) * (size_t)n * 3);
    j->o_rot = (double*)malloc(sizeof(double) * (size_t)n * 4);
    j->o_logs = (double*)malloc(sizeof(double) * (size_t)n * 3);
    j->o_opac = (double*)malloc(sizeof(double) * (size_t)n);
    j->o_sh = (double*)malloc(sizeof(double) * (size_t)n * K * 3);
    j->o_feat = (double*)malloc(sizeof(double) * (size_t)n * (d > 0 ? d : 1));
    pthread_create(&th[t], NULL, band_worker, j);
  }
  memset(o_pos, 0, sizeof(double) * (size_t)n * 3);
  memset(o_rot, 0, sizeof(double) * (size_t)n * 4);
  memset(o_logs, 0, sizeof(double) * (size_t)n * 3);
  memset(o_opac, 0, sizeof(double) * (size_t)n);
  memset(o_sh, 0, sizeof(double) * (size_t)n * K * 3);
  if (d > 0) memset(o_feat, 0, sizeof(double) * (size_t)n * d);
  if (pose6) memset(pose6, 0, sizeof(double) * 6);
  if (loss) *loss = 0.0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    band_job* j = &jobs[t];
    const size_t p0 = (size_t)j->win[1] * W, p1 = (size_t)j->win[3] * W;
    memcpy(rgb + p0 * 3, j->rgb + p0 * 3, sizeof(double) * (p1 - p0) * 3);
    memcpy(depth + p0, j->depth + p0, sizeof(double) * (p1 - p0));
    if (d > 0) memcpy(feat + p0 * d, j->feat + p0 * d, sizeof(double) * (p1 - p0) * d);
    memcpy(acc + p0, j->acc + p0, sizeof(double) * (p1 - p0));
    for (int64_t i = 0; i < n * 3; ++i) { o_pos[i] += j->o_pos[i]; o_logs[i] += j->o_logs[i]; }
    for (int64_t i = 0; i < n * 4; ++i) o_rot[i] += j->o_rot[i];
    for (int64_t i = 0; i < n; ++i) o_opac[i] += j->o_opac[i];
    for (int64_t i = 0; i < n * K * 3; ++i) o_sh[i] += j->o_sh[i];
    for (int64_t i = 0; i < n * d; ++i) o_feat[i] += j->o_feat[i];
    if (pose6)
      for (int a = 0; a < 6; ++a) pose6[a] += j->pose[a];
    if (loss) *loss += j->loss;
    free(j->rgb); free(j->depth); free(j->feat); free(j->acc);
    free(j->o_pos); free(j->o_rot); free(j->o_logs); free(j->o_opac); free(j->o_sh); free(j->o_feat);
  }
  free(jobs);
  free(th);
  return 0;
}

/* ======================================================================== */
/* (B) fp32 twin of the product preprocess + binning.  Same op order as      */
/* paper_2511_16144_b200/csrc/preprocess.cu (lgs_project_f32); compile with  */
/* -ffp-contract=off so only the explicit fmaf()s fuse.                      */
/* ======================================================================== */

/* Deterministic expf: identical code in csrc/lgs_math.cuh (lgs_expf). */
static float orc_expf(float x) {
  if (x != x) return x;
  if (x > 88.72f) return INFINITY;
  if (x < -103.97f) return 0.0f;
  const float k = rintf(x * 1.44269504088896341f);
  float r = fmaf(k, -0.693145751953125f, x);
  r = fmaf(k, -1.428606765330187045e-06f, r);
  float p = 1.98412698412698413e-04f;
  p = fmaf(p, r, 1.38888888888888889e-03f);
  p = fmaf(p, r, 8.33333333333333333e-03f);
  p = fmaf(p, r, 4.16666666666666667e-02f);
  p = fmaf(p, r, 1.66666666666666667e-01f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  const int ki = (int)k;
  const int k1 = ki / 2, k2 = ki - k1;
  union { uint32_t u; float f; } s1, s2;
  s1.u = (uint32_t)(k1 + 127) << 23;
  s2.u = (uint32_t)(k2 + 127) << 23;
  return (p * s1.f) * s2.f;
}

ORC_API float orc_expf_export(float x) { return orc_expf(x); }

/* Deterministic logf for x >= 1: identical code in csrc/lgs_internal.cuh (lgs_logf). */
static float orc_logf(float x) {
  union { float f; uint32_t u; } b, mb;
  b.f = x;
  int e = (int)((b.u >> 23) & 0xffu) - 127;
  mb.u = (b.u & 0x7fffffu) | 0x3f800000u;
  float m = mb.f;
  if (m > 1.41421356f) {
    m = m * 0.5f;
    e = e + 1;
  }
  const float s = (m - 1.0f) / (m + 1.0f);
  const float s2 = s * s;
  float p = fmaf(s2, 0.0909090909f, 0.111111111f);
  p = fmaf(s2, p, 0.142857143f);
  p = fmaf(s2, p, 0.2f);
  p = fmaf(s2, p, 0.333333333f);
  p = fmaf(s2, p, 1.0f);
  return fmaf((float)e, 0.693147181f, (2.0f * s) * p);
}

ORC_API float orc_logf_export(float x) { return orc_logf(x); }

typedef struct {
  float rcw[9], tcw[3], cc[3];
  float fx, fy, cx, cy;
  int32_t width, height;
  float near_plane, dilation, radius_sigma, alpha_skip;
} orc32_cam;

/* Host camera setup: double math of camera_setup, then rounded to float. */
ORC_API void orc32_camera_setup(const orc_camera* cam, const orc_config* cfg, orc32_cam* out) {
  double rcw[9], tcw[3], cc[3];
  camera_setup(cam, rcw, tcw, cc);
  for (int i = 0; i < 9; ++i) out->rcw[i] = (float)rcw[i];
  for (int i = 0; i < 3; ++i) { out->tcw[i] = (float)tcw[i]; out->cc[i] = (float)cc[i]; }
  out->fx = (float)cam->fx; out->fy = (float)cam->fy;
  out->cx = (float)cam->cx; out->cy = (float)cam->cy;
  out->width = cam->width; out->height = cam->height;
  out->near_plane = (float)cfg->near_plane;
  out->dilation = (float)cfg->dilation;
  out->radius_sigma = (float)cfg->radius_sigma;
  out->alpha_skip = (float)cfg->alpha_skip;
}

static const float SHF_C1 = 0.4886025119029199f;
static const float SHF_C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                                -1.0925484305920792f, 0.5462742152960396f};
static const float SHF_C3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                                0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                                -0.5900435899266435f};

/* fp32 SH colour, same op order as csrc/lgs_math.cuh lgs_sh_color */
static void orc32_sh_color(int deg, const float* c, float x, float y, float z, float out[3]) {
  float b[16];
  b[0] = 1.0f;
  int K = 1;
  if (deg >= 1) {
    b[1] = -SHF_C1 * y; b[2] = SHF_C1 * z; b[3] = -SHF_C1 * x;
    K = 4;
  }
  if (deg >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    b[4] = SHF_C2[0] * (x * y);
    b[5] = SHF_C2[1] * (y * z);
    b[6] = SHF_C2[2] * ((zz + zz) - xx - yy);
    b[7] = SHF_C2[3] * (x * z);
    b[8] = SHF_C2[4] * (xx - yy);
    K = 9;
    if (deg >= 3) {
      b[9] = SHF_C3[0] * y * (3.0f * xx - yy);
      b[10] = SHF_C3[1] * (x * y) * z;
      b[11] = SHF_C3[2] * y * (4.0f * zz - xx - yy);
      b[12] = SHF_C3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
      b[13] = SHF_C3[4] * x * (4.0f * zz - xx - yy);
      b[14] = SHF_C3[5] * z * (xx - yy);
      b[15] = SHF_C3[6] * x * (xx - 3.0f * yy);
      K = 16;
    }
  }
  for (int ch = 0; ch < 3; ++ch) {
    float s = c[ch];
    for (int k = 1; k < K; ++k) s = fmaf(b[k], c[k * 3 + ch], s);
    out[ch] = s;
  }
}

/* One Gaussian, fp32.  Returns 1 if visible.  Mirrors lgs_project_f32. */
static int orc32_project(const float* P, const float* Q, const float* LS, float ol, const float* sh, int deg,
                         const orc32_cam* c, float* u_o, float* v_o, float* depth_o, float conic_o[3],
                         float* radius_o, int32_t bbox_o[4], float* opac_o, float color_o[3]) {
  const float* R = c->rcw;
  const float t0 = fmaf(R[0], P[0], fmaf(R[1], P[1], fmaf(R[2], P[2], c->tcw[0])));
  const float t1 = fmaf(R[3], P[0], fmaf(R[4], P[1], fmaf(R[5], P[2], c->tcw[1])));
  const float t2 = fmaf(R[6], P[0], fmaf(R[7], P[1], fmaf(R[8], P[2], c->tcw[2])));
  if (!(t2 > c->near_plane)) return 0;
  /* normalized quaternion; storage x,y,z,w */
  const float n2 = fmaf(Q[3], Q[3], fmaf(Q[0], Q[0], fmaf(Q[1], Q[1], Q[2] * Q[2])));
  const float nrm = sqrtf(n2);
  const float qw = Q[3] / nrm, qx = Q[0] / nrm, qy = Q[1] / nrm, qz = Q[2] / nrm;
  const float tx = 2.0f * qx, ty = 2.0f * qy, tz = 2.0f * qz;
  const float twx = tx * qw, twy = ty * qw, twz = tz * qw;
  const float txx = tx * qx, txy = ty * qx, txz = tz * qx;
  const float tyy = ty * qy, tyz = tz * qy, tzz = tz * qz;
  const float G[9] = {1.0f - (tyy + tzz), txy - twz, txz + twy, txy + twz, 1.0f - (txx + tzz),
                      tyz - twx, txz - twy, tyz + twx, 1.0f - (txx + tyy)};
  const float s[3] = {orc_expf(LS[0]), orc_expf(LS[1]), orc_expf(LS[2])};
  /* M = R_cw * R_g * diag(s) */
  float M[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      M[i * 3 + j] = fmaf(R[i * 3 + 0], G[0 * 3 + j], fmaf(R[i * 3 + 1], G[1 * 3 + j], R[i * 3 + 2] * G[2 * 3 + j])) * s[j];
  const float iz = 1.0f / t2;
  const float xz = t0 * iz, yz = t1 * iz;
  const float jx = c->fx * iz, jy = c->fy * iz;
  float T0[3], T1[3];
  for (int j = 0; j < 3; ++j) {
    T0[j] = jx * fmaf(-xz, M[6 + j], M[0 + j]);
    T1[j] = jy * fmaf(-yz, M[6 + j], M[3 + j]);
  }
  const float ca = fmaf(T0[0], T0[0], fmaf(T0[1], T0[1], T0[2] * T0[2])) + c->dilation;
  const float cb = fmaf(T0[0], T1[0], fmaf(T0[1], T1[1], T0[2] * T1[2]));
  const float cc = fmaf(T1[0], T1[0], fmaf(T1[1], T1[1], T1[2] * T1[2])) + c->dilation;
  const float det = fmaf(ca, cc, -(cb * cb));
  const float mid = 0.5f * (ca + cc);
  const float disc = fmaxf(fmaf(mid, mid, -det), 0.0f);
  const float lam = mid + sqrtf(disc);
  const float radius = c->radius_sigma * sqrtf(lam);
  const float u = fmaf(c->fx, xz, c->cx);
  const float v = fmaf(c->fy, yz, c->cy);
  const float Wf = (float)c->width, Hf = (float)c->height;
  if (!(u + radius >= -0.5f && u - radius <= Wf - 0.5f && v + radius >= -0.5f && v - radius <= Hf - 0.5f))
    return 0;
  if (!(det > 0.0f)) return 0;
  /* Pixel rect of renderer.cpp:131-134 intersected with the bounding box of the alpha >= skip
   * ellipse q <= 2 ln(o / skip) (plus margin): pixels outside never pass renderer.cpp:147. */
  const float opacity = 1.0f / (1.0f + orc_expf(-ol));
  if (c->alpha_skip > 0.0f && !(opacity >= c->alpha_skip)) return 0;
  float ex = 3.0e38f, ey = 3.0e38f;
  if (c->alpha_skip > 0.0f) {
    const float Q = 2.0f * orc_logf(opacity / c->alpha_skip);
    const float Qm = fmaf(Q, 1.001f, 0.01f);
    ex = sqrtf(Qm * ca) + 0.01f;
    ey = sqrtf(Qm * cc) + 0.01f;
  }
  bbox_o[0] = (int32_t)fmaxf(fmaxf(0.0f, floorf(u - radius)), floorf(u - ex));
  bbox_o[1] = (int32_t)fminf(fminf(Wf - 1.0f, ceilf(u + radius)), ceilf(u + ex));
  bbox_o[2] = (int32_t)fmaxf(fmaxf(0.0f, floorf(v - radius)), floorf(v - ey));
  bbox_o[3] = (int32_t)fminf(fminf(Hf - 1.0f, ceilf(v + radius)), ceilf(v + ey));
  if (bbox_o[0] > bbox_o[1] || bbox_o[2] > bbox_o[3]) return 0;
  conic_o[0] = cc / det;
  conic_o[1] = -cb / det;
  conic_o[2] = ca / det;
  *u_o = u; *v_o = v; *depth_o = t2; *radius_o = radius;
  *opac_o = opacity;
  if (deg == 0) {
    color_o[0] = sh[0]; color_o[1] = sh[1]; color_o[2] = sh[2];
  } else {
    float dx = P[0] - c->cc[0], dy = P[1] - c->cc[1], dz = P[2] - c->cc[2];
    const float dn = sqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)));
    const float idn = 1.0f / dn;
    dx *= idn; dy *= idn; dz *= idn;
    orc32_sh_color(deg, sh, dx, dy, dz, color_o);
  }
  return 1;
}

/* Map arrays are fp32 in the reference logical layouts (rot x,y,z,w; sh [N][K][3]). */
ORC_API int64_t orc32_preprocess(int64_t n, int32_t sh_degree, const float* pos, const float* rot,
                                 const float* log_s, const float* opac, const float* sh, const orc32_cam* c,
                                 uint8_t* visible, float* u, float* v, float* depth, float* conic,
                                 float* radius, int32_t* bbox, float* opacity, float* color,
                                 int32_t* tiles_touched) {
  const int K = sh_coeffs(sh_degree);
  int64_t nvis = 0;
  for (int64_t i = 0; i < n; ++i) {
    visible[i] = (uint8_t)orc32_project(pos + i * 3, rot + i * 4, log_s + i * 3, opac[i], sh + i * K * 3,
                                        sh_degree, c, &u[i], &v[i], &depth[i], conic + i * 3, &radius[i],
                                        bbox + i * 4, &opacity[i], color + i * 3);
    if (visible[i]) {
      const int32_t* b = bbox + i * 4;
      tiles_touched[i] = (b[1] / 16 - b[0] / 16 + 1) * (b[3] / 16 - b[2] / 16 + 1);
      ++nvis;
    } else {
      tiles_touched[i] = 0;
      u[i] = v[i] = depth[i] = radius[i] = opacity[i] = 0.0f;
      conic[i * 3 + 0] = conic[i * 3 + 1] = conic[i * 3 + 2] = 0.0f;
      color[i * 3 + 0] = color[i * 3 + 1] = color[i * 3 + 2] = 0.0f;
      bbox[i * 4 + 0] = bbox[i * 4 + 1] = bbox[i * 4 + 2] = bbox[i * 4 + 3] = 0;
    }
  }
  return nvis;
}

typedef struct {
  uint64_t key;
  uint32_t val;
} orc_pair;

static int cmp_pair(const void* a, const void* b) {
  const orc_pair* x = (const orc_pair*)a;
  const orc_pair* y = (const orc_pair*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return (x->val > y->val) - (x->val < y->val);
}

/* Key duplication + stable sort + per-tile ranges.  key = (tile << 32) |
 * f32bits(depth), tile = ty * tiles_x + tx, emitted in ascending map index so
 * a stable sort breaks depth ties by index (renderer.cpp:114-117).  Pass
 * keys == NULL to get the pair count only. */
ORC_API int64_t orc32_bin(int64_t n, const uint8_t* visible, const float* depth, const int32_t* bbox,
                          int32_t width, int32_t height, uint64_t* keys, uint32_t* vals, uint32_t* ranges) {
  const int tiles_x = (width + 15) / 16, tiles_y = (height + 15) / 16;
  int64_t P = 0;
  for (int64_t i = 0; i < n; ++i)
    if (visible[i]) {
      const int32_t* b = bbox + i * 4;
      P += (int64_t)(b[1] / 16 - b[0] / 16 + 1) * (b[3] / 16 - b[2] / 16 + 1);
    }
  if (!keys) return P;
  orc_pair* pr = (orc_pair*)malloc(sizeof(orc_pair) * (size_t)(P > 0 ? P : 1));
  int64_t o = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!visible[i]) continue;
    const int32_t* b = bbox + i * 4;
    union { float f; uint32_t u; } db;
    db.f = depth[i];
    for (int ty = b[2] / 16; ty <= b[3] / 16; ++ty)
      for (int tx = b[0] / 16; tx <= b[1] / 16; ++tx) {
        pr[o].key = ((uint64_t)(uint32_t)(ty * tiles_x + tx) << 32) | db.u;
        pr[o].val = (uint32_t)i;
        ++o;
      }
  }
  qsort(pr, (size_t)P, sizeof(orc_pair), cmp_pair);
  const int ntiles = tiles_x * tiles_y;
  for (int t = 0; t < ntiles; ++t) { ranges[t * 2] = 0; ranges[t * 2 + 1] = 0; }
  for (int64_t i = 0; i < P; ++i) {
    keys[i] = pr[i].key;
    vals[i] = pr[i].val;
    const uint32_t t = (uint32_t)(pr[i].key >> 32);
    if (i == 0 || (uint32_t)(pr[i - 1].key >> 32) != t) ranges[t * 2] = (uint32_t)i;
    if (i == P - 1 || (uint32_t)(pr[i + 1].key >> 32) != t) ranges[t * 2 + 1] = (uint32_t)(i + 1);
  }
  free(pr);
  return P;
}

/* ======================================================================== */
/* (C) Rng: std::mt19937_64 (the published Matsumoto-Nishimura 64-bit MT,    */
/* default seeding) + random.hpp:19-44 transforms.                           */
/* ======================================================================== */
typedef struct {
  uint64_t mt[312];
  int idx;
  double spare;
  int has_spare;
} orc_rng;

ORC_API orc_rng* orc_rng_new(uint64_t seed) {
  orc_rng* r = (orc_rng*)calloc(1, sizeof(orc_rng));
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
  return r;
}

ORC_API void orc_rng_free(orc_rng* r) { free(r); }

ORC_API uint64_t orc_rng_next_u64(orc_rng* r) {
  static const uint64_t MAG[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  if (r->idx >= 312) {
    int i;
    for (i = 0; i < 312 - 156; ++i) {
      const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[i + 1] & 0x7FFFFFFFULL);
      r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ MAG[x & 1];
    }
    for (; i < 311; ++i) {
      const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[i + 1] & 0x7FFFFFFFULL);
      r->mt[i] = r->mt[i + 156 - 312] ^ (x >> 1) ^ MAG[x & 1];
    }
    const uint64_t x = (r->mt[311] & 0xFFFFFFFF80000000ULL) | (r->mt[0] & 0x7FFFFFFFULL);
    r->mt[311] = r->mt[155] ^ (x >> 1) ^ MAG[x & 1];
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* random.hpp:19-21 */
ORC_API double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53; }

/* random.hpp:31-44 */
ORC_API double orc_rng_normal(orc_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double u1 = orc_rng_uniform(r);
  double u2 = orc_rng_uniform(r);
  while (u1 <= 0.0) u1 = orc_rng_uniform(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double th = 2.0 * M_PI * u2;
  r->spare = rr * sin(th);
  r->has_spare = 1;
  return rr * cos(th);
}
