/*
 * prune_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product): part (D) of the CPU
 * oracle, linked into liblgs_oracle.so with lgs_oracle.c.
 *
 * (D) Map pruning, SPEC.md:471-535 ([MODULE] pruning).  The reference's proj/src/pruning.cpp is a
 *     one-line placeholder, so this restates the SPEC's operations directly, as a plain sequential
 *     sweep (the definition), with the reference KD-tree's neighbour order
 *     (proj/include/legoslam/kdtree.hpp:36-55: k nearest by ascending (squared distance, index),
 *     the live filter applied inside the search).  oracle/ref_bridge.cpp runs the same sweep on
 *     the reference's own KdTree3 (tests/test_pruning_oracle.py checks the two agree).
 *
 *   find_language_redundant (Eq. 4): for i = 0 .. n-1 in ascending index, if G_i
 *     is live, take its K nearest live others; each G_j among them with |p_i - p_j|^2 < tau^2 and
 *     cos(f_i, f_j) > tau_sim is marked, and a marked Gaussian is dead at once.  Only neighbours
 *     inside tau can be marked and the K nearest are taken in distance order, so the sweep only
 *     needs the live Gaussians inside the tau-ball (found through a uniform grid of cells of edge
 *     tau: a pair closer than tau is at most one cell apart on every axis).
 *     Arithmetic (matched by csrc/prune.cu and ref_bridge.cpp; build with -ffp-contract=off):
 *       d2  = (dx*dx + dy*dy) + dz*dz in fp64 from the fp32 positions,
 *       cos = dot / (|f_i| |f_j|), dot and |f|^2 summed channel by channel from 0, |f| = sqrt;
 *       a zero-norm feature is similar to nothing; d = 0 or n < 2 marks nothing.
 *   find_geometric: sigmoid(logit) < alpha_min OR max_a exp(log_scale_a) >
 *     scale_max.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int64_t cx, cy, cz;
  int64_t idx;
} orc_cell;

static int cell_cmp(const void* a, const void* b) {
  const orc_cell *p = (const orc_cell*)a, *q = (const orc_cell*)b;
  if (p->cx != q->cx) return p->cx < q->cx ? -1 : 1;
  if (p->cy != q->cy) return p->cy < q->cy ? -1 : 1;
  if (p->cz != q->cz) return p->cz < q->cz ? -1 : 1;
  return p->idx < q->idx ? -1 : (p->idx > q->idx);
}

typedef struct {
  double d2;
  int64_t j;
} orc_nb;

static int nb_cmp(const void* a, const void* b) {
  const orc_nb *p = (const orc_nb*)a, *q = (const orc_nb*)b;
  if (p->d2 != q->d2) return p->d2 < q->d2 ? -1 : 1;
  return p->j < q->j ? -1 : (p->j > q->j);
}

static int64_t cell_coord(double x, double inv_h) {
  double c = floor(x * inv_h);
  const double lim = 1048576.0;
  if (c < -lim) c = -lim;
  if (c > lim - 1) c = lim - 1;
  return (int64_t)c;
}

/* first slot of `cells` (sorted) with cell >= (cx, cy, cz) */
static int64_t lower_cell(const orc_cell* cells, int64_t n, int64_t cx, int64_t cy, int64_t cz) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    const orc_cell* c = cells + mid;
    const int less = c->cx != cx ? c->cx < cx : (c->cy != cy ? c->cy < cy : c->cz < cz);
    if (less)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

static double dist2(const double* pos, int64_t i, int64_t j) {
  const double dx = pos[i * 3 + 0] - pos[j * 3 + 0];
  const double dy = pos[i * 3 + 1] - pos[j * 3 + 1];
  const double dz = pos[i * 3 + 2] - pos[j * 3 + 2];
  return (dx * dx + dy * dy) + dz * dz;
}

static int similar(const double* feat, int64_t n, int32_t d, const double* norm, int64_t i, int64_t j,
                   double tau_sim) {
  if (!(norm[i] > 0.0) || !(norm[j] > 0.0)) return 0;
  double dot = 0.0;
  for (int32_t c = 0; c < d; ++c) dot += feat[(int64_t)c * n + i] * feat[(int64_t)c * n + j];
  return dot / (norm[i] * norm[j]) > tau_sim;
}

/* flags[i] = 1 for the Gaussians the sweep marks; returns their count (-1: out of memory).
 * pos [n][3], feat [d][n] (fp64 copies of the map's fp32 values). */
int64_t orc_find_language_redundant(int64_t n, int32_t d, const double* pos, const double* feat, int32_t k,
                                    double tau_dist, double tau_sim, uint8_t* flags) {
  memset(flags, 0, (size_t)n);
  if (n < 2 || d <= 0 || k <= 0) return 0;
  const double inv_h = 1.0 / (tau_dist * (1.0 + 1e-6));
  const double tau2 = tau_dist * tau_dist;
  orc_cell* cells = (orc_cell*)malloc(sizeof(orc_cell) * (size_t)n);
  double* norm = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t cap = 64;
  orc_nb* nb = (orc_nb*)malloc(sizeof(orc_nb) * (size_t)cap);
  if (!cells || !norm || !nb) {
    free(cells);
    free(norm);
    free(nb);
    return -1;
  }
  for (int64_t i = 0; i < n; ++i) {
    cells[i].cx = cell_coord(pos[i * 3 + 0], inv_h);
    cells[i].cy = cell_coord(pos[i * 3 + 1], inv_h);
    cells[i].cz = cell_coord(pos[i * 3 + 2], inv_h);
    cells[i].idx = i;
    double s = 0.0;
    for (int32_t c = 0; c < d; ++c) s += feat[(int64_t)c * n + i] * feat[(int64_t)c * n + i];
    norm[i] = sqrt(s);
  }
  qsort(cells, (size_t)n, sizeof(orc_cell), cell_cmp);
  int64_t marked = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (flags[i]) continue;  /* dead: marks nothing */
    const int64_t cx = cell_coord(pos[i * 3 + 0], inv_h), cy = cell_coord(pos[i * 3 + 1], inv_h),
                  cz = cell_coord(pos[i * 3 + 2], inv_h);
    int64_t m = 0;
    for (int64_t ax = cx - 1; ax <= cx + 1; ++ax)
      for (int64_t ay = cy - 1; ay <= cy + 1; ++ay)
        for (int64_t az = cz - 1; az <= cz + 1; ++az) {
          for (int64_t s = lower_cell(cells, n, ax, ay, az);
               s < n && cells[s].cx == ax && cells[s].cy == ay && cells[s].cz == az; ++s) {
            const int64_t j = cells[s].idx;
            if (j == i || flags[j]) continue;
            const double d2 = dist2(pos, i, j);
            if (!(d2 < tau2)) continue;
            if (m == cap) {
              cap *= 2;
              orc_nb* g = (orc_nb*)realloc(nb, sizeof(orc_nb) * (size_t)cap);
              if (!g) {
                free(cells);
                free(norm);
                free(nb);
                return -1;
              }
              nb = g;
            }
            nb[m].d2 = d2;
            nb[m].j = j;
            ++m;
          }
        }
    qsort(nb, (size_t)m, sizeof(orc_nb), nb_cmp);
    for (int64_t q = 0; q < m && q < k; ++q)
      if (similar(feat, n, d, norm, i, nb[q].j, tau_sim)) {
        flags[nb[q].j] = 1;
        ++marked;
      }
  }
  free(cells);
  free(norm);
  free(nb);
  return marked;
}

/* opacity_logit [n], log_scale [n][3] */
int64_t orc_find_geometric(int64_t n, const double* opacity_logit, const double* log_scale, double alpha_min,
                           double scale_max, uint8_t* flags) {
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double op = 1.0 / (1.0 + exp(-opacity_logit[i]));
    const double smax = fmax(fmax(exp(log_scale[i * 3 + 0]), exp(log_scale[i * 3 + 1])), exp(log_scale[i * 3 + 2]));
    flags[i] = (op < alpha_min || smax > scale_max) ? 1 : 0;
    c += flags[i];
  }
  return c;
}
