// prune.cu -- map pruning on the resident map.
//
// Language rule (Eq. 4), sequential by definition: Gaussians in ascending index;
// a live G_i takes its K nearest LIVE others (the reference KD-tree's order, kdtree.hpp:36-55:
// ascending (squared distance, index), the live filter inside the search) and kills each G_j
// among them closer than tau_dist with cos(f_i, f_j) > tau_sim.  Only G_j within tau_dist can be
// killed, so only the K-nearest prefix inside that ball matters.
//
// The B200 version resolves the sweep in parallel rounds, exactly:
//   * a spatial hash (cells of edge tau_dist, 27-cell ball queries) replaces the KD-tree;
//   * "candidates": Gaussians with a similar neighbour inside tau_dist.  The others are never
//     killed and kill nothing (similarity is symmetric); they only occupy neighbour slots.
//   * the candidates' tau-balls are listed once (CSR: neighbour | similar bit, squared distance),
//     so the rounds read lists instead of repeating the hash queries and cosines;
//   * each round, phase 1 computes U(x) for every candidate x = the smallest UNRESOLVED
//     Gaussian that could kill x (a similar neighbour within tau_dist); phase 2 resolves candidate
//     i when (a) it was already killed by an earlier Gaussian (death[i] < i), or (b) U(i) >= i and
//     U(m) >= i for every candidate m in its ball -- no Gaussian before i that is still undecided
//     can change i's liveness or the liveness of anything i sees.  i then takes its K nearest
//     others alive at "time i" (death[m] > i: death[] holds the index of the killer) and kills the
//     similar ones (atomicMin(death[m], i)).
//   * the smallest unresolved candidate always resolves, so the rounds terminate; concurrent
//     resolutions in one round touch disjoint state (a kill of m by k in the round blocks every
//     i < k that sees m through U(m) <= k; every i > k reads death[m] = k > i as alive, which is
//     the sequential answer since k kills after i's turn).
// Distances / cosines in fp64 with explicit round-to-nearest ops (no contraction): the fp32 map
// values give the oracle's (and the reference build's) fp64 numbers bit for bit.
//
// Geometric rule and the compaction of prune (map rows + Adam moments, order
// kept) are one elementwise pass each.  Roofline: the ball queries are L2/latency bound (a few
// hundred bytes per Gaussian per query); all of this runs every `period` (200) mapping
// iterations, not per step.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <climits>

#include "dev_cache.h"
#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

namespace {

constexpr int kKMax = 32;
constexpr int kCoordBits = 21;
constexpr int64_t kCoordLim = (int64_t)1 << (kCoordBits - 1);

struct Grid {
  double inv_h;
  int tbits;
  const uint32_t* start;  // [T + 1]
  const uint64_t* key;    // [n] cell key of each slot
  const float4* pos;      // [n] x, y, z, map index bits
};

struct Feats {
  const float* f;  // [n][dp]
  int d, dp;
  const double* norm;  // [n]
};

__device__ __forceinline__ int cell_coord(float x, double inv_h) {
  double c = floor(__dmul_rn((double)x, inv_h));
  c = fmin(fmax(c, (double)-kCoordLim), (double)(kCoordLim - 1));
  return (int)c;
}
__device__ __forceinline__ uint64_t cell_key(int cx, int cy, int cz) {
  const uint64_t m = ((uint64_t)1 << kCoordBits) - 1;
  return ((uint64_t)(cx + kCoordLim) & m) | (((uint64_t)(cy + kCoordLim) & m) << kCoordBits) |
         (((uint64_t)(cz + kCoordLim) & m) << (2 * kCoordBits));
}
__device__ __forceinline__ uint32_t bucket_of(uint64_t key, int tbits) {
  return (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> (64 - tbits));
}

// |p - q|^2 in fp64, ((dx dx + dy dy) + dz dz)
__device__ __forceinline__ double dist2(float4 p, float4 q) {
  const double dx = __dsub_rn((double)p.x, (double)q.x), dy = __dsub_rn((double)p.y, (double)q.y),
               dz = __dsub_rn((double)p.z, (double)q.z);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

// cos(f_i, f_j) > tau_sim; a zero-norm feature is similar to nothing
__device__ __forceinline__ bool similar(const Feats& F, uint32_t i, uint32_t j, double tau_sim) {
  const double ni = F.norm[i], nj = F.norm[j];
  if (!(ni > 0.0) || !(nj > 0.0)) return false;
  const float* a = F.f + (size_t)i * F.dp;
  const float* b = F.f + (size_t)j * F.dp;
  double dot = 0.0;
  for (int c = 0; c < F.d; ++c) dot = __dadd_rn(dot, __dmul_rn((double)__ldg(a + c), (double)__ldg(b + c)));
  return __ddiv_rn(dot, __dmul_rn(ni, nj)) > tau_sim;
}

// f(slot) for every slot of the 27 cells around (cx, cy, cz); stops when f returns false
template <int R, class F>
__device__ __forceinline__ bool for_ball(const Grid& g, int cx, int cy, int cz, F&& f) {
  for (int dz = -R; dz <= R; ++dz)
    for (int dy = -R; dy <= R; ++dy)
      for (int dx = -R; dx <= R; ++dx) {
        const uint64_t key = cell_key(cx + dx, cy + dy, cz + dz);
        const uint32_t b = bucket_of(key, g.tbits);
        const uint32_t e = g.start[b + 1];
        for (uint32_t s = g.start[b]; s < e; ++s)
          if (g.key[s] == key && !f(s)) return false;
      }
  return true;
}

// ---------------------------------------------------------------------------------------------
// spatial hash: counting sort of the Gaussians by bucket of their cell
__global__ void hash_count_kernel(const float4* __restrict__ po, int64_t n, double inv_h, int tbits,
                                  uint64_t* __restrict__ key_of, uint32_t* __restrict__ count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 p = po[i];
  const uint64_t k = cell_key(cell_coord(p.x, inv_h), cell_coord(p.y, inv_h), cell_coord(p.z, inv_h));
  key_of[i] = k;
  atomicAdd(count + bucket_of(k, tbits), 1u);
}

// slots inside a bucket in any order (every query visits the whole bucket)
__global__ void hash_scatter_kernel(const float4* __restrict__ po, int64_t n, int tbits,
                                    const uint64_t* __restrict__ key_of, const uint32_t* __restrict__ start,
                                    uint32_t* __restrict__ cursor, uint64_t* __restrict__ skey,
                                    float4* __restrict__ spos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = key_of[i];
  const uint32_t b = bucket_of(k, tbits);
  const uint32_t s = start[b] + atomicAdd(cursor + b, 1u);
  const float4 p = po[i];
  skey[s] = k;
  spos[s] = make_float4(p.x, p.y, p.z, __uint_as_float((uint32_t)i));
}

__global__ void feat_norm_kernel(const float* __restrict__ f, int64_t n, int d, int dp, double* __restrict__ norm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* a = f + (size_t)i * dp;
  double s = 0.0;
  for (int c = 0; c < d; ++c) {
    const double v = (double)a[c];
    s = __dadd_rn(s, __dmul_rn(v, v));
  }
  norm[i] = __dsqrt_rn(s);
}

// candidates: a similar neighbour inside tau_dist; listed (any order) for the rounds
__global__ void candidates_kernel(Grid g, Feats F, int64_t n, double tau2, double tau_sim,
                                  uint8_t* __restrict__ cand, uint32_t* __restrict__ list1,
                                  uint32_t* __restrict__ list2, uint32_t* __restrict__ counts) {
  const int64_t s0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s0 >= n) return;
  const float4 p = g.pos[s0];
  const uint32_t i = __float_as_uint(p.w);
  const int cx = cell_coord(p.x, g.inv_h), cy = cell_coord(p.y, g.inv_h), cz = cell_coord(p.z, g.inv_h);
  bool found = false;
  for_ball<1>(g, cx, cy, cz, [&](uint32_t s) {
    const float4 q = g.pos[s];
    const uint32_t j = __float_as_uint(q.w);
    if (j != i && dist2(p, q) < tau2 && similar(F, i, j, tau_sim)) found = true;
    return !found;
  });
  cand[i] = found ? 1 : 0;
  if (found) {
    const uint32_t k = atomicAdd(counts, 1u);
    list1[k] = i;
    list2[k] = i;
  }
}

// Neighbour lists of the candidates (CSR over their list positions): every other Gaussian inside
// tau_dist, as (index | similar << 31) and its squared distance.  Built once: the rounds then read
// them instead of repeating the ball queries and the cosines every round.
__global__ void nb_count_kernel(Grid g, const uint32_t* __restrict__ list, const uint32_t* __restrict__ ncand,
                                const float4* __restrict__ po, double tau2, uint32_t* __restrict__ cnt) {
  const uint32_t nc = *ncand;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nc; k += gridDim.x * blockDim.x) {
    const uint32_t i = list[k];
    const float4 p = po[i];
    const int cx = cell_coord(p.x, g.inv_h), cy = cell_coord(p.y, g.inv_h), cz = cell_coord(p.z, g.inv_h);
    uint32_t c = 0;
    for_ball<1>(g, cx, cy, cz, [&](uint32_t s) {
      const float4 q = g.pos[s];
      if (__float_as_uint(q.w) != i && dist2(p, q) < tau2) ++c;
      return true;
    });
    cnt[k] = c;
  }
}

__global__ void nb_fill_kernel(Grid g, Feats F, const uint32_t* __restrict__ list, const uint32_t* __restrict__ ncand,
                               const float4* __restrict__ po, double tau2, double tau_sim,
                               const uint32_t* __restrict__ off, uint32_t* __restrict__ nb, double* __restrict__ nbd2,
                               uint32_t* __restrict__ pos_of) {
  const uint32_t nc = *ncand;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nc; k += gridDim.x * blockDim.x) {
    const uint32_t i = list[k];
    pos_of[i] = k;
    const float4 p = po[i];
    const int cx = cell_coord(p.x, g.inv_h), cy = cell_coord(p.y, g.inv_h), cz = cell_coord(p.z, g.inv_h);
    uint32_t w = off[k];
    for_ball<1>(g, cx, cy, cz, [&](uint32_t s) {
      const float4 q = g.pos[s];
      const uint32_t j = __float_as_uint(q.w);
      if (j == i) return true;
      const double d2 = dist2(p, q);
      if (!(d2 < tau2)) return true;
      nb[w] = j | (similar(F, i, j, tau_sim) ? 0x80000000u : 0u);
      nbd2[w] = d2;
      ++w;
      return true;
    });
  }
}

struct Rounds {
  int K;
  const uint8_t* cand;
  uint8_t* res;      // resolved
  uint32_t* death;   // index of the killer (UINT_MAX: alive)
  uint32_t* U;       // smallest unresolved potential killer (UINT_MAX: none)
  uint32_t* counts;  // [parity * 2 + {0: list1, 1: list2}]
  uint32_t* list1[2];
  uint32_t* list2[2];
  uint32_t* rounds;  // rounds that found work
  const uint32_t* pos_of;  // map index -> candidate list position (CSR row)
  const uint32_t* off;     // CSR offsets
  const uint32_t* nb;      // neighbour | similar << 31
  const double* nbd2;      // squared distance
};

// phase 1: U(x) for the listed candidates; a candidate whose potential killers are all resolved
// stays settled (U = UINT_MAX) and leaves the list
__global__ void round_u_kernel(Rounds r, int par) {
  const uint32_t cnt = r.counts[par * 2 + 0];
  const uint32_t* in = r.list1[par];
  uint32_t* out = r.list1[par ^ 1];
  uint32_t* out_cnt = r.counts + (par ^ 1) * 2 + 0;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
    const uint32_t x = in[t];
    const uint32_t k = r.pos_of[x];
    uint32_t u = UINT_MAX;
    for (uint32_t e = r.off[k], e1 = r.off[k + 1]; e < e1; ++e) {
      const uint32_t v = r.nb[e];
      const uint32_t j = v & 0x7fffffffu;
      if ((v >> 31) && j < u && !r.res[j]) u = j;
    }
    r.U[x] = u;
    if (u != UINT_MAX) out[atomicAdd(out_cnt, 1u)] = x;
  }
}

// phase 2: resolve the candidates nothing undecided can still influence
__global__ void round_resolve_kernel(Rounds r, int par) {
  const uint32_t cnt = r.counts[par * 2 + 1];
  if (blockIdx.x == 0 && threadIdx.x == 0 && cnt) atomicAdd(r.rounds, 1u);
  const uint32_t* in = r.list2[par];
  uint32_t* out = r.list2[par ^ 1];
  uint32_t* out_cnt = r.counts + (par ^ 1) * 2 + 1;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
    const uint32_t i = in[t];
    if (r.death[i] < i) {  // killed by an earlier Gaussian: dead at its turn, kills nothing
      r.res[i] = 1;
      continue;
    }
    bool blocked = r.U[i] < i;
    const uint32_t k0 = r.pos_of[i];
    const uint32_t e0 = r.off[k0], e1 = r.off[k0 + 1];
    for (uint32_t e = e0; e < e1 && !blocked; ++e) {
      const uint32_t m = r.nb[e] & 0x7fffffffu;
      blocked = r.cand[m] && r.U[m] < i;
    }
    if (blocked) {
      out[atomicAdd(out_cnt, 1u)] = i;
      continue;
    }
    // the K nearest others alive at time i, ascending (d2, index)
    double bd[kKMax] = {};
    uint32_t bi[kKMax] = {};  // neighbour | similar << 31
    int nbk = 0;
    for (uint32_t e = e0; e < e1; ++e) {
      const uint32_t v = r.nb[e];
      const uint32_t m = v & 0x7fffffffu;
      if (r.death[m] <= i) continue;  // dead before i's turn
      const double d2 = r.nbd2[e];
      if (nbk == r.K && !(d2 < bd[nbk - 1] || (d2 == bd[nbk - 1] && m < (bi[nbk - 1] & 0x7fffffffu)))) continue;
      int q = nbk < r.K ? nbk++ : nbk - 1;
      while (q > 0 && (d2 < bd[q - 1] || (d2 == bd[q - 1] && m < (bi[q - 1] & 0x7fffffffu)))) {
        bd[q] = bd[q - 1];
        bi[q] = bi[q - 1];
        --q;
      }
      bd[q] = d2;
      bi[q] = v;
    }
    for (int q = 0; q < nbk; ++q)
      if (bi[q] >> 31) atomicMin(r.death + (bi[q] & 0x7fffffffu), i);
    r.res[i] = 1;
  }
}

__global__ void death_flags_kernel(const uint32_t* __restrict__ death, int64_t n, uint8_t* __restrict__ flags,
                                   unsigned long long* __restrict__ total) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool f = false;
  if (i < n) {
    f = death[i] != UINT_MAX;
    flags[i] = f ? 1 : 0;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(total, (unsigned long long)__popc(bal));
}

__global__ void geometric_kernel(const float4* __restrict__ po, const float4* __restrict__ sc, int64_t n,
                                 double alpha_min, double scale_max, uint8_t* __restrict__ flags,
                                 unsigned long long* __restrict__ total) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool f = false;
  if (i < n) {
    const double op = 1.0 / (1.0 + exp(-(double)po[i].w));
    const float4 s = sc[i];
    const double smax = fmax(fmax(exp((double)s.x), exp((double)s.y)), exp((double)s.z));
    f = op < alpha_min || smax > scale_max;
    flags[i] = f ? 1 : 0;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(total, (unsigned long long)__popc(bal));
}

}  // namespace

// ---------------------------------------------------------------------------------------------
static int table_bits(int64_t n) {
  int b = 8;
  while (b < 31 && ((int64_t)1 << b) < 2 * n) ++b;
  return b;
}

size_t prune_scratch_bytes(int64_t n) {
  const size_t T = (size_t)1 << table_bits(n);
  size_t scan = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)(T + 1));
  size_t scan2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan2, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)std::max<int64_t>(n, 1));
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t nn = (size_t)std::max<int64_t>(n, 1);
  return al(8 * nn) * 2 + al(16 * nn) + al(4 * (T + 1)) * 2 + al(8 * nn) + al(nn) * 2 + al(4 * nn) * 6 + al(64) +
         al(std::max(scan, scan2));
}

namespace {
struct Carve {
  uint64_t *key_of, *skey;
  float4* spos;
  uint32_t *count, *start;
  double* norm;
  uint8_t *cand, *res;
  uint32_t *death, *U, *l1[2], *l2[2];
  uint32_t* small;  // [0..3] list counts by parity, [4] rounds, [8..9] u64 total
  void* scan_tmp;
  size_t scan_bytes;
};

Carve carve(void* base, int64_t n, int tbits) {
  const size_t T = (size_t)1 << tbits;
  const size_t nn = (size_t)std::max<int64_t>(n, 1);
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  uint8_t* p = static_cast<uint8_t*>(base);
  Carve c{};
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += al(bytes);
    return r;
  };
  c.key_of = reinterpret_cast<uint64_t*>(take(8 * nn));
  c.skey = reinterpret_cast<uint64_t*>(take(8 * nn));
  c.spos = reinterpret_cast<float4*>(take(16 * nn));
  c.count = reinterpret_cast<uint32_t*>(take(4 * (T + 1)));
  c.start = reinterpret_cast<uint32_t*>(take(4 * (T + 1)));
  c.norm = reinterpret_cast<double*>(take(8 * nn));
  c.cand = take(nn);
  c.res = take(nn);
  c.death = reinterpret_cast<uint32_t*>(take(4 * nn));
  c.U = reinterpret_cast<uint32_t*>(take(4 * nn));
  c.l1[0] = reinterpret_cast<uint32_t*>(take(4 * nn));
  c.l1[1] = reinterpret_cast<uint32_t*>(take(4 * nn));
  c.l2[0] = reinterpret_cast<uint32_t*>(take(4 * nn));
  c.l2[1] = reinterpret_cast<uint32_t*>(take(4 * nn));
  c.small = reinterpret_cast<uint32_t*>(take(64));
  c.scan_tmp = p;
  cub::DeviceScan::ExclusiveSum(nullptr, c.scan_bytes, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)(T + 1));
  return c;
}
}  // namespace

cudaError_t run_language_redundant(const PruneIn& in, const PruneParams& pp, uint8_t* flags, void* scratch,
                                   int64_t* count, int64_t* candidates, int64_t* rounds, cudaStream_t s) {
  const int64_t n = in.n;
  if (count) *count = 0;
  if (candidates) *candidates = 0;
  if (rounds) *rounds = 0;
  if (n == 0) return cudaSuccess;
  if (n < 2 || in.d == 0) return cudaMemsetAsync(flags, 0, (size_t)n, s);
  const int tbits = table_bits(n);
  const size_t T = (size_t)1 << tbits;
  Carve c = carve(scratch, n, tbits);
  const double h = pp.tau_dist * (1.0 + 1e-6);  // a pair closer than tau_dist is never two cells apart
  const double inv_h = 1.0 / h;
  const unsigned nb = (unsigned)((n + 255) / 256);
  cudaMemsetAsync(c.count, 0, 4 * (T + 1), s);
  hash_count_kernel<<<nb, 256, 0, s>>>(in.pos_opa, n, inv_h, tbits, c.key_of, c.count);
  size_t sb = c.scan_bytes;
  cub::DeviceScan::ExclusiveSum(c.scan_tmp, sb, c.count, c.start, (int)(T + 1), s);
  cudaMemsetAsync(c.count, 0, 4 * T, s);
  hash_scatter_kernel<<<nb, 256, 0, s>>>(in.pos_opa, n, tbits, c.key_of, c.start, c.count, c.skey, c.spos);
  feat_norm_kernel<<<nb, 256, 0, s>>>(in.feat, n, in.d, in.dp, c.norm);
  cudaMemsetAsync(c.small, 0, 64, s);
  cudaMemsetAsync(c.res, 0, (size_t)n, s);
  cudaMemsetAsync(c.death, 0xff, 4 * (size_t)n, s);
  Grid g{inv_h, tbits, c.start, c.skey, c.spos};
  Feats F{in.feat, in.d, in.dp, c.norm};
  const double tau2 = pp.tau_dist * pp.tau_dist;
  candidates_kernel<<<nb, 256, 0, s>>>(g, F, n, tau2, pp.tau_sim, c.cand, c.l1[0], c.l2[0], c.small);
  // list 2 starts with the same count as list 1
  cudaMemcpyAsync(c.small + 1, c.small, 4, cudaMemcpyDeviceToDevice, s);
  uint32_t host_cand = 0;
  cudaMemcpyAsync(&host_cand, c.small, 4, cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  if (candidates) *candidates = host_cand;
  // the candidates' neighbour lists (CSR), built once for all rounds
  uint32_t *cnt = nullptr, *off = nullptr, *pos_of = nullptr, *nbl = nullptr;
  double* nbd2 = nullptr;
  auto release = [&]() {
    if (cnt) cudaFreeAsync(cnt, s);
    if (off) cudaFreeAsync(off, s);
    if (pos_of) cudaFreeAsync(pos_of, s);
    if (nbl) cudaFreeAsync(nbl, s);
    if (nbd2) cudaFreeAsync(nbd2, s);
  };
  if (host_cand) {
    const unsigned grid = (unsigned)std::min<int64_t>((host_cand + 255) / 256, (int64_t)device_sm_count() * 8);
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&cnt), sizeof(uint32_t) * (host_cand + 1), s)) != cudaSuccess ||
        (e = cudaMallocAsync(reinterpret_cast<void**>(&off), sizeof(uint32_t) * (host_cand + 1), s)) != cudaSuccess ||
        (e = cudaMallocAsync(reinterpret_cast<void**>(&pos_of), sizeof(uint32_t) * (size_t)n, s)) != cudaSuccess) {
      release();
      return e;
    }
    cudaMemsetAsync(cnt + host_cand, 0, sizeof(uint32_t), s);
    nb_count_kernel<<<grid, 256, 0, s>>>(g, c.l1[0], c.small, in.pos_opa, tau2, cnt);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int)host_cand + 1);
    void* tmp = nullptr;
    if ((e = cudaMallocAsync(&tmp, tb, s)) != cudaSuccess) {
      release();
      return e;
    }
    cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, (int)host_cand + 1, s);
    cudaFreeAsync(tmp, s);
    uint32_t entries = 0;
    cudaMemcpyAsync(&entries, off + host_cand, 4, cudaMemcpyDeviceToHost, s);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) {
      release();
      return e;
    }
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&nbl), sizeof(uint32_t) * std::max<uint32_t>(entries, 1), s)) !=
            cudaSuccess ||
        (e = cudaMallocAsync(reinterpret_cast<void**>(&nbd2), sizeof(double) * std::max<uint32_t>(entries, 1), s)) !=
            cudaSuccess) {
      release();
      return e;
    }
    nb_fill_kernel<<<grid, 256, 0, s>>>(g, F, c.l1[0], c.small, in.pos_opa, tau2, pp.tau_sim, off, nbl, nbd2, pos_of);
  }
  Rounds r{pp.k, c.cand, c.res, c.death, c.U, c.small, {c.l1[0], c.l1[1]}, {c.l2[0], c.l2[1]}, c.small + 4,
           pos_of, off, nbl, nbd2};
  if (host_cand) {
    const unsigned grid = (unsigned)std::min<int64_t>((host_cand + 255) / 256, (int64_t)device_sm_count() * 8);
    int par = 0;
    uint32_t left = host_cand;
    constexpr int kBatch = 8;  // rounds between host checks (an idle round costs two empty launches)
    int64_t issued = 0;
    while (left) {
      // every round resolves at least the smallest unresolved candidate: more rounds than
      // candidates would be a bug, not a slow map -- fail instead of spinning
      if (issued > (int64_t)host_cand + kBatch) {
        release();
        return cudaErrorUnknown;
      }
      issued += kBatch;
      for (int b = 0; b < kBatch; ++b) {
        cudaMemsetAsync(c.small + (par ^ 1) * 2, 0, 8, s);
        round_u_kernel<<<grid, 256, 0, s>>>(r, par);
        round_resolve_kernel<<<grid, 256, 0, s>>>(r, par);
        par ^= 1;
      }
      cudaMemcpyAsync(&left, c.small + par * 2 + 1, 4, cudaMemcpyDeviceToHost, s);
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) {
        release();
        return e;
      }
    }
  }
  release();
  unsigned long long* total = reinterpret_cast<unsigned long long*>(c.small + 8);
  death_flags_kernel<<<nb, 256, 0, s>>>(c.death, n, flags, total);
  unsigned long long host_total = 0;
  uint32_t host_rounds = 0;
  cudaMemcpyAsync(&host_total, total, 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&host_rounds, c.small + 4, 4, cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  if (count) *count = (int64_t)host_total;
  if (rounds) *rounds = host_rounds;
  return cudaGetLastError();
}

cudaError_t run_geometric(const PruneIn& in, const PruneParams& pp, uint8_t* flags, void* scratch, int64_t* count,
                          cudaStream_t s) {
  if (count) *count = 0;
  if (in.n == 0) return cudaSuccess;
  unsigned long long* total = static_cast<unsigned long long*>(scratch);
  cudaMemsetAsync(total, 0, 8, s);
  geometric_kernel<<<(unsigned)((in.n + 255) / 256), 256, 0, s>>>(in.pos_opa, in.scale, in.n, pp.alpha_min,
                                                                   pp.scale_max, flags, total);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, total, 8, cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  if (count) *count = (int64_t)h;
  return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// compaction: new index of every surviving row (exclusive scan of keep), then row copies
namespace {
__global__ void keep_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t n,
                            uint32_t* __restrict__ keep) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keep[i] = (a && a[i]) || (b && b[i]) ? 0u : 1u;
}

__global__ void compact_rows_kernel(RowCopies rc, const uint32_t* __restrict__ keep,
                                    const uint32_t* __restrict__ dst_of, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !keep[i]) return;
  const uint32_t o = dst_of[i];
  for (int a = 0; a < rc.count; ++a) {
    const int w = rc.width[a];
    const float* src = rc.src[a] + (size_t)i * w;
    float* dst = rc.dst[a] + (size_t)o * w;
    if ((w & 3) == 0) {
      for (int k = 0; k < w; k += 4)
        *reinterpret_cast<float4*>(dst + k) = *reinterpret_cast<const float4*>(src + k);
    } else {
      for (int k = 0; k < w; ++k) dst[k] = src[k];
    }
  }
}
}  // namespace

size_t compact_scratch_bytes(int64_t n) {
  size_t scan = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)std::max<int64_t>(n, 1));
  const size_t nn = (size_t)std::max<int64_t>(n, 1);
  return ((8 * nn + 255) & ~(size_t)255) + scan + 256;
}

cudaError_t run_compact(const uint8_t* drop_a, const uint8_t* drop_b, int64_t n, void* scratch, int64_t* kept,
                        uint32_t** keep_out, uint32_t** dst_out, cudaStream_t s) {
  const size_t nn = (size_t)std::max<int64_t>(n, 1);
  uint32_t* keep = static_cast<uint32_t*>(scratch);
  uint32_t* dst = keep + nn;
  void* tmp = reinterpret_cast<uint8_t*>(scratch) + ((8 * nn + 255) & ~(size_t)255);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, keep, dst, (int)nn);
  keep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(drop_a, drop_b, n, keep);
  cub::DeviceScan::ExclusiveSum(tmp, tb, keep, dst, (int)n, s);
  uint32_t last[2] = {0, 0};
  cudaMemcpyAsync(&last[0], dst + n - 1, 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&last[1], keep + n - 1, 4, cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  *kept = (int64_t)last[0] + last[1];
  *keep_out = keep;
  *dst_out = dst;
  return cudaGetLastError();
}

void launch_compact_rows(const RowCopies& rc, const uint32_t* keep, const uint32_t* dst_of, int64_t n,
                         cudaStream_t s) {
  if (n == 0 || rc.count == 0) return;
  compact_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(rc, keep, dst_of, n);
}

}  // namespace lgs
