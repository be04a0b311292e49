"""Seeded synthetic scenes for the BASELINE.json configs (numpy PCG64, fp32-rounded).

No public dataset ships with the reference or this container: the paper's
Replica / TUM-RGBD / ScanNet scenes are replaced by seeded
synthetic Gaussian maps with the shapes and value distributions BASELINE.json
states.  Every value is drawn in float64 then rounded to float32 (the
"draw through float" trick of proj/tests/test_map.cpp:17-18), so the fp64 CPU
oracle and the fp32 GPU path see bit-identical inputs.

Layouts are the reference's (proj/include/legoslam/gaussian_map.hpp:57-93):
pos [N,3], rot [N,4] in Eigen storage order (x,y,z,w), log_s [N,3],
opac [N] (logits), sh [N,K,3] (K=1 is the reference ``colors``), feat [d,N]
(the column-major N x d Eigen matrix).

Choices BASELINE.json leaves open are pinned here and
recorded in DESIGN.md: config-1 pose = identity; config-2 camera on the room
wall looking along +z; config-3 circle plane; config-4 arc and the remaining
30% of Gaussians; L1 target ranges; seeds = 1000 + config id.
"""
from __future__ import annotations

import math

import numpy as np

CONFIG_NAMES = ("c0", "c1", "c1_500k", "c2", "c3", "c4")


class RefRng:
    """The reference's lego::Rng (proj/include/legoslam/random.hpp:12-50) as a numpy generator with
    the subset of the numpy Generator API the configs use, so a scene can be drawn from the
    reference's own stream (``make_config(..., rng="reference")``): std::mt19937_64 (vectorized
    twist, standard seeding and tempering), uniform() = (u64 >> 11) * 2^-53, uniform(lo, hi) =
    lo + (hi - lo) uniform(), uniform_int(n) = int(uniform() n), normal() = Box-Muller with the
    cached second value.  Draw order: every call consumes the stream in C order of its output;
    normal(mu, sigma) = mu + sigma * normal() (the reference has only the standard normal).
    Bit-identical to the C restatement in oracle/lgs_oracle.c (tests/test_scenes_rng.py), which is
    pinned to the C++ standard's known mt19937_64 value."""

    _N, _M = 312, 156
    _MAG = np.uint64(0xB5026F5AA96619E9)
    _UP, _LO = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [int(seed) & 0xFFFFFFFFFFFFFFFF]
        for i in range(1, self._N):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
        self._mt = np.array(mt, dtype=np.uint64)
        self._buf = np.zeros(0, np.uint64)
        self._spare = None

    def _twist(self):
        mt, N, M = self._mt, self._N, self._M
        one = np.uint64(1)
        x = (mt[:N - M] & self._UP) | (mt[1:N - M + 1] & self._LO)
        mt[:N - M] = mt[M:] ^ (x >> one) ^ np.where((x & one) != 0, self._MAG, np.uint64(0))
        x = (mt[N - M:N - 1] & self._UP) | (mt[N - M + 1:N] & self._LO)
        mt[N - M:N - 1] = mt[:M - 1] ^ (x >> one) ^ np.where((x & one) != 0, self._MAG, np.uint64(0))
        x = (mt[N - 1] & self._UP) | (mt[0] & self._LO)
        mt[N - 1] = mt[M - 1] ^ (x >> one) ^ (self._MAG if int(x) & 1 else np.uint64(0))
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        return y

    def next_u64(self, k: int) -> np.ndarray:
        out = [self._buf]
        have = self._buf.size
        while have < k:
            blk = self._twist()
            out.append(blk)
            have += blk.size
        allv = np.concatenate(out) if len(out) > 1 else out[0]
        self._buf = allv[k:]
        return allv[:k]

    def _unit(self, k: int) -> np.ndarray:  # random.hpp:20-22
        return (self.next_u64(k) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def uniform(self, lo=0.0, hi=1.0, size=None):
        shape = () if size is None else size
        k = int(np.prod(shape))
        v = lo + (hi - lo) * self._unit(k)
        return v.reshape(shape) if size is not None else float(v[0])

    def integers(self, lo, hi, size=None):  # uniform_int(hi - lo) + lo, random.hpp:27-29
        shape = () if size is None else size
        k = int(np.prod(shape))
        v = (self._unit(k) * float(hi - lo)).astype(np.int64) + lo
        return v.reshape(shape)

    def _normal(self, k: int) -> np.ndarray:  # random.hpp:31-44, the spare kept across calls
        out = np.empty(k, np.float64)
        i = 0
        if k and self._spare is not None:
            out[0] = self._spare
            self._spare = None
            i = 1
        need = k - i
        pairs = (need + 1) // 2
        if pairs:
            u = self._unit(2 * pairs).reshape(pairs, 2)
            if np.any(u[:, 0] <= 0.0):  # the reference redraws u1 until positive (p = 2^-53): exact slow path
                vals = []
                for a, b in u:
                    while a <= 0.0:
                        a = self._unit(1)[0]
                    r = np.sqrt(-2.0 * np.log(a))
                    vals += [r * np.cos(2.0 * np.pi * b), r * np.sin(2.0 * np.pi * b)]
                z = np.array(vals)
            else:
                r = np.sqrt(-2.0 * np.log(u[:, 0]))
                th = 2.0 * np.pi * u[:, 1]
                z = np.stack([r * np.cos(th), r * np.sin(th)], 1).reshape(-1)
            out[i:] = z[:need]
            if z.size > need:
                self._spare = float(z[need])
        return out

    def standard_normal(self, size=None):
        shape = () if size is None else size
        v = self._normal(int(np.prod(shape)))
        return v.reshape(shape) if size is not None else float(v[0])

    def normal(self, mu=0.0, sigma=1.0, size=None):
        shape = () if size is None else size
        v = mu + sigma * self._normal(int(np.prod(shape)))
        return v.reshape(shape) if size is not None else float(v[0])


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))


def camera(width, height, fx, fy, cx, cy, q=(1.0, 0.0, 0.0, 0.0), t=(0.0, 0.0, 0.0)):
    """cam_pose is world<-camera (gaussian_map.hpp:30), q = (w,x,y,z); +z forward, +y down."""
    return dict(q=np.array(q, np.float64), t=np.array(t, np.float64), fx=float(fx), fy=float(fy),
                cx=float(cx), cy=float(cy), width=int(width), height=int(height))


def _rot_to_quat(m):
    tr = m[0, 0] + m[1, 1] + m[2, 2]
    if tr > 0:
        s = math.sqrt(tr + 1.0) * 2
        w, x, y, z = 0.25 * s, (m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s, (m[1, 0] - m[0, 1]) / s
    elif m[0, 0] > m[1, 1] and m[0, 0] > m[2, 2]:
        s = math.sqrt(1.0 + m[0, 0] - m[1, 1] - m[2, 2]) * 2
        w, x, y, z = (m[2, 1] - m[1, 2]) / s, 0.25 * s, (m[0, 1] + m[1, 0]) / s, (m[0, 2] + m[2, 0]) / s
    elif m[1, 1] > m[2, 2]:
        s = math.sqrt(1.0 + m[1, 1] - m[0, 0] - m[2, 2]) * 2
        w, x, y, z = (m[0, 2] - m[2, 0]) / s, (m[0, 1] + m[1, 0]) / s, 0.25 * s, (m[1, 2] + m[2, 1]) / s
    else:
        s = math.sqrt(1.0 + m[2, 2] - m[0, 0] - m[1, 1]) * 2
        w, x, y, z = (m[1, 0] - m[0, 1]) / s, (m[0, 2] + m[2, 0]) / s, (m[1, 2] + m[2, 1]) / s, 0.25 * s
    q = np.array([w, x, y, z])
    return q / np.linalg.norm(q)


def look_at(center, target):
    """world<-camera pose at ``center`` with +z towards ``target`` and +y along world +y (down)."""
    c = np.asarray(center, np.float64)
    z = np.asarray(target, np.float64) - c
    z /= np.linalg.norm(z)
    x = np.cross(np.array([0.0, 1.0, 0.0]), z)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    return _rot_to_quat(np.stack([x, y, z], axis=1)), c


def _unit_quats(rng, n):
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q  # drawn as (w,x,y,z)


def _pack(pos, q_wxyz, log_s, opac, sh, feat_nd):
    rot = np.concatenate([q_wxyz[:, 1:4], q_wxyz[:, 0:1]], axis=1)  # -> Eigen storage x,y,z,w
    return dict(pos=_f32(pos), rot=_f32(rot), log_s=_f32(log_s), opac=_f32(opac), sh=_f32(sh),
                feat=_f32(np.ascontiguousarray(feat_nd.T)))


def _features(rng, n, d):
    f = rng.standard_normal((n, d))
    f /= np.linalg.norm(f, axis=1, keepdims=True)
    return f


def _sh(rng, n, deg, dc=None):
    K = (deg + 1) ** 2
    sh = np.zeros((n, K, 3))
    sh[:, 0, :] = rng.uniform(0.0, 1.0, (n, 3)) if dc is None else dc
    if K > 1:
        sh[:, 1:, :] = rng.normal(0.0, 0.05, (n, K - 1, 3))
    return sh


def make_config(name: str, n: int | None = None, d: int = 16, rng: str = "pcg64"):
    """Returns (scene, [cameras], info) for a BASELINE.json config.

    c0      : configs[0]  160x120, 10k, SH0, identity pose.
    c1      : configs[1]  640x480, 200k, SH3, identity pose (+ pose gradient).
    c1_500k : the BASELINE metric workload: configs[1] distributions at 500k.
    c2      : configs[2]  1200x680, 1M, 200 blobs, SH3.
    c3      : configs[3]  500k (config-1 distributions), 8 views on a 1 m circle.
    c4      : configs[4]  3M, 70% in a 0.5 m sphere, 16 views on a 2 m arc.
    rng     : "pcg64" (numpy, the default of every test and bench line) or "reference" (the same
              draws from the reference's lego::Rng stream, RefRng: reproducible by a C++ program
              calling the reference's generator in the same order).
    """
    cid = {"c0": 0, "c1": 1, "c1_500k": 1, "c2": 2, "c3": 3, "c4": 4}[name]
    if rng not in ("pcg64", "reference"):
        raise ValueError(rng)
    info = dict(config=name, seed=1000 + cid, rng=rng)
    # rng="reference": the same draws from the reference's own lego::Rng stream (RefRng)
    rng = RefRng(1000 + cid) if rng == "reference" else np.random.Generator(np.random.PCG64(1000 + cid))
    if name == "c0":
        n = n or 10_000
        pos = np.stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), rng.uniform(2, 5, n)], 1)
        scene = _pack(pos, _unit_quats(rng, n), rng.normal(-3, 0.5, (n, 3)), rng.normal(0, 1, n), _sh(rng, n, 0),
                      _features(rng, n, d))
        cams = [camera(160, 120, 140, 140, 80, 60)]
        info.update(depth_range=(2.0, 5.0))
    elif name in ("c1", "c1_500k", "c3"):
        n = n or (200_000 if name == "c1" else 500_000)
        pos = np.stack([rng.uniform(-2, 2, n), rng.uniform(-2, 2, n), rng.uniform(0.5, 6, n)], 1)
        scene = _pack(pos, _unit_quats(rng, n), rng.normal(-3, 0.5, (n, 3)), rng.normal(0, 1, n), _sh(rng, n, 3),
                      _features(rng, n, d))
        K = dict(width=640, height=480, fx=577.6, fy=577.6, cx=319.5, cy=239.5)
        if name == "c3":
            # pinned: 8 cameras on a 1 m circle in the z = 0 plane around the optical axis of
            # config 1, each looking at the cloud centre (0, 0, 3.25)
            cams = []
            for i in range(8):
                th = 2 * math.pi * i / 8
                q, t = look_at([math.cos(th), math.sin(th), 0.0], [0.0, 0.0, 3.25])
                cams.append(camera(q=q, t=t, **K))
        else:
            cams = [camera(**K)]
        info.update(depth_range=(0.5, 6.0))
    elif name == "c2":
        n = n or 1_000_000
        nb = 200
        centres = np.stack([rng.uniform(-3, 3, nb), rng.uniform(-1.5, 1.5, nb), rng.uniform(-3, 3, nb)], 1)
        blob_feat = rng.standard_normal((nb, d))
        which = rng.integers(0, nb, n)
        pos = centres[which] + rng.normal(0, 0.3, (n, 3))
        f = blob_feat[which] + rng.normal(0, 0.1, (n, d))
        f /= np.linalg.norm(f, axis=1, keepdims=True)
        scene = _pack(pos, _unit_quats(rng, n), rng.normal(-4, 0.7, (n, 3)), rng.normal(0, 1, n), _sh(rng, n, 3), f)
        # pinned: camera on the room wall z = -3.2, looking along +z through the room centre
        cams = [camera(1200, 680, 600, 600, 599.5, 339.5, t=(0.0, 0.0, -3.2))]
        info.update(depth_range=(0.5, 6.5))
    elif name == "c4":
        n = n or 3_000_000
        n_in = int(round(0.7 * n))
        n_out = n - n_in
        # 70%: uniform in a 0.5 m ball at (0, 0, 1.5), anisotropic scales
        v = rng.standard_normal((n_in, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        r = 0.5 * rng.uniform(0, 1, n_in) ** (1.0 / 3.0)
        p_in = v * r[:, None] + np.array([0.0, 0.0, 1.5])
        ls_in = np.stack([rng.normal(-1, 0.3, n_in), rng.normal(-5, 0.3, n_in), rng.normal(-5, 0.3, n_in)], 1)
        ol_in = rng.normal(1, 1, n_in)
        # pinned: remaining 30% follow the config-1 distributions
        p_out = np.stack([rng.uniform(-2, 2, n_out), rng.uniform(-2, 2, n_out), rng.uniform(0.5, 6, n_out)], 1)
        ls_out = rng.normal(-3, 0.5, (n_out, 3))
        ol_out = rng.normal(0, 1, n_out)
        pos = np.concatenate([p_in, p_out])
        scene = _pack(pos, _unit_quats(rng, n), np.concatenate([ls_in, ls_out]), np.concatenate([ol_in, ol_out]),
                      _sh(rng, n, 3), _features(rng, n, d))
        # pinned: 16 cameras on a 2 m long arc of radius 1.5 m around the sphere centre (x-z plane)
        cams = []
        span = 2.0 / 1.5
        for i in range(16):
            th = (i / 15.0 - 0.5) * span
            q, t = look_at([1.5 * math.sin(th), 0.0, 1.5 - 1.5 * math.cos(th)], [0.0, 0.0, 1.5])
            cams.append(camera(1200, 680, 600, 600, 599.5, 339.5, q=q, t=t))
        info.update(depth_range=(0.5, 6.0))
    else:
        raise ValueError(name)
    info["n"] = n
    return scene, cams, info


def make_targets(cam, d, depth_range, seed):
    """Seeded L1 targets (pinned): rgb U[0,1], depth U[depth_range], feature U[-1,1]; HWC fp32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    H, W = cam["height"], cam["width"]
    return dict(rgb=_f32(rng.uniform(0, 1, (H, W, 3))), depth=_f32(rng.uniform(*depth_range, (H, W))),
                feat=_f32(rng.uniform(-1, 1, (H, W, d))))


def l1_cotangents(rgb, depth, feat, targets):
    """dL/d(image) of L = mean|rgb-T| + mean|depth-T| + mean|feat-T| (sign(0) = 0)."""
    g_rgb = np.sign(rgb - targets["rgb"]) / rgb.size
    g_depth = np.sign(depth - targets["depth"]) / depth.size
    g_feat = np.sign(feat - targets["feat"]) / max(feat.size, 1)
    return g_rgb, g_depth, g_feat


def make_decoder(D: int, hidden: int, d: int, seed: int):
    """Seeded stand-in for a pretrained codec decoder (no checkpoint ships with the reference):
    (w1 [hidden, d], b1 [hidden], w2 [D, hidden], b2 [D]) float32, weights with the reference's
    Xavier-uniform scale (proj/src/codec.cpp:16-23), small random biases (a pretrained decoder has
    non-zero biases)."""
    r = np.random.default_rng(seed)

    def xavier(rows, cols):
        a = np.sqrt(6.0 / (rows + cols))
        return r.uniform(-a, a, size=(rows, cols))

    w1 = xavier(hidden, d)
    w2 = xavier(D, hidden)
    b1 = r.normal(0.0, 0.05, size=hidden)
    b2 = r.normal(0.0, 0.05, size=D)
    return tuple(x.astype(np.float32) for x in (w1, b1, w2, b2))


def make_prune_scene(n: int = 20000, d: int = 16, seed: int = 5, objects: int = 24, duplicate: float = 0.5,
                     jitter: float = 0.004, feat_noise: float = 0.05, coherent: bool = True, extent: float = 1.0):
    """A cluttered synthetic map for the pruning study ("duplicated insertion pass",
    InsertConfig duplicate / duplicate_jitter = 0.004 m, gaussian_map.hpp:102-110): `objects`
    spheres in an `extent`-metre box, each with its own unit feature; a Gaussian lies on its
    sphere with that feature plus N(0, feat_noise) noise; a `duplicate` fraction of them is
    inserted a second time `jitter` metres (N(0, jitter) per axis) away with fresh feature noise.
    Opacity logits U(-4, 3) and scales U(0.002, 0.05) m (5 %: U(0.4, 0.9) m) make some Gaussians
    fail the geometric criteria.  `coherent`: IDs in insertion order (object by object, the duplicates
    after them) as a SLAM map grows; else a random permutation."""
    rng = np.random.default_rng(seed)
    base_n = max(1, int(round(n / (1.0 + duplicate))))
    centers = rng.uniform(-extent / 2, extent / 2, (objects, 3))
    radii = rng.uniform(0.05, 0.25, objects)
    fobj = rng.standard_normal((objects, max(d, 1)))
    fobj /= np.linalg.norm(fobj, axis=1, keepdims=True)
    obj = np.sort(rng.integers(0, objects, base_n))
    dirs = rng.standard_normal((base_n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    pos = centers[obj] + radii[obj, None] * dirs
    feat = fobj[obj] + feat_noise * rng.standard_normal((base_n, max(d, 1)))
    nd = n - base_n
    src = np.sort(rng.choice(base_n, size=nd, replace=nd > base_n)) if nd > 0 else np.zeros(0, np.int64)
    pos = np.concatenate([pos, pos[src] + jitter * rng.standard_normal((nd, 3))])
    feat = np.concatenate([feat, feat[src] + feat_noise * rng.standard_normal((nd, max(d, 1)))])
    if not coherent:
        perm = rng.permutation(n)
        pos, feat = pos[perm], feat[perm]
    log_s = np.log(np.where(rng.uniform(size=(n, 1)) < 0.05, rng.uniform(0.4, 0.9, (n, 3)),
                            rng.uniform(0.002, 0.05, (n, 3))))
    opac = rng.uniform(-4.0, 3.0, n)
    return _pack(pos, _unit_quats(rng, n), log_s, opac, _sh(rng, n, 0), feat[:, :d])
