"""Scene builders that restate the reference's renderer test fixtures.

proj/tests/test_renderer.cpp:14-36 (small_camera, splat_at, logit) and
proj/tests/gradcheck.hpp:31-78 (make_grad_scene) + :80-148 (scene_loss,
rel_err, gradcheck_scene).  Draws use the reference Rng (random.hpp) through
the oracle.  C++ leaves constructor-argument evaluation order unspecified; the
reference built here with g++ (oracle/_ref, tests/test_reference_build.py)
evaluates them right to left, so multi-draw constructors (Vec3(u(), u(), u()),
Quat(n(), n(), n(), n())) are drawn last argument first, which makes
make_grad_scene reproduce the reference's seed-101 scene value for value.
"""
import math

import numpy as np


def small_camera():
    """test_renderer.cpp:14-20."""
    return dict(q=[1.0, 0.0, 0.0, 0.0], t=[0.0, 0.0, 0.0], fx=100.0, fy=100.0, cx=31.5, cy=31.5, width=64,
                height=64)


def logit(p):
    return math.log(p / (1.0 - p))


class MapBuilder:
    """Minimal GaussianMap (gaussian_map.hpp:41-94) restated as growable lists."""

    def __init__(self, d, sh_degree=0):
        self.d = d
        self.K = (sh_degree + 1) ** 2
        self.pos, self.rot, self.log_s, self.opac, self.sh, self.feat = [], [], [], [], [], []

    def insert(self, position, rotation_wxyz, log_scale, opacity_logit, color, feature, sh_rest=None):
        q = np.asarray(rotation_wxyz, dtype=np.float64)
        if abs(np.linalg.norm(q) - 1.0) > 1e-6:  # gaussian_map.cpp:23-24
            q = q / np.linalg.norm(q)
        self.pos.append(list(position))
        self.rot.append([q[1], q[2], q[3], q[0]])  # Eigen storage x,y,z,w
        self.log_s.append(list(log_scale))
        self.opac.append(opacity_logit)
        sh = np.zeros((self.K, 3))
        sh[0] = color
        if sh_rest is not None:
            sh[1:] = sh_rest
        self.sh.append(sh)
        self.feat.append(list(feature))

    def scene(self):
        n = len(self.pos)
        return dict(pos=np.array(self.pos, dtype=np.float64).reshape(n, 3),
                    rot=np.array(self.rot, dtype=np.float64).reshape(n, 4),
                    log_s=np.array(self.log_s, dtype=np.float64).reshape(n, 3),
                    opac=np.array(self.opac, dtype=np.float64).reshape(n),
                    sh=np.array(self.sh, dtype=np.float64).reshape(n, self.K, 3),
                    feat=np.array(self.feat, dtype=np.float64).reshape(n, self.d).T.copy())


def splat_at(mb, p, scale, opacity_logit, color, feature=None):
    """test_renderer.cpp:22-32."""
    mb.insert(p, [1, 0, 0, 0], [math.log(scale)] * 3, opacity_logit, color,
              feature if feature is not None else [0.0] * mb.d)


def make_grad_scene(o, n_gaussians, image_size, feat_dim, seed, sh_degree=0):
    """gradcheck.hpp:31-78.  Returns (scene, cam, cfg, w_rgb, w_depth, w_feat).

    With sh_degree > 0 (EXT) the higher SH bands are drawn after all reference
    draws, so the SH0 part of the scene is unchanged."""
    rng = o.Rng(seed)
    mb = MapBuilder(feat_dim, sh_degree)
    cam = dict(q=[1.0, 0, 0, 0], t=[0.0, 0, 0], fx=1.4 * image_size, fy=1.4 * image_size,
               cx=(image_size - 1) / 2.0, cy=(image_size - 1) / 2.0, width=image_size, height=image_size)
    cfg = dict(radius_sigma=1e3, alpha_skip=1e-12, transmittance_min=0.0)  # :41-43
    for _ in range(n_gaussians):
        # constructor arguments in GCC's right-to-left evaluation order (see the module docstring)
        z = rng.uniform(0.8, 2.2)
        py_ = rng.uniform(-0.3, 0.3) * z
        p = [rng.uniform(-0.3, 0.3) * z, py_, z]
        q = np.array([rng.normal(), rng.normal(), rng.normal(), rng.normal()])[::-1].copy()  # Quat(w,x,y,z)
        # q.normalize(): the norm summed in Eigen's storage order (x, y, z, w)
        q /= math.sqrt(((q[1] * q[1] + q[2] * q[2]) + q[3] * q[3]) + q[0] * q[0])
        ls = [math.log(rng.uniform(0.04, 0.12)) for _ in range(3)][::-1]
        ol = rng.uniform(0.5, 2.2)
        col = [rng.uniform(0.05, 0.95) for _ in range(3)][::-1]
        f = [0.5 * rng.normal() for _ in range(feat_dim)]
        mb.insert(p, q, ls, ol, col, f)
    scene = mb.scene()
    w_rgb = np.array([rng.uniform(-1, 1) for _ in range(image_size * image_size * 3)]).reshape(
        image_size, image_size, 3)
    w_feat = np.array([rng.uniform(-1, 1) for _ in range(image_size * image_size * feat_dim)]).reshape(
        image_size, image_size, feat_dim)
    base = o.render(scene, cam, cfg)
    w_depth = np.zeros((image_size, image_size))
    for y in range(image_size):
        for x in range(image_size):
            w_depth[y, x] = rng.uniform(-1, 1) if base.acc[y, x] > 0.2 else 0.0
    if sh_degree > 0:
        K = (sh_degree + 1) ** 2
        rest = np.array([0.2 * rng.normal() for _ in range(n_gaussians * (K - 1) * 3)]).reshape(
            n_gaussians, K - 1, 3)
        scene["sh"][:, 1:, :] = rest
    return scene, cam, cfg, w_rgb, w_depth, w_feat


def scene_loss(o, scene, cam, cfg, w_rgb, w_depth, w_feat):
    """gradcheck.hpp:80-93."""
    out = o.render(scene, cam, cfg)
    return float((out.rgb * w_rgb).sum() + (out.feat * w_feat).sum() + (out.depth * w_depth).sum())


def rel_err(a, b):
    """gradcheck.hpp:101-103 (absolute floor 1e-2)."""
    return abs(a - b) / max(abs(a), abs(b), 1e-2)
