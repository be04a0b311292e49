"""TEST INFRASTRUCTURE ONLY -- ctypes front end of oracle/_ref/liblgs_ref.so: the reference's own
renderer (/root/reference/proj/src/renderer.cpp + geometry.cpp, unmodified) compiled here by
oracle/Makefile against the self-written Eigen subset in oracle/eigen_shim (see ref_bridge.cpp).

Only tests/, tests/golden/make_ref_golden.py and bench.py's --impl reference / cpu_baseline legs
load it; it exists only where /root/reference was present at build time (this container) or where
the built .so travelled with the repo snapshot.  Layouts are oracle A's (oracle.py).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from oracle.oracle import OrcCamera, OrcConfig, OrcMap, _scene64, make_camera, make_config

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "liblgs_ref.so")
UNIT_TESTS = os.path.join(_HERE, "_ref", "ref_unit_tests")

_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.ref_find_language_redundant.restype = C.c_int64
        L.ref_find_language_redundant.argtypes = [C.c_int64, C.c_int32, _dp, _dp, C.c_int32, C.c_double,
                                                  C.c_double, C.POINTER(C.c_uint8)]
        L.ref_render.restype = C.c_void_p
        L.ref_render.argtypes = [C.POINTER(OrcMap), C.POINTER(OrcCamera), C.POINTER(OrcConfig), _dp, _dp, _dp, _dp]
        L.ref_num_projected.restype = C.c_int64
        L.ref_num_projected.argtypes = [C.c_void_p]
        L.ref_sorted_indices.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        L.ref_contrib_counts.argtypes = [C.c_void_p, _i32p]
        L.ref_render_backward.restype = C.c_int
        L.ref_render_backward.argtypes = [C.c_void_p, _dp, _i32p, _dp, _i32p, _dp, _i32p, _dp, _dp, _dp, _dp, _dp, _dp]
        L.ref_render_free.argtypes = [C.c_void_p]
        L.ref_project_gaussian.restype = C.c_int
        L.ref_project_gaussian.argtypes = [C.POINTER(OrcMap), C.c_int64, C.POINTER(OrcCamera), C.POINTER(OrcConfig), _dp,
                                           _dp, _dp]
        L.ref_grad_scene.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, _dp, _dp, _dp, _dp, _dp, _dp,
                                     C.POINTER(OrcCamera), C.POINTER(OrcConfig), _dp, _dp, _dp]
        L.ref_gradcheck.restype = C.c_double
        L.ref_gradcheck.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64]
        L.ref_bench_bands.restype = C.c_double
        L.ref_bench_bands.argtypes = [C.POINTER(OrcMap), C.POINTER(OrcCamera), C.POINTER(OrcConfig), _dp, _dp, _dp,
                                      C.c_int, C.c_int, _dp]
        L.ref_bench.restype = C.c_double
        L.ref_bench.argtypes = [C.POINTER(OrcMap), C.POINTER(OrcCamera), C.POINTER(OrcConfig), _dp, _dp, _dp, C.c_int,
                                C.c_int, _dp]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _sh0(scene):
    """The reference has colours only (SH degree 0): higher bands are rejected, not dropped."""
    if scene["sh"].shape[1] != 1:
        raise ValueError("the reference renderer has SH degree 0 (colours) only")


class RefRender:
    def __init__(self, h, keep, rgb, depth, feat, acc, n, d):
        self._h, self._keep = h, keep
        self.rgb, self.depth, self.feat, self.acc = rgb, depth, feat, acc
        self.n, self.d = n, d

    @property
    def num_projected(self):
        return lib().ref_num_projected(self._h)

    def sorted_indices(self):
        out = np.zeros(self.num_projected, np.int64)
        lib().ref_sorted_indices(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out

    def contrib_counts(self):
        out = np.zeros(self.depth.shape, np.int32)
        lib().ref_contrib_counts(self._h, out.ctypes.data_as(_i32p))
        return out

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_render_free(self._h)
            self._h = None


def render(scene, cam, cfg=None) -> RefRender:
    """lego::render (renderer.cpp:94-167) of the reference build.  HWC fp64 images."""
    _sh0(scene)
    m, s = _scene64(scene)
    c = make_camera(cam)
    cfg = cfg if isinstance(cfg, OrcConfig) else make_config(**(cfg or {}))
    H, W, d = c.height, c.width, m.d
    rgb, depth, acc = np.zeros((H, W, 3)), np.zeros((H, W)), np.zeros((H, W))
    feat = np.zeros((H, W, d))
    h = lib().ref_render(C.byref(m), C.byref(c), C.byref(cfg), _ptr(rgb), _ptr(depth), _ptr(feat) if d else None,
                         _ptr(acc))
    return RefRender(h, (m, s, c, cfg), rgb, depth, feat, acc, m.n, d)


def render_backward(r: RefRender, g_rgb=None, g_depth=None, g_feat=None):
    """lego::render_backward (renderer.cpp:169-356).  None = the reference's empty image.  Raises
    ValueError where the reference throws std::invalid_argument (cotangent shape mismatch)."""
    n, d = r.n, r.d

    def img(g, ch):
        if g is None:
            return None, None
        g = np.ascontiguousarray(g, dtype=np.float64)
        shp = g.shape if g.ndim == 3 else (g.shape + (1,) if g.ndim == 2 else g.shape)
        return g, np.array(shp if len(shp) == 3 else (0, 0, 0), np.int32)

    (gr, sr), (gd, sd), (gf, sf) = img(g_rgb, 3), img(g_depth, 1), img(g_feat, d)
    out = dict(position=np.zeros((n, 3)), rotation=np.zeros((n, 4)), log_scale=np.zeros((n, 3)),
               opacity_logit=np.zeros(n), sh=np.zeros((n, 1, 3)), feature=np.zeros((d, n)))
    rc = lib().ref_render_backward(r._h, _ptr(gr), sr.ctypes.data_as(_i32p) if sr is not None else None, _ptr(gd),
                                   sd.ctypes.data_as(_i32p) if sd is not None else None, _ptr(gf),
                                   sf.ctypes.data_as(_i32p) if sf is not None else None,
                                   *(_ptr(out[k]) for k in ("position", "rotation", "log_scale", "opacity_logit",
                                                            "sh", "feature")))
    if rc == 1:
        raise ValueError("render_backward: bad cotangent shape (std::invalid_argument)")
    return out


def project_gaussian(scene, index, cam, cfg=None):
    m, s = _scene64(scene)
    c = make_camera(cam)
    cfg = cfg if isinstance(cfg, OrcConfig) else make_config(**(cfg or {}))
    a, cov, con = np.zeros(4), np.zeros(4), np.zeros(4)
    if not lib().ref_project_gaussian(C.byref(m), index, C.byref(c), C.byref(cfg), _ptr(a), _ptr(cov), _ptr(con)):
        return None
    return dict(u=a[0], v=a[1], depth=a[2], radius=a[3], cov2d=cov.reshape(2, 2), conic=con.reshape(2, 2))


def grad_scene(n=12, size=16, d=8, seed=101):
    """legotest::make_grad_scene (gradcheck.hpp:31-78) as built by this compiler: (scene, cam, cfg,
    w_rgb, w_depth, w_feat) with scene in oracle layouts (SH0)."""
    pos, rot, log_s = np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 3))
    opac, color, feat = np.zeros(n), np.zeros((n, 3)), np.zeros((d, n))
    cam, cfg = OrcCamera(), OrcConfig()
    w_rgb, w_depth, w_feat = np.zeros((size, size, 3)), np.zeros((size, size)), np.zeros((size, size, d))
    lib().ref_grad_scene(n, size, d, seed, *(_ptr(x) for x in (pos, rot, log_s, opac, color, feat)), C.byref(cam),
                         C.byref(cfg), _ptr(w_rgb), _ptr(w_depth), _ptr(w_feat))
    scene = dict(pos=pos, rot=rot, log_s=log_s, opac=opac, sh=color.reshape(n, 1, 3), feat=feat)
    camd = dict(q=list(cam.q), t=list(cam.t), fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=cam.width,
                height=cam.height)
    cfgd = {k: getattr(cfg, k) for k, _ in OrcConfig._fields_}
    return scene, camd, cfgd, w_rgb, w_depth, w_feat


def gradcheck(n=12, size=16, d=8, seed=101) -> float:
    """legotest::gradcheck_scene: max relative FD error of the reference's own backward."""
    return lib().ref_gradcheck(n, size, d, seed)


def bench(scene, cam, targets, threads, iters, cfg=None):
    """Wall seconds for `threads` x `iters` reference steps (render, L1 cotangents, render_backward)."""
    _sh0(scene)
    m, s = _scene64(scene)
    c = make_camera(cam)
    cfg = cfg if isinstance(cfg, OrcConfig) else make_config(**(cfg or {}))
    t = [np.ascontiguousarray(targets[k], dtype=np.float64) for k in ("rgb", "depth", "feat")]
    loss = np.zeros(1)
    sec = lib().ref_bench(C.byref(m), C.byref(c), C.byref(cfg), *(_ptr(x) for x in t), threads, iters, _ptr(loss))
    return sec, float(loss[0])


def bench_bands(scene, cam, targets, threads, iters, cfg=None):
    """Seconds per step of the full image's fwd+bwd split into `threads` row bands, each band the
    reference's own lego::render + render_backward (ref_bridge.cpp ref_bench_bands); and the L1 loss."""
    _sh0(scene)
    m, s = _scene64(scene)
    c = make_camera(cam)
    cfg = cfg if isinstance(cfg, OrcConfig) else make_config(**(cfg or {}))
    t = [np.ascontiguousarray(targets[k], dtype=np.float64) for k in ("rgb", "depth", "feat")]
    loss = np.zeros(1)
    sec = lib().ref_bench_bands(C.byref(m), C.byref(c), C.byref(cfg), *(_ptr(x) for x in t), threads, iters,
                                _ptr(loss))
    return sec, float(loss[0])


def find_language_redundant(scene, k=8, tau_dist=0.02, tau_sim=0.9):
    """The SPEC's Eq. 4 sweep on the reference's own KdTree3 (ref_bridge.cpp); uint8 flags."""
    from oracle.oracle import prune_inputs
    pos, feat = prune_inputs(scene)
    n, d = pos.shape[0], feat.shape[0]
    flags = np.zeros(max(n, 1), np.uint8)
    lib().ref_find_language_redundant(n, d, _ptr(pos), _ptr(feat), int(k), float(tau_dist), float(tau_sim),
                                      flags.ctypes.data_as(C.POINTER(C.c_uint8)))
    return flags[:n]
