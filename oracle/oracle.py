"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle (liblgs_oracle.so).

The oracle is the checker for the CUDA rasterizer, never the product: only
tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs import it.

* ``render`` / ``render_backward``: oracle A, the fp64 restatement of the
  reference ``lego::render`` / ``lego::render_backward``
  (proj/src/renderer.cpp:94-356), with the SH / pose / window / injection
  extensions described in lgs_oracle.c.
* ``preprocess_f32`` / ``bin_f32``: oracle B, the fp32 twin of the product
  preprocess and the (tile | depth) key list, stable sort and tile ranges.
* ``Rng``: the reference's seeded generator (proj/include/legoslam/random.hpp).

Scenes are plain dicts of numpy arrays in the reference layouts
(gaussian_map.hpp:57-93): ``pos`` [N,3], ``rot`` [N,4] (x,y,z,w),
``log_s`` [N,3], ``opac`` [N] (logits), ``sh`` [N,K,3], ``feat`` [d,N].
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblgs_oracle.so")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)


class OrcConfig(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "near_plane", "dilation", "alpha_clamp", "alpha_skip", "transmittance_min", "radius_sigma")]


class OrcCamera(C.Structure):
    _fields_ = [("q", C.c_double * 4), ("t", C.c_double * 3), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("width", C.c_int32), ("height", C.c_int32)]


class OrcMap(C.Structure):
    _fields_ = [("n", C.c_int64), ("d", C.c_int32), ("sh_degree", C.c_int32), ("pos", _dp), ("rot", _dp),
                ("log_s", _dp), ("opac", _dp), ("sh", _dp), ("feat", _dp)]


class OrcInject(C.Structure):
    _fields_ = [("visible", _u8p), ("u", _fp), ("v", _fp), ("conic", _fp), ("depth", _fp), ("bbox", _i32p),
                ("opacity", _fp), ("color", _fp)]


class Orc32Cam(C.Structure):
    _fields_ = [("rcw", C.c_float * 9), ("tcw", C.c_float * 3), ("cc", C.c_float * 3), ("fx", C.c_float),
                ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32),
                ("height", C.c_int32), ("near_plane", C.c_float), ("dilation", C.c_float),
                ("radius_sigma", C.c_float), ("alpha_skip", C.c_float)]


def build():
    """Compile liblgs_oracle.so (gcc, see oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
                os.path.getmtime(os.path.join(_HERE, f)) for f in ("lgs_oracle.c", "prune_oracle.c")):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_render_forward.restype = C.c_void_p
        L.orc_render_forward.argtypes = [C.POINTER(OrcMap), C.POINTER(OrcCamera), C.POINTER(OrcConfig),
                                         C.POINTER(OrcInject), _i32p, _dp, _dp, _dp, _dp]
        L.orc_render_backward.restype = C.c_int
        L.orc_render_backward.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_render_free.argtypes = [C.c_void_p]
        L.orc_find_language_redundant.restype = C.c_int64
        L.orc_find_language_redundant.argtypes = [C.c_int64, C.c_int32, _dp, _dp, C.c_int32, C.c_double, C.c_double,
                                                  _u8p]
        L.orc_find_geometric.restype = C.c_int64
        L.orc_find_geometric.argtypes = [C.c_int64, _dp, _dp, C.c_double, C.c_double, _u8p]
        for f in ("orc_render_num_projected", "orc_render_num_evaluated", "orc_render_num_contributions"):
            getattr(L, f).restype = C.c_int64
            getattr(L, f).argtypes = [C.c_void_p]
        L.orc_render_contrib_counts.argtypes = [C.c_void_p, _i32p]
        L.orc_render_flags.restype = C.c_int
        L.orc_render_flags.argtypes = [C.c_void_p, _u8p, _u8p]
        L.orc_render_sorted_indices.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        L.orc_project_gaussian.restype = C.c_int
        L.orc_project_gaussian.argtypes = [C.POINTER(OrcMap), C.c_int64, C.POINTER(OrcCamera),
                                           C.POINTER(OrcConfig), _dp, _dp, _dp]
        L.orc_perturb_pose.argtypes = [_dp, _dp, _dp, _dp, _dp]
        L.orc_fwd_bwd_bands.restype = C.c_int
        L.orc_fwd_bwd_bands.argtypes = [C.POINTER(OrcMap), C.POINTER(OrcCamera), C.POINTER(OrcConfig), C.c_int32,
                                        C.c_int32, C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                        _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_expf_export.restype = C.c_float
        L.orc_expf_export.argtypes = [C.c_float]
        L.orc_logf_export.restype = C.c_float
        L.orc_logf_export.argtypes = [C.c_float]
        L.orc32_camera_setup.argtypes = [C.POINTER(OrcCamera), C.POINTER(OrcConfig), C.POINTER(Orc32Cam)]
        L.orc32_preprocess.restype = C.c_int64
        L.orc32_preprocess.argtypes = [C.c_int64, C.c_int32, _fp, _fp, _fp, _fp, _fp, C.POINTER(Orc32Cam), _u8p,
                                       _fp, _fp, _fp, _fp, _fp, _i32p, _fp, _fp, _i32p]
        L.orc32_bin.restype = C.c_int64
        L.orc32_bin.argtypes = [C.c_int64, _u8p, _fp, _i32p, C.c_int32, C.c_int32, C.POINTER(C.c_uint64),
                                C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.orc_rng_new.restype = C.c_void_p
        L.orc_rng_new.argtypes = [C.c_uint64]
        L.orc_rng_free.argtypes = [C.c_void_p]
        L.orc_rng_next_u64.restype = C.c_uint64
        L.orc_rng_next_u64.argtypes = [C.c_void_p]
        L.orc_rng_uniform.restype = C.c_double
        L.orc_rng_uniform.argtypes = [C.c_void_p]
        L.orc_rng_normal.restype = C.c_double
        L.orc_rng_normal.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


# --------------------------------------------------------------------------------------------
# configs / cameras
# --------------------------------------------------------------------------------------------

DEFAULT_CONFIG = dict(near_plane=0.01, dilation=0.3, alpha_clamp=0.99, alpha_skip=1.0 / 255.0,
                      transmittance_min=1e-4, radius_sigma=3.0)  # renderer.hpp:15-22


def make_config(**kw):
    d = dict(DEFAULT_CONFIG)
    d.update(kw)
    return OrcConfig(**d)


def make_camera(cam):
    """cam: dict with q (w,x,y,z), t, fx, fy, cx, cy, width, height."""
    c = OrcCamera()
    for i in range(4):
        c.q[i] = float(cam["q"][i])
    for i in range(3):
        c.t[i] = float(cam["t"][i])
    c.fx, c.fy, c.cx, c.cy = (float(cam[k]) for k in ("fx", "fy", "cx", "cy"))
    c.width, c.height = int(cam["width"]), int(cam["height"])
    return c


def _scene64(scene):
    s = {}
    for k in ("pos", "rot", "log_s", "opac", "sh", "feat"):
        s[k] = np.ascontiguousarray(scene[k], dtype=np.float64)
    n = s["pos"].shape[0]
    d = s["feat"].shape[0]
    K = s["sh"].shape[1] if s["sh"].ndim == 3 else 1
    deg = {1: 0, 4: 1, 9: 2, 16: 3}[K]
    m = OrcMap(n=n, d=d, sh_degree=deg, pos=_ptr(s["pos"], _dp), rot=_ptr(s["rot"], _dp),
               log_s=_ptr(s["log_s"], _dp), opac=_ptr(s["opac"], _dp), sh=_ptr(s["sh"], _dp),
               feat=_ptr(s["feat"], _dp))
    return m, s


# --------------------------------------------------------------------------------------------
# oracle A
# --------------------------------------------------------------------------------------------

class Render:
    """Holds the oracle's RenderOutput (renderer.hpp:33-45) and the arrays it points to."""

    def __init__(self, handle, keep, rgb, depth, feat, acc, n, d, K):
        self._h = handle
        self._keep = keep
        self.rgb, self.depth, self.feat, self.acc = rgb, depth, feat, acc
        self.n, self.d, self.K = n, d, K

    @property
    def num_projected(self):
        return lib().orc_render_num_projected(self._h)

    @property
    def num_evaluated(self):
        return lib().orc_render_num_evaluated(self._h)

    @property
    def num_contributions(self):
        return lib().orc_render_num_contributions(self._h)

    def contrib_counts(self):
        out = np.zeros(self.depth.shape[:2], np.int32)
        lib().orc_render_contrib_counts(self._h, _ptr(out, _i32p))
        return out

    def flags(self):
        """fp32 decision-twin flags of an injected render (lgs_oracle.c orc_render.pix_flag):
        (pixel flags [H,W] uint8, Gaussian flags [N] uint8), or None without injection."""
        pf = np.zeros(self.depth.shape[:2], np.uint8)
        gf = np.zeros(max(self.n, 1), np.uint8)
        if not lib().orc_render_flags(self._h, _ptr(pf, _u8p), _ptr(gf, _u8p)):
            return None
        return pf, gf[:self.n]

    def sorted_indices(self):
        out = np.zeros(self.num_projected, np.int64)
        lib().orc_render_sorted_indices(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_render_free(self._h)
            self._h = None


def render(scene, cam, cfg=None, inject=None, window=None):
    """Oracle A forward (renderer.cpp:94-167).  Returns a Render with HWC fp64 images."""
    L = lib()
    m, s = _scene64(scene)
    c = make_camera(cam)
    cfg = cfg if isinstance(cfg, OrcConfig) else make_config(**(cfg or {}))
    H, W, d = c.height, c.width, m.d
    rgb = np.zeros((H, W, 3))
    depth = np.zeros((H, W))
    feat = np.zeros((H, W, max(d, 1)))[:, :, :d] if d == 0 else np.zeros((H, W, d))
    acc = np.zeros((H, W))
    keep = [s, m, c, cfg]
    inj = None
    if inject is not None:
        ia = {k: np.ascontiguousarray(inject[k]) for k in inject}
        ia["visible"] = ia["visible"].astype(np.uint8)
        for k in ("u", "v", "conic", "depth", "opacity", "color"):
            ia[k] = ia[k].astype(np.float32)
        ia["bbox"] = ia["bbox"].astype(np.int32)
        inj = OrcInject(visible=_ptr(ia["visible"], _u8p), u=_ptr(ia["u"], _fp), v=_ptr(ia["v"], _fp),
                        conic=_ptr(ia["conic"], _fp), depth=_ptr(ia["depth"], _fp), bbox=_ptr(ia["bbox"], _i32p),
                        opacity=_ptr(ia["opacity"], _fp), color=_ptr(ia["color"], _fp))
        keep += [ia, inj]
    win = None
    if window is not None:
        win = np.ascontiguousarray(window, dtype=np.int32)
        keep.append(win)
    fbuf = feat if d > 0 else np.zeros(1)
    h = L.orc_render_forward(C.byref(m), C.byref(c), C.byref(cfg), C.byref(inj) if inj is not None else None,
                             _ptr(win, _i32p), _ptr(rgb, _dp), _ptr(depth, _dp), _ptr(fbuf, _dp), _ptr(acc, _dp))
    keep.append(fbuf)
    K = s["sh"].shape[1]
    return Render(h, keep, rgb, depth, feat, acc, m.n, d, K)


def render_backward(r: Render, g_rgb=None, g_depth=None, g_feat=None, pose=False):
    """Oracle A backward (renderer.cpp:169-356).  None cotangent = the reference's empty image.

    Returns dict: position [N,3], rotation [N,4] (w,x,y,z), log_scale [N,3], opacity_logit [N],
    sh [N,K,3], feature [d,N], and pose [6] (omega, nu) if ``pose``.
    """
    L = lib()
    n, d, K = r.n, r.d, r.K
    H, W = r.depth.shape

    def chk(g, ch, name):
        if g is None:
            return None
        g = np.ascontiguousarray(g, dtype=np.float64)
        if g.size == 0:
            return None
        if g.reshape(H, W, -1).shape != (H, W, ch) and not (ch == 1 and g.shape == (H, W)):
            raise ValueError(f"render_backward: bad shape for {name}")  # renderer.cpp:176-178
        return g

    g_rgb = chk(g_rgb, 3, "grad_rgb")
    g_depth = chk(g_depth, 1, "grad_depth")
    g_feat = chk(g_feat, d, "grad_feat") if d > 0 else None
    out = dict(position=np.zeros((n, 3)), rotation=np.zeros((n, 4)), log_scale=np.zeros((n, 3)),
               opacity_logit=np.zeros(n), sh=np.zeros((n, K, 3)), feature=np.zeros((max(d, 0), n)))
    pose6 = np.zeros(6) if pose else None
    fbuf = out["feature"] if d > 0 else np.zeros(1)
    L.orc_render_backward(r._h, _ptr(g_rgb, _dp), _ptr(g_depth, _dp), _ptr(g_feat, _dp),
                          _ptr(out["position"], _dp), _ptr(out["rotation"], _dp), _ptr(out["log_scale"], _dp),
                          _ptr(out["opacity_logit"], _dp), _ptr(out["sh"], _dp), _ptr(fbuf, _dp),
                          _ptr(pose6, _dp))
    if pose:
        out["pose"] = pose6
    return out


def project_gaussian(scene, index, cam, cfg=None):
    """renderer.cpp:53-92.  Returns None when culled, else dict(u, v, depth, radius, cov2d, conic)."""
    m, s = _scene64(scene)
    c = make_camera(cam)
    cfg = cfg if isinstance(cfg, OrcConfig) else make_config(**(cfg or {}))
    a = np.zeros(4)
    cov = np.zeros(4)
    con = np.zeros(4)
    ok = lib().orc_project_gaussian(C.byref(m), index, C.byref(c), C.byref(cfg), _ptr(a, _dp), _ptr(cov, _dp),
                                    _ptr(con, _dp))
    if not ok:
        return None
    return dict(u=a[0], v=a[1], depth=a[2], radius=a[3], cov2d=cov.reshape(2, 2), conic=con.reshape(2, 2))


def perturb_pose(cam, xi):
    """cam with pose replaced by compose(se3_exp(xi), pose) (geometry.cpp:8-13, 22-41)."""
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    q = np.ascontiguousarray(cam["q"], dtype=np.float64)
    t = np.ascontiguousarray(cam["t"], dtype=np.float64)
    qo = np.zeros(4)
    to = np.zeros(3)
    lib().orc_perturb_pose(_ptr(xi, _dp), _ptr(q, _dp), _ptr(t, _dp), _ptr(qo, _dp), _ptr(to, _dp))
    c2 = dict(cam)
    c2["q"], c2["t"] = qo, to
    return c2


def fwd_bwd_bands(scene, cam, g_rgb, g_depth, g_feat, threads, rows=None, cfg=None, targets=None):
    """All-cores reference fwd+bwd over image rows [lo, hi) (EXT, see lgs_oracle.c).

    With ``targets`` (dict rgb/depth/feat) the cotangents are the L1-loss ones computed per band
    from the band's own forward output (g_* are then ignored) and ``loss`` is returned."""
    L = lib()
    m, s = _scene64(scene)
    c = make_camera(cam)
    cfg = cfg if isinstance(cfg, OrcConfig) else make_config(**(cfg or {}))
    H, W, d, n = c.height, c.width, m.d, m.n
    K = s["sh"].shape[1]
    lo, hi = rows if rows is not None else (0, H)
    out = dict(rgb=np.zeros((H, W, 3)), depth=np.zeros((H, W)), feat=np.zeros((H, W, max(d, 1))),
               acc=np.zeros((H, W)), position=np.zeros((n, 3)), rotation=np.zeros((n, 4)),
               log_scale=np.zeros((n, 3)), opacity_logit=np.zeros(n), sh=np.zeros((n, K, 3)),
               feature=np.zeros((max(d, 1), n)), pose=np.zeros(6))
    g = [None if x is None else np.ascontiguousarray(x, dtype=np.float64) for x in (g_rgb, g_depth, g_feat)]
    t = [None, None, None]
    if targets is not None:
        t = [np.ascontiguousarray(targets[k], dtype=np.float64) for k in ("rgb", "depth", "feat")]
    loss = np.zeros(1)
    L.orc_fwd_bwd_bands(C.byref(m), C.byref(c), C.byref(cfg), lo, hi, threads, *(_ptr(x, _dp) for x in g),
                        *(_ptr(out[k], _dp) for k in ("rgb", "depth", "feat", "acc", "position", "rotation",
                                                       "log_scale", "opacity_logit", "sh", "feature", "pose")),
                        *(_ptr(x, _dp) for x in t), _ptr(loss, _dp))
    out["loss"] = float(loss[0])
    return out


# --------------------------------------------------------------------------------------------
# oracle B (fp32 twin)
# --------------------------------------------------------------------------------------------

def expf32(x: float) -> float:
    return lib().orc_expf_export(float(x))


def camera_f32(cam, cfg=None):
    c = make_camera(cam)
    cfg = cfg if isinstance(cfg, OrcConfig) else make_config(**(cfg or {}))
    out = Orc32Cam()
    lib().orc32_camera_setup(C.byref(c), C.byref(cfg), C.byref(out))
    return out


def preprocess_f32(scene, cam, cfg=None):
    """fp32 twin of the product preprocess.  Returns per-map-index records."""
    L = lib()
    c32 = camera_f32(cam, cfg)
    f = {k: np.ascontiguousarray(scene[k], dtype=np.float32) for k in ("pos", "rot", "log_s", "opac", "sh")}
    n = f["pos"].shape[0]
    K = f["sh"].shape[1]
    deg = {1: 0, 4: 1, 9: 2, 16: 3}[K]
    r = dict(visible=np.zeros(n, np.uint8), u=np.zeros(n, np.float32), v=np.zeros(n, np.float32),
             depth=np.zeros(n, np.float32), conic=np.zeros((n, 3), np.float32), radius=np.zeros(n, np.float32),
             bbox=np.zeros((n, 4), np.int32), opacity=np.zeros(n, np.float32), color=np.zeros((n, 3), np.float32),
             tiles_touched=np.zeros(n, np.int32))
    L.orc32_preprocess(n, deg, *(_ptr(f[k], _fp) for k in ("pos", "rot", "log_s", "opac", "sh")), C.byref(c32),
                       _ptr(r["visible"], _u8p), _ptr(r["u"], _fp), _ptr(r["v"], _fp), _ptr(r["depth"], _fp),
                       _ptr(r["conic"], _fp), _ptr(r["radius"], _fp), _ptr(r["bbox"], _i32p),
                       _ptr(r["opacity"], _fp), _ptr(r["color"], _fp), _ptr(r["tiles_touched"], _i32p))
    return r


def bin_f32(pre, width, height):
    """Key list (u64), values (u32 map index) and per-tile [begin, end) ranges."""
    L = lib()
    n = pre["visible"].shape[0]
    args = (n, _ptr(pre["visible"], _u8p), _ptr(pre["depth"], _fp), _ptr(pre["bbox"], _i32p), width, height)
    P = L.orc32_bin(*args, None, None, None)
    keys = np.zeros(max(P, 1), np.uint64)
    vals = np.zeros(max(P, 1), np.uint32)
    ntiles = ((width + 15) // 16) * ((height + 15) // 16)
    ranges = np.zeros((ntiles, 2), np.uint32)
    L.orc32_bin(*args, keys.ctypes.data_as(C.POINTER(C.c_uint64)), vals.ctypes.data_as(C.POINTER(C.c_uint32)),
                ranges.ctypes.data_as(C.POINTER(C.c_uint32)))
    return keys[:P], vals[:P], ranges


# --------------------------------------------------------------------------------------------
# Rng (random.hpp)
# --------------------------------------------------------------------------------------------

class Rng:
    def __init__(self, seed):
        self._h = lib().orc_rng_new(seed)

    def next_u64(self):
        return lib().orc_rng_next_u64(self._h)

    def uniform(self, lo=None, hi=None):
        u = lib().orc_rng_uniform(self._h)
        if lo is None:
            return u
        return lo + (hi - lo) * u  # random.hpp:23

    def normal(self):
        return lib().orc_rng_normal(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_rng_free(self._h)
            self._h = None


# --------------------------------------------------------------------------------------------
# (D) map pruning (prune_oracle.c)
# --------------------------------------------------------------------------------------------

def prune_inputs(scene):
    """fp64 copies of the map's fp32 values, as the GPU sees them: pos [N][3], feat [d][N]."""
    pos = np.ascontiguousarray(np.asarray(scene["pos"], np.float32), dtype=np.float64)
    feat = np.ascontiguousarray(np.asarray(scene["feat"], np.float32), dtype=np.float64)
    return pos, feat


def find_language_redundant(scene, k=8, tau_dist=0.02, tau_sim=0.9) -> np.ndarray:
    """uint8 flags of the SPEC's greedy Eq. 4 sweep (prune_oracle.c)."""
    pos, feat = prune_inputs(scene)
    n, d = pos.shape[0], feat.shape[0]
    flags = np.zeros(max(n, 1), np.uint8)
    r = lib().orc_find_language_redundant(n, d, _ptr(pos, _dp), _ptr(feat, _dp), int(k), float(tau_dist),
                                          float(tau_sim), _ptr(flags, _u8p))
    if r < 0:
        raise MemoryError("orc_find_language_redundant")
    return flags[:n]


def find_geometric(scene, alpha_min=0.05, scale_max=0.5) -> np.ndarray:
    op = np.ascontiguousarray(np.asarray(scene["opac"], np.float32), dtype=np.float64)
    ls = np.ascontiguousarray(np.asarray(scene["log_s"], np.float32), dtype=np.float64)
    flags = np.zeros(max(op.shape[0], 1), np.uint8)
    lib().orc_find_geometric(op.shape[0], _ptr(op, _dp), _ptr(ls, _dp), float(alpha_min), float(scale_max),
                             _ptr(flags, _u8p))
    return flags[:op.shape[0]]
