"""Host-side mirror of the reference renderer interface over the C ABI.

Reference (proj/include/legoslam/renderer.hpp):
    RenderConfig                                   -> RenderConfig
    RenderOutput render(map, cam_pose, K, cfg)     -> render(map, camera, cfg) -> RenderOutput
    MapGradients render_backward(map, out, grad_rgb, grad_depth, grad_feat)
                                                   -> render_backward(map, out, grad_rgb, grad_depth, grad_feat)
    project_gaussian(map, i, cam_pose, K, cfg)     -> RenderOutput.projected() (all i at once)

Same argument meaning and error behaviour: an empty / None cotangent is zero, a cotangent of the
wrong shape raises ValueError (the reference's std::invalid_argument, renderer.cpp:176-178),
gradients are dense over the map (zeros for culled Gaussians) with rotations ordered (w,x,y,z)
and features [d][N].  Every call goes through liblgs.so on the GPU; there is no CPU fallback.

Maps are scene dicts in the reference layouts (see scenes.py) holding either numpy arrays (host
memory: copied in/out by the library, like the reference API) or CUDA torch tensors (device
memory, zero-copy), or a DeviceMap already resident in HBM.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import LGS_MEM_DEVICE, LGS_MEM_HOST, LGS_MEM_HOST_MAPPED, check

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


@dataclass
class RenderConfig:
    """renderer.hpp:15-22."""
    near_plane: float = 0.01
    dilation: float = 0.3
    alpha_clamp: float = 0.99
    alpha_skip: float = 1.0 / 255.0
    transmittance_min: float = 1e-4
    radius_sigma: float = 3.0

    def c(self):
        return _lib.LgsRenderConfig(self.near_plane, self.dilation, self.alpha_clamp, self.alpha_skip,
                                    self.transmittance_min, self.radius_sigma)


def _is_torch(x):
    return torch is not None and isinstance(x, torch.Tensor)


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        assert x.is_contiguous()
        return x.data_ptr()
    assert isinstance(x, np.ndarray) and x.flags.c_contiguous and x.dtype == np.float32, (type(x), getattr(x, "dtype", None))
    return x.ctypes.data


def _mem(x):
    if _is_torch(x):
        return LGS_MEM_DEVICE if x.is_cuda else LGS_MEM_HOST
    return LGS_MEM_HOST


def _f32(x):
    if _is_torch(x):
        return x.contiguous().float() if x.dtype != torch.float32 or not x.is_contiguous() else x
    return np.ascontiguousarray(x, dtype=np.float32)


def make_camera(cam) -> _lib.LgsCamera:
    c = _lib.LgsCamera()
    for i in range(4):
        c.q[i] = float(cam["q"][i])
    for i in range(3):
        c.t[i] = float(cam["t"][i])
    c.fx, c.fy, c.cx, c.cy = (float(cam[k]) for k in ("fx", "fy", "cx", "cy"))
    c.width, c.height = int(cam["width"]), int(cam["height"])
    return c


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


class Context:
    """One CUDA stream + stream-ordered memory pool (lgs_ctx).  By default the library enqueues on
    torch's current stream so torch tensors and library calls stay ordered; ``stream="own"`` gives
    the context a private non-blocking stream (independent host threads rendering concurrently,
    the reference's "concurrent renders between map mutations" contract)."""

    def __init__(self, device: int = 0, stream=None, full_lists: bool = False, radix_depth_order: bool = False,
                 fused_eager: bool = False, host_grad_delta: bool = False, speculative_plans: bool = True):
        L = _lib.load()
        if stream == "own":
            stream = None
        elif stream is None and torch is not None and torch.cuda.is_available():
            with torch.cuda.device(device):
                stream = torch.cuda.current_stream(device).cuda_stream
            if stream == 0:
                stream = CUDA_STREAM_LEGACY  # torch's default stream is the legacy NULL stream
        h = C.c_void_p()
        check(L.lgs_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(h)))
        self.h = h
        self.device = device
        if full_lists:  # complete (tile, Gaussian) lists instead of the depth-layered binning
            check(L.lgs_ctx_set_full_tile_lists(h, 1))
        # context options of include/lgs.h (LGS_OPT_*): cross-check depth order, profiling-only fusion
        if radix_depth_order:
            check(L.lgs_ctx_set_option(h, _lib.LGS_OPT_RADIX_DEPTH_ORDER, 1))
        if fused_eager:
            check(L.lgs_ctx_set_option(h, _lib.LGS_OPT_FUSED_EAGER, 1))
        if host_grad_delta:  # host gradient buffers reused unchanged: row-sparse rewrites (include/lgs.h)
            check(L.lgs_ctx_set_option(h, _lib.LGS_OPT_HOST_GRAD_DELTA, 1))
        if not speculative_plans:  # plans always capture the layered binning's second pass
            check(L.lgs_ctx_set_option(h, _lib.LGS_OPT_SPECULATIVE_PLANS, 0))

    def synchronize(self):
        check(_lib.load().lgs_ctx_synchronize(self.h))

    def transfer_bytes(self):
        """(host->device, device->host) bytes this context has copied since creation."""
        a, b = C.c_int64(), C.c_int64()
        check(_lib.load().lgs_ctx_transfer_bytes(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    @property
    def layer_div(self) -> int:
        """Layer-A size policy of the depth-layered binning (lgs_ctx_layer_div; diagnostics)."""
        return int(_lib.load().lgs_ctx_layer_div(self.h))

    @property
    def launches(self) -> int:
        return int(_lib.load().lgs_ctx_launch_count(self.h))

    def profile(self, enable: bool = True):
        check(_lib.load().lgs_ctx_profile(self.h, 1 if enable else 0))

    def phase_times(self, reset: bool = True) -> dict:
        """{phase name: (device ms accumulated, launches)} from the CUDA events around each phase."""
        L = _lib.load()
        ms = (C.c_double * _lib.LGS_PHASE_COUNT)()
        cnt = (C.c_int64 * _lib.LGS_PHASE_COUNT)()
        check(L.lgs_ctx_phase_times(self.h, ms, cnt, 1 if reset else 0))
        return {L.lgs_phase_name(i).decode(): (ms[i], cnt[i]) for i in range(_lib.LGS_PHASE_COUNT)}

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib._lib is not None:
                _lib._lib.lgs_ctx_destroy(self.h)
                self.h = None
        except (AttributeError, TypeError):  # interpreter shutdown
            pass


_default_ctx: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def _gaussians_struct(scene, host_mapped=False):
    arrs = {k: _f32(scene[k]) for k in ("pos", "rot", "log_s", "opac", "sh", "feat")}
    n = int(arrs["pos"].shape[0])
    d = int(arrs["feat"].shape[0]) if arrs["feat"].ndim == 2 else 0
    K = int(arrs["sh"].shape[1])
    deg = {1: 0, 4: 1, 9: 2, 16: 3}[K]
    mem = _mem(arrs["pos"])
    if host_mapped:
        assert mem == LGS_MEM_HOST, "host_mapped needs a host (page-locked) scene"
        mem = LGS_MEM_HOST_MAPPED
    g = _lib.LgsGaussians(n, d, deg, _ptr(arrs["pos"]), _ptr(arrs["rot"]), _ptr(arrs["log_s"]), _ptr(arrs["opac"]),
                          _ptr(arrs["sh"]), _ptr(arrs["feat"]) if d else None, mem)
    return g, arrs


class DeviceMap:
    """A Gaussian map resident in HBM in the kernels' packed layout (lgs_map)."""

    def __init__(self, scene, ctx: Context | None = None, host_mapped: bool = False):
        """``host_mapped``: the scene is page-locked host memory that the device reads in place
        (LGS_MEM_HOST_MAPPED: SH rows and features of just the listed Gaussians cross PCIe); the
        arrays must stay unchanged while this map and its renders are alive (they are referenced)."""
        self.ctx = ctx or default_context()
        self.host_mapped = host_mapped
        g, self._arrs = _gaussians_struct(scene, host_mapped)
        self.n, self.d, self.sh_degree = g.n, g.feature_dim, g.sh_degree
        self.K = (self.sh_degree + 1) ** 2
        h = C.c_void_p()
        check(_lib.load().lgs_map_create(self.ctx.h, C.byref(g), C.byref(h)))
        self.h = h
        if not host_mapped:
            self._arrs = None  # the library copied (host) or packed (device) the attributes

    def update(self, scene):
        g, keep = _gaussians_struct(scene)
        check(_lib.load().lgs_map_update(self.ctx.h, self.h, C.byref(g)))
        del keep

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib._lib is not None:
                _lib._lib.lgs_map_destroy(self.h)
                self.h = None
        except (AttributeError, TypeError):  # interpreter shutdown
            pass


class RenderOutput:
    """renderer.hpp:33-45: images + the backward tape (lgs_saved)."""

    def __init__(self, ctx, tape, rgb, depth, feat, acc, n, d, K, cam, dmap):
        self.ctx, self.tape = ctx, tape
        self.rgb, self.depth, self.feat, self.acc = rgb, depth, feat, acc
        self.n, self.d, self.K = n, d, K
        self.camera = cam
        self._map = dmap  # keeps the device map alive for the backward

    def stats(self):
        s = _lib.LgsRenderStats()
        check(_lib.load().lgs_saved_stats(self.tape, C.byref(s)))
        return dict(visible=s.visible, pairs=s.pairs, tiles=s.tiles, max_tile_list=s.max_tile_list, listed=s.listed,
                    active=s.active, host_rows=s.host_rows)

    def work(self):
        """(evaluated (pixel, Gaussian) pairs, contributing pairs) of this forward."""
        e, c = C.c_int64(), C.c_int64()
        check(_lib.load().lgs_saved_work(self.tape, C.byref(e), C.byref(c)))
        return e.value, c.value

    def l1_loss(self) -> float:
        v = C.c_double()
        check(_lib.load().lgs_saved_l1_loss(self.ctx.h, self.tape, C.byref(v)))
        return v.value

    def projected(self):
        """Per map index fp32 projected records (the batched project_gaussian, renderer.cpp:53-92)."""
        n = self.n
        r = dict(visible=np.zeros(n, np.uint8), u=np.zeros(n, np.float32), v=np.zeros(n, np.float32),
                 depth=np.zeros(n, np.float32), conic=np.zeros((n, 3), np.float32), radius=np.zeros(n, np.float32),
                 bbox=np.zeros((n, 4), np.int32), opacity=np.zeros(n, np.float32), color=np.zeros((n, 3), np.float32))
        check(_lib.load().lgs_debug_projected(self.ctx.h, self.tape, *(r[k].ctypes.data for k in (
            "visible", "u", "v", "depth", "conic", "radius", "bbox", "opacity", "color"))))
        return r

    def tile_keys(self):
        """(keys u64 = tile << 32 | f32bits(depth), vals u32 map index, ranges [tiles, 2])."""
        st = self.stats()
        keys = np.zeros(max(st["listed"], 1), np.uint64)
        vals = np.zeros(max(st["listed"], 1), np.uint32)
        ranges = np.zeros((st["tiles"], 2), np.uint32)
        check(_lib.load().lgs_debug_tile_keys(self.ctx.h, self.tape, keys.ctypes.data, vals.ctypes.data,
                                              ranges.ctypes.data))
        return keys[:st["listed"]], vals[:st["listed"]], ranges

    def pixel_state(self):
        H, W = self.camera.height, self.camera.width
        ft = np.zeros((H, W), np.float32)
        nc = np.zeros((H, W), np.uint32)
        check(_lib.load().lgs_debug_pixel_state(self.ctx.h, self.tape, ft.ctypes.data, nc.ctypes.data))
        return ft, nc

    def cotangents(self):
        """(g_rgb [H,W,3], g_depth [H,W], g_feat [H,W,d]) held by the tape (fused L1 / mapping loss)."""
        H, W = self.camera.height, self.camera.width
        r = np.zeros((H, W, 3), np.float32)
        dd = np.zeros((H, W), np.float32)
        f = np.zeros((H, W, self.d), np.float32)
        check(_lib.load().lgs_debug_cotangents(self.ctx.h, self.tape, r.ctypes.data, dd.ctypes.data,
                                               f.ctypes.data if self.d else None))
        return r, dd, f

    def __del__(self):
        try:
            if getattr(self, "tape", None) and _lib._lib is not None:
                _lib._lib.lgs_saved_destroy(self.tape)
                self.tape = None
        except (AttributeError, TypeError):  # interpreter shutdown
            pass


def _alloc_like(device_side, shape, device):
    if device_side:
        return torch.empty(shape, dtype=torch.float32, device=f"cuda:{device}")
    return np.empty(shape, np.float32)


def render(map_, camera, cfg: RenderConfig | None = None, targets=None, ctx: Context | None = None,
           out: dict | None = None, host_mapped: bool = False) -> RenderOutput:
    """lego::render (renderer.hpp:55-56).  ``map_``: DeviceMap or scene dict (numpy / CUDA tensors).
    ``host_mapped``: a host scene in page-locked memory is read in place where few rows are
    needed (DeviceMap(host_mapped=True)) instead of being copied whole.

    ``targets`` (optional dict rgb/depth/feat) fuses the L1 loss of SURVEY.md §8d into the forward.
    Output images are CUDA tensors when the map is device-resident, numpy otherwise (or ``out``).
    """
    ctx = ctx or (map_.ctx if isinstance(map_, DeviceMap) else default_context())
    dmap = map_ if isinstance(map_, DeviceMap) else None
    host_scene = False
    if dmap is None:
        host_scene = _mem(map_["pos"]) == LGS_MEM_HOST
        dmap = DeviceMap(map_, ctx, host_mapped=host_mapped and host_scene)
    cam = make_camera(camera)
    H, W, d = cam.height, cam.width, dmap.d
    if out is None:
        dev = not host_scene
        out = dict(rgb=_alloc_like(dev, (H, W, 3), ctx.device), depth=_alloc_like(dev, (H, W), ctx.device),
                   feat=_alloc_like(dev, (H, W, d), ctx.device), acc=_alloc_like(dev, (H, W), ctx.device))
    imgs = _lib.LgsImages(_ptr(out["rgb"]), _ptr(out["depth"]), _ptr(out["feat"]) if d else None, _ptr(out["acc"]),
                          _mem(out["rgb"]))
    tg = None
    keep = None
    if targets is not None:
        keep = {k: _f32(targets[k]) for k in ("rgb", "depth", "feat")}
        tg = _lib.LgsL1Targets(_ptr(keep["rgb"]), _ptr(keep["depth"]), _ptr(keep["feat"]) if d else None,
                               _mem(keep["rgb"]))
    c = (cfg or RenderConfig()).c()
    tape = C.c_void_p()
    check(_lib.load().lgs_render_forward(ctx.h, dmap.h, C.byref(cam), C.byref(c), C.byref(tg) if tg else None,
                                         C.byref(imgs), C.byref(tape)))
    del keep
    return RenderOutput(ctx, tape, out["rgb"], out["depth"], out["feat"], out["acc"], dmap.n, d, dmap.K, cam, dmap)


def alloc_grads(n, d, K, device=None, flat=None):
    """MapGradients (renderer.hpp:59-68) as views into one flat fp32 buffer (NCCL-friendly):
    position [N,3] | rotation [N,4] (w,x,y,z) | log_scale [N,3] | opacity_logit [N] | sh [N,K,3] | feature [d,N]."""
    sizes = [("position", (n, 3)), ("rotation", (n, 4)), ("log_scale", (n, 3)), ("opacity_logit", (n,)),
             ("sh", (n, K, 3)), ("feature", (d, n))]
    total = sum(int(np.prod(s)) for _, s in sizes)
    if flat is None:
        flat = (torch.zeros(total, dtype=torch.float32, device=f"cuda:{device}") if device is not None
                else np.zeros(total, np.float32))
    out, o = {"flat": flat}, 0
    for name, s in sizes:
        k = int(np.prod(s))
        out[name] = flat[o:o + k].reshape(s)
        o += k
    return out


def _size(x):
    return x.numel() if _is_torch(x) else x.size


def _grads_struct(g, accumulate):
    ptrs = [_ptr(g[k]) if _size(g[k]) else None
            for k in ("position", "rotation", "log_scale", "opacity_logit", "sh", "feature")]
    return _lib.LgsMapGrads(*ptrs, _mem(g["position"]), 1 if accumulate else 0)


def _check_cot(x, shape, name):
    if x is None:
        return None
    if (x.numel() if _is_torch(x) else x.size) == 0:
        return None  # empty image = zero cotangent (renderer.hpp:70-71)
    s = tuple(x.shape)
    if len(s) == 2:
        s = s + (1,)
    if s != shape:
        raise ValueError(f"render_backward: bad shape for {name}")  # renderer.cpp:176-178
    return _f32(x)


def render_backward(map_, out: RenderOutput, grad_rgb=None, grad_depth=None, grad_feat=None, pose: bool = False,
                    into: dict | None = None, accumulate: bool = False):
    """lego::render_backward (renderer.hpp:72-74).  ``map_`` is accepted for signature parity (the
    tape references the map it was rendered from, which must be unchanged -- SPEC.md:278).

    Returns the MapGradients dict (+ ``pose`` [6] = dL/d(omega, nu) when ``pose``)."""
    H, W, d = out.camera.height, out.camera.width, out.d
    cr = _check_cot(grad_rgb, (H, W, 3), "grad_rgb")
    cd = _check_cot(grad_depth, (H, W, 1), "grad_depth")
    cf = _check_cot(grad_feat, (H, W, d), "grad_feat") if d else None
    mems = {_mem(x) for x in (cr, cd, cf) if x is not None}
    if len(mems) > 1:
        raise ValueError("cotangents must all be host or all be device memory")
    cot = _lib.LgsCotangents(_ptr(cr), _ptr(cd), _ptr(cf), mems.pop() if mems else LGS_MEM_DEVICE)
    dev = _is_torch(out.rgb) and out.rgb.is_cuda
    g = into or alloc_grads(out.n, d, out.K, device=out.ctx.device if dev else None)
    gs = _grads_struct(g, accumulate)
    pg = (C.c_float * 6)() if pose else None
    check(_lib.load().lgs_render_backward(out.ctx.h, out.tape, C.byref(cot), C.byref(gs), pg))
    del cr, cd, cf
    if pose:
        g["pose"] = np.array(list(pg), dtype=np.float64)
    return g


def render_backward_l1(out: RenderOutput, pose: bool = False, into: dict | None = None, accumulate: bool = False):
    """Backward of the L1 loss fused into ``render(..., targets=...)``."""
    dev = _is_torch(out.rgb) and out.rgb.is_cuda
    g = into or alloc_grads(out.n, out.d, out.K, device=out.ctx.device if dev else None)
    gs = _grads_struct(g, accumulate)
    pg = (C.c_float * 6)() if pose else None
    check(_lib.load().lgs_render_backward_l1(out.ctx.h, out.tape, C.byref(gs), pg))
    if pose:
        g["pose"] = np.array(list(pg), dtype=np.float64)
    return g


def mapping_loss(out: RenderOutput, keyframe: dict, decoder=None, w_l1: float = 0.8, w_depth: float = 0.5,
                 w_feat: float = 1.0, readback: bool = True):
    """SPEC.md:418-426 compute_losses on the GPU (lgs_mapping_loss): stores d l_total / d images in
    the tape for render_backward_loss and returns the LossBreakdown (or None without readback).

    ``keyframe``: rgb [H,W,3], depth [H,W] (<= 0 / non-finite = invalid), feat_gt [H,W,D];
    ``decoder``: (w1 [hidden,d], b1 [hidden], w2 [D,hidden], b2 [D]) -- the frozen codec decoder."""
    H, W, d = out.camera.height, out.camera.width, out.d
    keep = {k: _f32(keyframe[k]) for k in ("rgb", "depth") if keyframe.get(k) is not None}
    kmem = _mem(keep["rgb"])
    if d:
        keep["feat_gt"] = _f32(keyframe["feat_gt"])
        w1, b1, w2, b2 = (_f32(x) for x in decoder)
        keep.update(w1=w1, b1=b1, w2=w2, b2=b2)
        dec = _lib.LgsDecoder(int(w2.shape[0]), int(w1.shape[0]), int(w1.shape[1]), _ptr(w1), _ptr(b1), _ptr(w2),
                              _ptr(b2), _mem(w1))
    kf = _lib.LgsKeyframe(_ptr(keep["rgb"]), _ptr(keep["depth"]), _ptr(keep.get("feat_gt")), kmem)
    rendered = _lib.LgsImages(_ptr(out.rgb), None, _ptr(out.feat) if d else None, None, _mem(out.rgb))
    w = _lib.LgsLossWeights(w_l1, w_depth, w_feat)
    br = _lib.LgsLossBreakdown() if readback else None
    check(_lib.load().lgs_mapping_loss(out.ctx.h, out.tape, C.byref(rendered), C.byref(kf),
                                       C.byref(dec) if d else None, C.byref(w), C.byref(br) if br else None))
    del keep
    if br is None:
        return None
    return dict(l_rgb=br.l_rgb, l_depth=br.l_depth, l_feat=br.l_feat, l_total=br.l_total, ssim=br.ssim,
                depth_pixels=br.depth_pixels)


def render_backward_loss_async(out: RenderOutput, into: dict, pose_out=None, accumulate: bool = False):
    """Asynchronous backward of the tape's loss (device gradients); ``pose_out`` (a CUDA tensor or a
    pinned host tensor of 6 float32) receives dL/d(omega, nu) in stream order -- no host wait."""
    gs = _grads_struct(into, accumulate)
    check(_lib.load().lgs_render_backward_loss_async(out.ctx.h, out.tape, C.byref(gs),
                                                     pose_out.data_ptr() if pose_out is not None else None))
    return into


def render_backward_loss(out: RenderOutput, pose: bool = False, into: dict | None = None, accumulate: bool = False):
    """Backward of the loss whose cotangents the tape holds (fused L1 or mapping_loss)."""
    dev = _is_torch(out.rgb) and out.rgb.is_cuda
    g = into or alloc_grads(out.n, out.d, out.K, device=out.ctx.device if dev else None)
    gs = _grads_struct(g, accumulate)
    pg = (C.c_float * 6)() if pose else None
    check(_lib.load().lgs_render_backward_loss(out.ctx.h, out.tape, C.byref(gs), pg))
    if pose:
        g["pose"] = np.array(list(pg), dtype=np.float64)
    return g


def map_download(dmap: DeviceMap, device: bool = False) -> dict:
    """The resident map in the reference layouts (pos, rot x,y,z,w, log_s, opac, sh, feat [d,N])."""
    n, d, K = dmap.n, dmap.d, dmap.K
    shapes = {"pos": (n, 3), "rot": (n, 4), "log_s": (n, 3), "opac": (n,), "sh": (n, K, 3), "feat": (d, n)}
    out = {k: _alloc_like(device, s, dmap.ctx.device) for k, s in shapes.items()}
    g = _lib.LgsGaussians(n, d, dmap.sh_degree, _ptr(out["pos"]), _ptr(out["rot"]), _ptr(out["log_s"]),
                          _ptr(out["opac"]), _ptr(out["sh"]), _ptr(out["feat"]) if d else None,
                          LGS_MEM_DEVICE if device else LGS_MEM_HOST)
    check(_lib.load().lgs_map_download(dmap.ctx.h, dmap.h, C.byref(g)))
    return out


class Adam:
    """Per-attribute Adam on a resident map (lgs_adam_*; SPEC.md:430 learning rates)."""

    def __init__(self, dmap: DeviceMap, **cfg):
        L = _lib.load()
        c = L.lgs_adam_config_default()
        for k, v in cfg.items():
            if not hasattr(c, k):
                raise TypeError(f"unknown Adam option {k}")
            setattr(c, k, float(v))
        self.config = {k: getattr(c, k) for k, _ in _lib.LgsAdamConfig._fields_}
        h = C.c_void_p()
        check(L.lgs_adam_create(dmap.ctx.h, dmap.h, C.byref(c), C.byref(h)))
        self.h, self.map = h, dmap

    @property
    def steps(self) -> int:
        return int(_lib.load().lgs_adam_steps(self.h))

    def step(self, grads: dict):
        gs = _grads_struct(grads, False)
        check(_lib.load().lgs_adam_step(self.map.ctx.h, self.h, self.map.h, C.byref(gs)))

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib._lib is not None:
                _lib._lib.lgs_adam_destroy(self.h)
                self.h = None
        except (AttributeError, TypeError):  # interpreter shutdown
            pass


def map_file_info(path: str):
    """(feature_dim, count) of a LEGOMAP1 file (gaussian_map.cpp:220-237 header)."""
    d, n = C.c_int32(), C.c_int64()
    check(_lib.load().lgs_map_file_info(str(path).encode(), C.byref(d), C.byref(n)))
    return d.value, n.value


def map_file_read(path: str, expected_dim: int = 0):
    """lego::deserialize_map (gaussian_map.cpp:220-259) -> (scene dict in the reference layouts,
    anchors u64 [N]).  Raises LgsIoError (an OSError) like the reference's IoError."""
    d, n = map_file_info(path)
    scene = {"pos": np.zeros((n, 3), np.float32), "rot": np.zeros((n, 4), np.float32),
             "log_s": np.zeros((n, 3), np.float32), "opac": np.zeros(n, np.float32),
             "sh": np.zeros((n, 1, 3), np.float32), "feat": np.zeros((d, n), np.float32)}
    anchors = np.zeros(n, np.uint64)
    g = _lib.LgsGaussians(n, d, 0, *(scene[k].ctypes.data for k in ("pos", "rot", "log_s", "opac", "sh", "feat")),
                          LGS_MEM_HOST)
    check(_lib.load().lgs_map_file_read(str(path).encode(), int(expected_dim), C.byref(g), anchors.ctypes.data))
    return scene, anchors


def map_file_write(path: str, scene, anchors=None):
    """lego::serialize_map (gaussian_map.cpp:196-218) from a scene dict (SH degree 0)."""
    g, keep = _gaussians_struct(scene)
    a = None if anchors is None else np.ascontiguousarray(anchors, np.uint64)
    check(_lib.load().lgs_map_file_write(str(path).encode(), C.byref(g), a.ctypes.data if a is not None else None))
    del keep


def map_load(path: str, ctx: Context | None = None, expected_dim: int = 0) -> DeviceMap:
    """LEGOMAP1 file -> resident device map (lgs_map_load)."""
    ctx = ctx or default_context()
    dm = DeviceMap.__new__(DeviceMap)
    h = C.c_void_p()
    check(_lib.load().lgs_map_load(ctx.h, str(path).encode(), int(expected_dim), C.byref(h)))
    dm.ctx, dm.h, dm._arrs = ctx, h, None
    dm.d, dm.n = map_file_info(path)
    dm.sh_degree, dm.K = 0, 1
    return dm


def map_save(dmap: DeviceMap, path: str, anchors=None):
    a = None if anchors is None else np.ascontiguousarray(anchors, np.uint64)
    check(_lib.load().lgs_map_save(dmap.ctx.h, dmap.h, str(path).encode(), a.ctypes.data if a is not None else None))


def coverage_mask(out: RenderOutput, measured_depth):
    """SPEC.md:225 insertion coverage mask on the GPU: (uint8 mask [H, W], selected count).  The
    mask is a CUDA tensor for device depth input, numpy otherwise."""
    H, W = out.camera.height, out.camera.width
    md = _f32(measured_depth)
    if tuple(md.shape) != (H, W):
        raise ValueError("coverage_mask: measured depth must be [H, W]")
    dev = _is_torch(md) and md.is_cuda
    mask = torch.empty((H, W), dtype=torch.uint8, device=md.device) if dev else np.empty((H, W), np.uint8)
    cnt = C.c_int64()
    check(_lib.load().lgs_coverage_mask(out.ctx.h, out.tape, _ptr(md), _mem(md), _ptr_any(mask), _mem(mask),
                                        C.byref(cnt)))
    return mask, cnt.value


def _ptr_any(x):
    return x.data_ptr() if _is_torch(x) else x.ctypes.data


class Plan:
    """One fused-L1 forward + backward step captured into a CUDA graph (lgs_plan_*): ``run()``
    enqueues the whole step with one graph launch; ``sync()`` waits for it (re-capturing if the
    tile lists outgrew their capacity).  ``targets``, ``grads`` and the optional ``images`` are CUDA
    buffers whose contents may change between runs; ``pose_out`` (pinned host or CUDA, 6 float32)
    receives the pose gradient in stream order.  ``accumulate``: the step adds its gradients into
    ``grads`` (the later views of a multi-view batch) instead of overwriting them."""

    def __init__(self, dmap: DeviceMap, camera, targets: dict, grads: dict, images: dict | None = None,
                 pose_out=None, cfg: RenderConfig | None = None, accumulate: bool = False):
        self.ctx = dmap.ctx
        self._keep = (targets, grads, images, pose_out)
        cam = make_camera(camera)
        d = dmap.d
        tg = _lib.LgsL1Targets(_ptr(targets["rgb"]), _ptr(targets["depth"]), _ptr(targets["feat"]) if d else None,
                               LGS_MEM_DEVICE)
        imgs = None
        if images is not None:
            imgs = _lib.LgsImages(_ptr(images["rgb"]), _ptr(images["depth"]), _ptr(images["feat"]) if d else None,
                                  _ptr(images["acc"]), LGS_MEM_DEVICE)
        gs = _grads_struct(grads, accumulate)  # accumulate: add into grads (later views of a batch)
        c = (cfg or RenderConfig()).c()
        h = C.c_void_p()
        check(_lib.load().lgs_plan_create(self.ctx.h, dmap.h, C.byref(cam), C.byref(c), C.byref(tg),
                                          C.byref(imgs) if imgs is not None else None, C.byref(gs),
                                          pose_out.data_ptr() if pose_out is not None else None, C.byref(h)))
        self.h = h

    def run(self):
        check(_lib.load().lgs_plan_run(self.ctx.h, self.h))

    def sync(self) -> int:
        p = C.c_int64()
        check(_lib.load().lgs_plan_sync(self.ctx.h, self.h, C.byref(p)))
        return p.value

    def set_camera(self, camera):
        cam = make_camera(camera)
        check(_lib.load().lgs_plan_set_camera(self.ctx.h, self.h, C.byref(cam)))

    def set_profiling(self, on: bool = True):
        """Re-capture with per-phase event nodes (costs a few us per phase per replay)."""
        check(_lib.load().lgs_plan_set_profiling(self.ctx.h, self.h, 1 if on else 0))

    def phase_times(self) -> dict:
        """Device ms per phase of the last replay (events recorded inside the graph)."""
        L = _lib.load()
        ms = (C.c_double * _lib.LGS_PHASE_COUNT)()
        check(L.lgs_plan_phase_times(self.h, ms))
        return {L.lgs_phase_name(i).decode(): ms[i] for i in range(_lib.LGS_PHASE_COUNT) if ms[i] > 0.0}

    def elapsed_ms(self) -> float:
        v = C.c_float()
        check(_lib.load().lgs_plan_elapsed_ms(self.h, C.byref(v)))
        return v.value

    @property
    def launches(self) -> int:
        return int(_lib.load().lgs_plan_launches(self.h))

    @property
    def recaptures(self) -> int:
        """How often sync() re-captured and re-ran the step (the tile lists outgrew the capacity)."""
        return int(_lib.load().lgs_plan_recaptures(self.h))

    @property
    def speculative(self) -> bool:
        """Captured without the layered binning's second pass (every warm-up tile saturated on
        its first-pass list); a replay that leaves a tile unsaturated is re-run by sync()."""
        return bool(_lib.load().lgs_plan_speculative(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib._lib is not None:
                _lib._lib.lgs_plan_destroy(self.h)
                self.h = None
        except (AttributeError, TypeError):  # interpreter shutdown
            pass


def sync_plans(plans):
    """Wait for a batch of plans sharing one gradient buffer (the first writes, the others
    accumulate) and finish it exactly: lgs_plan_sync re-runs a replay that outgrew its tile lists
    or missed its speculation, having added nothing; when that is the FIRST plan, its re-run
    rewrites the buffer, so the accumulating plans that already added are run again.  Returns the
    pair counts."""
    before = [p.recaptures for p in plans]
    pairs = [p.sync() for p in plans]
    if plans and plans[0].recaptures != before[0]:
        redo = [p for p, b in zip(plans[1:], before[1:]) if p.recaptures == b]
        for p in redo:
            p.run()
        for p in redo:
            p.sync()
    return pairs
