"""Shared comparison helpers for the GPU parity tests (tolerances are written here, once).

Images: |gpu - ref| <= 1e-5 + 1e-4 |ref| elementwise (BASELINE north star: 1e-4 relative /
1e-5 absolute).  The reference compositor is fp64 while the kernels are fp32, so a threshold test
(alpha >= 1/255, T >= 1e-4, opacity*G > 0.99) can flip when the two sides land within fp32
rounding of the threshold; such pixels are reported and must stay a tiny fraction
(``max_flip_frac``).

Gradients: |gpu - ref| <= 1e-3 (|ref| + floor_g) per component, where floor_g is 1e-2 x the RMS of
that attribute group in the reference -- the reference's own gradcheck uses the same kind of
absolute floor (rel_err in gradcheck.hpp:101-103, floor 1e-2), which keeps components that are
pure cancellation noise from dominating.  Atomic accumulation order differs from the reference's
sequential order, hence the 1e-3 (north star).
"""
import numpy as np

IMG_RTOL = 1e-4
IMG_ATOL = 1e-5
GRAD_RTOL = 1e-3
GRAD_FLOOR = 1e-2


def to_np(x):
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().cpu().numpy()
    except ImportError:
        pass
    return np.asarray(x)


def image_mismatch(gpu, ref, rtol=IMG_RTOL, atol=IMG_ATOL):
    """Fraction of pixels (any channel) outside tolerance, and the max abs error."""
    g = to_np(gpu).astype(np.float64)
    r = to_np(ref).astype(np.float64)
    bad = np.abs(g - r) > atol + rtol * np.abs(r)
    if bad.ndim == 3:
        bad = bad.any(axis=2)
    return float(bad.mean()) if bad.size else 0.0, float(np.abs(g - r).max()) if g.size else 0.0


def grad_mismatch(gpu, ref, rtol=GRAD_RTOL, floor=GRAD_FLOOR):
    """Fraction of components outside tolerance and the worst normalized error."""
    g = to_np(gpu).astype(np.float64).ravel()
    r = to_np(ref).astype(np.float64).ravel()
    if r.size == 0:
        return 0.0, 0.0
    rms = float(np.sqrt(np.mean(r * r)))
    den = np.abs(r) + floor * rms + 1e-30
    e = np.abs(g - r) / den
    return float((e > rtol).mean()), float(e.max())


GROUPS = ("position", "rotation", "log_scale", "opacity_logit", "sh", "feature")


# ---- explained mismatches (the large-scale parity tests) -------------------------------------------
#
# At scale a blanket "fraction outside tolerance" hides what the outliers are.  Oracle A, run on the
# GPU's own fp32 projected records, also runs an fp32 twin of the kernel's per-pair arithmetic
# (lgs_oracle.c, orc_render.pix_flag) and flags every pixel where an alpha-skip, transmittance or
# clamp decision differs between fp64 and fp32 (or sits inside fp32 rounding of its threshold),
# and every Gaussian that took part in such a decision or contributes at such a pixel.  Every element
# outside tolerance must be one of those: the count of flagged ("explained") outliers is reported and
# the count of unexplained ones must be zero.

def explain_image(gpu, ref, pix_flag, rtol=IMG_RTOL, atol=IMG_ATOL):
    """Pixels (any channel) outside |gpu - ref| <= atol + rtol |ref|, split by the fp32-twin flags."""
    g = to_np(gpu).astype(np.float64)
    r = to_np(ref).astype(np.float64)
    err = np.abs(g - r)
    bad = err > atol + rtol * np.abs(r)
    if bad.ndim == 3:
        bad = bad.any(axis=2)
        err = err.max(axis=2)
    flagged = (pix_flag & 3) != 0
    unexpl = bad & ~flagged
    return dict(outside=int(bad.sum()), explained=int((bad & flagged).sum()), unexplained=int(unexpl.sum()),
                max_err=float(err.max()) if err.size else 0.0,
                max_err_unflagged=float(err[~flagged].max()) if (~flagged).any() else 0.0)


def explain_grad(gpu, ref, g_flag, rows_last=False, rtol=GRAD_RTOL, floor=GRAD_FLOOR):
    """Components outside |gpu - ref| <= rtol (|ref| + floor rms(ref)), split by the Gaussian flags of
    their rows.  Arrays are [N, ...] or, with rows_last, [..., N] (the [d][N] feature layout)."""
    g = to_np(gpu).astype(np.float64)
    r = to_np(ref).astype(np.float64)
    if rows_last:
        g, r = np.moveaxis(g, -1, 0), np.moveaxis(r, -1, 0)
    g = g.reshape(g.shape[0], -1)
    r = r.reshape(r.shape[0], -1)
    rms = float(np.sqrt(np.mean(r * r))) if r.size else 0.0
    e = np.abs(g - r) / (np.abs(r) + floor * rms + 1e-30)
    bad = e > rtol
    flagged = (to_np(g_flag) != 0)[:, None]
    unexpl = bad & ~flagged
    return dict(outside=int(bad.sum()), explained=int((bad & flagged).sum()), unexplained=int(unexpl.sum()),
                components=int(bad.size), max_err=float(e.max()) if e.size else 0.0,
                max_err_unflagged=float(e[~np.broadcast_to(flagged, e.shape)].max()) if e.size and (~flagged).any()
                else 0.0)


def l1_cotangents_f32(rgb, depth, feat, targets):
    """The fused-L1 kernel's cotangents (blend_fused.cu epilogue) from ITS OWN fp32 images:
    sign(image - target) times the fp32 reciprocal counts 1/(3HW), 1/HW, 1/(dHW)."""
    rgb, depth, feat = (to_np(x).astype(np.float32) for x in (rgb, depth, feat))
    H, W = depth.shape
    npx = np.float32(W) * np.float32(H)
    inv_rgb = np.float32(1.0) / (np.float32(3.0) * npx)
    inv_d = np.float32(1.0) / npx
    d = feat.shape[2]
    inv_f = np.float32(1.0) / (np.float32(d) * npx) if d else np.float32(0)
    s = lambda a, t: np.sign(a - to_np(t).astype(np.float32)).astype(np.float32)  # noqa: E731
    return (s(rgb, targets["rgb"]) * inv_rgb, s(depth, targets["depth"]) * inv_d,
            s(feat, targets["feat"]) * inv_f)
