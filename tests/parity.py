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
