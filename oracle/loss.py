"""TEST INFRASTRUCTURE ONLY -- fp64 numpy restatement of the mapping losses and the decoder chain.

The checker for the CUDA loss kernels (csrc/loss.cu); only tests/ and bench.py's CPU legs use it.

Restates:
* ``ssim`` -- SPEC.md:410-417: SSIM with an 11x11 Gaussian window (sigma 1.5), C1 = 0.01^2,
  C2 = 0.03^2, channel-averaged.  The reference has no implementation (proj/src/metrics.cpp is a
  placeholder); the SPEC's closed form for constant images holds only when every
  window lies inside the image, so the statistics are taken at the 'valid' window positions (the
  original Wang et al. formulation) and averaged over them.
* ``compute_losses`` -- SPEC.md:418-426: l_rgb = w_l1 L1(rgb) + (1 - w_l1) (1 - ssim) / 2
  (w_l1 = 0.8); l_depth = L1 over pixels whose measured depth is valid (finite, > 0)
  and whose rendered acc > 0.5, averaged over those pixels; l_feat = L1(decode(feat), F_gt);
  l_total = l_rgb + w_depth l_depth + w_feat l_feat (defaults 0.5 / 1.0).
  sign(0) = 0 in every L1 cotangent (as Eigen's .sign() in codec.cpp:193).
* ``decode`` / ``decode_backward_input`` -- proj/src/codec.cpp:88-143 (apply_net, :88-103;
  decode, :114-119; decode_backward_input, :121-143): y = W2 relu(W1 z + b1) + b2 per pixel,
  g_z = W1^T ((W1 z + b1 > 0) * (W2^T g_y)).
Returns the loss breakdown and the cotangents (grad_rgb, grad_depth, grad_feat) that
lgs_render_backward consumes.
"""
from __future__ import annotations

import numpy as np

WIN = 11
SIGMA = 1.5
C1 = 0.01 ** 2
C2 = 0.03 ** 2


def gauss_window(size=WIN, sigma=SIGMA):
    x = np.arange(size, dtype=np.float64) - (size - 1) / 2.0
    w = np.exp(-(x * x) / (2.0 * sigma * sigma))
    return w / w.sum()


def _blur_valid(img, w):
    """Separable 'valid' correlation of [H, W] with the 1-D window w (both axes)."""
    k = w.size
    H, W = img.shape
    t = np.zeros((H, W - k + 1))
    for i in range(k):
        t += w[i] * img[:, i:i + W - k + 1]
    o = np.zeros((H - k + 1, W - k + 1))
    for i in range(k):
        o += w[i] * t[i:i + H - k + 1, :]
    return o


def _blur_full_adjoint(m, w, H, W):
    """Adjoint of _blur_valid: scatter a [H-k+1, W-k+1] map back onto [H, W]."""
    k = w.size
    t = np.zeros((H, m.shape[1]))
    for i in range(k):
        t[i:i + m.shape[0], :] += w[i] * m
    o = np.zeros((H, W))
    for i in range(k):
        o[:, i:i + m.shape[1]] += w[i] * t
    return o


def ssim(a, b, with_grad=False):
    """Mean SSIM over channels and valid window positions; optionally d ssim / d a."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.shape != b.shape:
        raise ValueError("ssim: shape mismatch")
    if a.ndim == 2:
        a, b = a[..., None], b[..., None]
    H, W, Cn = a.shape
    if H < WIN or W < WIN:
        raise ValueError("ssim: image smaller than the 11x11 window")
    w = gauss_window()
    total = 0.0
    grad = np.zeros_like(a) if with_grad else None
    npos = (H - WIN + 1) * (W - WIN + 1)
    for c in range(Cn):
        x, y = a[..., c], b[..., c]
        mx, my = _blur_valid(x, w), _blur_valid(y, w)
        exx, eyy, exy = _blur_valid(x * x, w), _blur_valid(y * y, w), _blur_valid(x * y, w)
        sxx, syy, sxy = exx - mx * mx, eyy - my * my, exy - mx * my
        n1, n2 = 2 * mx * my + C1, 2 * sxy + C2
        d1, d2 = mx * mx + my * my + C1, sxx + syy + C2
        s = n1 * n2 / (d1 * d2)
        total += s.sum()
        if with_grad:
            k = 1.0 / (npos * Cn)  # d mean / d s_p
            dA = k * s * (2 * my / n1 - 2 * my / n2 - 2 * mx / d1 + 2 * mx / d2)  # d/d mu_x
            dB = k * s * (-1.0 / d2)                                              # d/d E[x^2]
            dC = k * s * (2.0 / n2)                                               # d/d E[xy]
            grad[..., c] = (_blur_full_adjoint(dA, w, H, W) + 2 * x * _blur_full_adjoint(dB, w, H, W)
                            + y * _blur_full_adjoint(dC, w, H, W))
    val = total / (npos * Cn)
    return (val, grad) if with_grad else val


def decode(z, w1, b1, w2, b2):
    """codec.cpp:88-103 apply_net (via Codec::decode, :114-119) (decoder weights): z [..., d] -> y [..., D]."""
    z = np.asarray(z, np.float64)
    pre = z @ np.asarray(w1, np.float64).T + b1
    return np.maximum(pre, 0.0) @ np.asarray(w2, np.float64).T + b2


def decode_backward_input(z, g_out, w1, b1, w2):
    """codec.cpp:121-143 (ReLU mask of the pre-activation at :136)."""
    z = np.asarray(z, np.float64)
    pre = z @ np.asarray(w1, np.float64).T + b1
    gh = np.asarray(g_out, np.float64) @ np.asarray(w2, np.float64)
    gh = np.where(pre > 0.0, gh, 0.0)
    return gh @ np.asarray(w1, np.float64)


def compute_losses(rgb, depth, feat, acc, kf_rgb, kf_depth, kf_feat, dec, w_depth=0.5, w_feat=1.0, w_l1=0.8):
    """SPEC.md:418-426 compute_losses + the cotangents of l_total w.r.t. the rendered images.

    ``dec`` = (w1 [Hd, d], b1 [Hd], w2 [D, Hd], b2 [D]).  Returns (breakdown dict, g_rgb, g_depth,
    g_feat)."""
    rgb = np.asarray(rgb, np.float64)
    depth = np.asarray(depth, np.float64)
    feat = np.asarray(feat, np.float64)
    acc = np.asarray(acc, np.float64)
    kf_rgb = np.asarray(kf_rgb, np.float64)
    kf_depth = np.asarray(kf_depth, np.float64)
    kf_feat = np.asarray(kf_feat, np.float64)
    H, W, _ = rgb.shape
    if kf_rgb.shape != rgb.shape or kf_depth.shape != depth.shape or kf_feat.shape[:2] != (H, W):
        raise ValueError("compute_losses: shape mismatch")
    w1, b1, w2, b2 = (np.asarray(x, np.float64) for x in dec)

    # rgb: w_l1 L1 + (1 - w_l1) D-SSIM
    diff = rgb - kf_rgb
    l1 = np.abs(diff).mean()
    s, gs = ssim(rgb, kf_rgb, with_grad=True)
    l_rgb = w_l1 * l1 + (1.0 - w_l1) * (1.0 - s) / 2.0
    g_rgb = w_l1 * np.sign(diff) / diff.size - (1.0 - w_l1) / 2.0 * gs

    # depth: masked L1 (valid measurement and acc > 0.5), mean over the mask
    valid = np.isfinite(kf_depth) & (kf_depth > 0.0) & (acc > 0.5)
    cnt = int(valid.sum())
    dd = np.where(valid, depth - np.where(valid, kf_depth, 0.0), 0.0)
    l_depth = float(np.abs(dd).sum() / cnt) if cnt else 0.0
    g_depth = w_depth * np.sign(dd) / cnt if cnt else np.zeros_like(depth)

    # feature distillation through the decoder
    y = decode(feat, w1, b1, w2, b2)
    fd = y - kf_feat
    l_feat = float(np.abs(fd).mean())
    g_y = w_feat * np.sign(fd) / fd.size
    g_feat = decode_backward_input(feat, g_y, w1, b1, w2)

    l_total = l_rgb + w_depth * l_depth + w_feat * l_feat
    br = dict(l_rgb=float(l_rgb), l_depth=l_depth, l_feat=l_feat, l_total=float(l_total), ssim=float(s),
              depth_pixels=cnt)
    return br, g_rgb, g_depth, g_feat


def coverage_mask(acc, depth, measured):
    """SPEC.md:225 insertion coverage: acc < 0.5 OR (measured valid and |depth - measured| >
    max(0.05 m, 0.05 measured)), evaluated in float32 like the kernel (so masks compare exactly)."""
    f = np.float32
    acc = np.asarray(acc, f)
    depth = np.asarray(depth, f)
    m = np.asarray(measured, f)
    valid = np.isfinite(m) & (m > f(0))
    with np.errstate(invalid="ignore"):
        err = np.abs(depth - m) > np.maximum(f(0.05), f(0.05) * m)
    return ((acc < f(0.5)) | (valid & err)).astype(np.uint8)
