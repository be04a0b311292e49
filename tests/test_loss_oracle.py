"""Pins the loss / decoder-chain oracle (oracle/loss.py) against the reference's own examples for
these operations (SPEC.md:410-426 ssim / compute_losses, SPEC.md:446-450 invariants, codec
examples SPEC.md:330-340) and against central finite differences, before it is used to check the
CUDA loss kernels."""
import numpy as np
import pytest

from oracle import loss as L
from paper_2511_16144_b200 import scenes


def _rng(seed=0):
    return np.random.default_rng(seed)


def test_ssim_self_is_one():
    a = _rng().uniform(0, 1, (24, 30, 3))
    assert L.ssim(a, a) == pytest.approx(1.0, abs=1e-12)


def test_ssim_constant_images_closed_form():
    """constant v vs constant w -> (2vw + C1)(0 + C2) / ((v^2 + w^2 + C1)(0 + 0 + C2))."""
    for v, w in ((0.2, 0.7), (0.5, 0.5), (0.0, 1.0)):
        a = np.full((16, 16, 3), v)
        b = np.full((16, 16, 3), w)
        want = (2 * v * w + L.C1) * L.C2 / ((v * v + w * w + L.C1) * L.C2)
        assert L.ssim(a, b) == pytest.approx(want, rel=1e-12)


def test_ssim_anticorrelated_checker_negative():
    """ssim(a, 1 - a) on a black/white checker is negative."""
    yy, xx = np.mgrid[0:20, 0:20]
    a = ((xx + yy) % 2).astype(np.float64)[..., None].repeat(3, axis=2)
    assert L.ssim(a, 1.0 - a) < 0.0


def test_ssim_rejects_shape_mismatch_and_small_images():
    with pytest.raises(ValueError):
        L.ssim(np.zeros((12, 12, 3)), np.zeros((12, 13, 3)))
    with pytest.raises(ValueError):
        L.ssim(np.zeros((10, 12, 3)), np.zeros((10, 12, 3)))


def _frame(seed, H=20, W=24, d=4, D=6, hidden=8):
    r = _rng(seed)
    rgb = r.uniform(0, 1, (H, W, 3))
    depth = r.uniform(1, 3, (H, W))
    feat = r.normal(0, 1, (H, W, d))
    acc = r.uniform(0, 1, (H, W))
    kf_rgb = r.uniform(0, 1, (H, W, 3))
    kf_depth = r.uniform(1, 3, (H, W))
    kf_depth[r.uniform(size=(H, W)) < 0.2] = 0.0  # invalid measurements
    kf_feat = r.normal(0, 1, (H, W, D))
    dec = tuple(np.asarray(x, np.float64) for x in scenes.make_decoder(D, hidden, d, seed))
    return rgb, depth, feat, acc, kf_rgb, kf_depth, kf_feat, dec


def test_perfect_fit_all_zero():
    """rendered = ground truth exactly -> all losses 0."""
    rgb, depth, feat, acc, _, _, _, dec = _frame(1)
    kf_feat = L.decode(feat, *dec)
    br, g_rgb, g_depth, g_feat = L.compute_losses(rgb, depth, feat, np.ones_like(acc), rgb, depth, kf_feat, dec)
    assert br["l_rgb"] == pytest.approx(0.0, abs=1e-12)
    assert br["l_depth"] == 0.0 and br["l_feat"] == pytest.approx(0.0, abs=1e-12)
    assert br["l_total"] == pytest.approx(0.0, abs=1e-12)


def test_constant_rgb_offset_closed_form():
    """rgb off by +0.1 everywhere -> l_rgb = 0.8 * 0.1 + 0.2 * D-SSIM(offset), where for
    x = y + 0.1 every window has sigma_x = sigma_y = sigma_xy, so
    SSIM = (2 mu_x mu_y + C1) / (mu_x^2 + mu_y^2 + C1) with mu_x = mu_y + 0.1."""
    rgb, depth, feat, acc, kf_rgb, kf_depth, _, dec = _frame(2)
    kf_rgb = np.clip(kf_rgb, 0.0, 0.9)
    kf_feat = L.decode(feat, *dec)
    br, *_ = L.compute_losses(kf_rgb + 0.1, depth, feat, acc, kf_rgb, kf_depth, kf_feat, dec)
    w = L.gauss_window()
    s = []
    for c in range(3):
        my = L._blur_valid(kf_rgb[..., c], w)
        mx = my + 0.1
        s.append(((2 * mx * my + L.C1) / (mx * mx + my * my + L.C1)).mean())
    want = 0.8 * 0.1 + 0.2 * (1.0 - np.mean(s)) / 2.0
    assert br["l_rgb"] == pytest.approx(want, rel=1e-10)


def test_invalid_depth_frame():
    """invalid-depth frame -> l_depth = 0 and no depth cotangent."""
    rgb, depth, feat, acc, kf_rgb, _, kf_feat, dec = _frame(3)
    kf_depth = np.zeros_like(depth)
    kf_depth[0, 0] = np.nan
    br, _, g_depth, _ = L.compute_losses(rgb, depth, feat, acc, kf_rgb, kf_depth, kf_feat, dec)
    assert br["l_depth"] == 0.0 and br["depth_pixels"] == 0
    assert not g_depth.any()


def test_total_decomposition_and_zero_feature_weight():
    """SPEC.md:401 l_total identity (1e-9); w_feat = 0 -> exactly zero feature gradient."""
    rgb, depth, feat, acc, kf_rgb, kf_depth, kf_feat, dec = _frame(4)
    br, *_ = L.compute_losses(rgb, depth, feat, acc, kf_rgb, kf_depth, kf_feat, dec, w_depth=0.5, w_feat=1.0)
    assert br["l_total"] == pytest.approx(br["l_rgb"] + 0.5 * br["l_depth"] + br["l_feat"], abs=1e-9)
    _, _, _, g_feat = L.compute_losses(rgb, depth, feat, acc, kf_rgb, kf_depth, kf_feat, dec, w_feat=0.0)
    assert not g_feat.any()


def test_decoder_zero_in_zero_out_and_pixel_independence():
    """zero input through a zero-bias decoder -> zero; 1x1 image = single vector."""
    w1, b1, w2, b2 = (np.asarray(x, np.float64) for x in scenes.make_decoder(6, 8, 4, 5))
    assert not L.decode(np.zeros((3, 3, 4)), w1, 0 * b1, w2, 0 * b2).any()
    z = _rng(5).normal(size=(5, 7, 4))
    full = L.decode(z, w1, b1, w2, b2)
    one = L.decode(z[2:3, 4:5], w1, b1, w2, b2)
    assert np.allclose(full[2:3, 4:5], one, rtol=1e-14, atol=0)  # BLAS blocking: last-bit only


def test_cotangents_match_finite_differences():
    """SPEC.md:449 style: the loss gradient w.r.t. the rendered images matches central differences
    (h = 1e-4) within 1e-3 relative, through the SSIM and the decoder chain."""
    rgb, depth, feat, acc, kf_rgb, kf_depth, kf_feat, dec = _frame(6, H=14, W=15)
    _, g_rgb, g_depth, g_feat = L.compute_losses(rgb, depth, feat, acc, kf_rgb, kf_depth, kf_feat, dec)
    h = 1e-4
    r = _rng(7)

    def total(rg, dp, ft):
        return L.compute_losses(rg, dp, ft, acc, kf_rgb, kf_depth, kf_feat, dec)[0]["l_total"]

    for name, arr, g in (("rgb", rgb, g_rgb), ("depth", depth, g_depth), ("feat", feat, g_feat)):
        for _ in range(12):
            idx = tuple(r.integers(0, s) for s in arr.shape)
            ap, am = arr.copy(), arr.copy()
            ap[idx] += h
            am[idx] -= h
            args_p = {"rgb": (ap, depth, feat), "depth": (rgb, ap, feat), "feat": (rgb, depth, ap)}[name]
            args_m = {"rgb": (am, depth, feat), "depth": (rgb, am, feat), "feat": (rgb, depth, am)}[name]
            fd = (total(*args_p) - total(*args_m)) / (2 * h)
            assert abs(fd - g[idx]) <= 1e-3 * (abs(fd) + 1e-6), (name, idx, fd, g[idx])


def test_coverage_mask_rule():
    """selected iff acc < 0.5 OR |depth - measured| > max(0.05 m, 0.05 depth)."""
    acc = np.array([0.4, 0.9, 0.9, 0.9, 0.9, 0.9])
    depth = np.array([1.0, 1.0, 1.0, 4.0, 4.0, 1.0])
    meas = np.array([1.0, 1.04, 1.06, 4.19, 4.25, 0.0])
    assert list(L.coverage_mask(acc, depth, meas)) == [1, 0, 1, 0, 1, 0]
