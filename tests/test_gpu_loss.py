"""GPU parity of the mapping losses (lgs_mapping_loss, csrc/loss.cu) against the fp64 oracle
(oracle/loss.py, pinned in test_loss_oracle.py) on the same rendered images.

Loss values: 1e-5 relative.  Cotangents: rgb (L1 sign + SSIM adjoint) and depth within
1e-4 relative plus 1e-4 of the channel's max magnitude; the feature cotangent goes through
sign(decode(feat) - F_gt), so a component may flip where the fp32 decoder output lies within
rounding of F_gt: such components must stay below 1e-3 of the total.  Map gradients through the
rasterizer backward: the 1e-3 bound of tests/parity.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import loss as OL  # noqa: E402
from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402
from tests.parity import GROUPS, grad_mismatch, to_np  # noqa: E402

D_TEACHER = 32
HIDDEN = 64


def _setup(name="c0", n=None, seed=3, invalid_frac=0.2):
    scene, cams, info = scenes.make_config(name, n=n)
    cam = cams[0]
    dscene = {k: torch.from_numpy(v).cuda() for k, v in scene.items()}
    out = R.render(dscene, cam)
    torch.cuda.synchronize()
    H, W = cam["height"], cam["width"]
    r = np.random.default_rng(seed)
    lo, hi = info["depth_range"]
    kf_depth = r.uniform(lo, hi, (H, W)).astype(np.float32)
    kf_depth[r.uniform(size=(H, W)) < invalid_frac] = 0.0
    kf = {"rgb": r.uniform(0, 1, (H, W, 3)).astype(np.float32), "depth": kf_depth,
          "feat_gt": r.normal(0, 0.5, (H, W, D_TEACHER)).astype(np.float32)}
    dec = scenes.make_decoder(D_TEACHER, HIDDEN, out.d, seed)
    return out, kf, dec


def _oracle(out, kf, dec, **w):
    return OL.compute_losses(to_np(out.rgb), to_np(out.depth), to_np(out.feat), to_np(out.acc), kf["rgb"],
                             kf["depth"], kf["feat_gt"], dec, **w)


def _close(got, ref, rtol=1e-4, frac_floor=1e-4):
    ref = np.asarray(ref, np.float64)
    tol = rtol * np.abs(ref) + frac_floor * (np.abs(ref).max() + 1e-30)
    return np.abs(np.asarray(got, np.float64) - ref) <= tol


@pytest.mark.parametrize("name,n", [("c0", None), ("c1", 40_000)])
def test_losses_and_cotangents_match_oracle(name, n):
    out, kf, dec = _setup(name, n)
    dkf = {k: torch.from_numpy(v).cuda() for k, v in kf.items()}
    ddec = tuple(torch.from_numpy(x).cuda() for x in dec)
    br = R.mapping_loss(out, dkf, ddec)
    ref, g_rgb, g_depth, g_feat = _oracle(out, kf, dec)
    for k in ("l_rgb", "l_depth", "l_feat", "l_total", "ssim"):
        assert br[k] == pytest.approx(ref[k], rel=1e-5, abs=1e-9), k
    assert br["depth_pixels"] == ref["depth_pixels"]
    c_rgb, c_depth, c_feat = out.cotangents()
    assert _close(c_rgb, g_rgb).all(), np.abs(c_rgb - g_rgb).max()
    assert _close(c_depth, g_depth).all()
    bad = ~_close(c_feat, g_feat)
    assert bad.mean() < 1e-3, (bad.mean(), np.abs(c_feat - g_feat).max())


def test_backward_through_loss_matches_explicit_cotangents():
    """render_backward_loss (tape cotangents) == render_backward fed the oracle's cotangents."""
    out, kf, dec = _setup("c0")
    R.mapping_loss(out, kf, dec)  # host keyframe / decoder: staged by the library
    g1 = R.render_backward_loss(out, pose=True)
    _, g_rgb, g_depth, g_feat = _oracle(out, kf, dec)
    cot = [torch.from_numpy(np.ascontiguousarray(c, np.float32)).cuda() for c in (g_rgb, g_depth, g_feat)]
    g2 = R.render_backward(None, out, *cot, pose=True)
    for k in GROUPS:
        frac, worst = grad_mismatch(g1[k], g2[k])
        assert frac < 1e-3, (k, frac, worst)


def test_invalid_depth_and_zero_feature_weight():
    """SPEC.md:426 invalid-depth frame -> l_depth = 0, no depth cotangent; SPEC.md:450 w_feat = 0 ->
    the map's feature gradient is exactly zero."""
    out, kf, dec = _setup("c0", invalid_frac=1.0)
    br = R.mapping_loss(out, kf, dec, w_feat=0.0)
    assert br["l_depth"] == 0.0 and br["depth_pixels"] == 0
    c_rgb, c_depth, c_feat = out.cotangents()
    assert not c_depth.any() and not c_feat.any()
    g = R.render_backward_loss(out)
    assert not g["feature"].any()


def test_perfect_fit_is_zero():
    """rendered = ground truth -> all losses 0 (the feature target is the decoder's
    own output on the rendered features, computed by the oracle)."""
    out, kf, dec = _setup("c0")
    rgb, depth, feat, acc = (to_np(x) for x in (out.rgb, out.depth, out.feat, out.acc))
    kf = {"rgb": rgb.copy(), "depth": depth.copy(), "feat_gt": OL.decode(feat, *dec).astype(np.float32)}
    br = R.mapping_loss(out, kf, dec)
    assert br["l_rgb"] == pytest.approx(0.0, abs=1e-6)
    assert br["l_depth"] == 0.0
    assert br["l_feat"] < 1e-6  # fp32 decoder vs fp64 target: rounding only


def test_argument_errors():
    out, kf, dec = _setup("c0")
    w1, b1, w2, b2 = dec
    with pytest.raises(ValueError):
        R.mapping_loss(out, kf, (w1[:, :4].copy(), b1, w2, b2))  # decoder low dim != map feature dim
    small, cams, _ = scenes.make_config("c0", n=500)
    cam = dict(cams[0], width=10, height=30)
    o2 = R.render({k: torch.from_numpy(v).cuda() for k, v in small.items()}, cam)
    kf2 = {"rgb": np.zeros((30, 10, 3), np.float32), "depth": np.zeros((30, 10), np.float32),
           "feat_gt": np.zeros((30, 10, D_TEACHER), np.float32)}
    with pytest.raises(ValueError):
        R.mapping_loss(o2, kf2, dec)  # narrower than the 11x11 SSIM window
