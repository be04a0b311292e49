"""Oracle self-checks beyond the reference's own tests (CPU only).

* the reference Rng restatement (random.hpp) against the C++ standard's mt19937_64 known value;
* the EXT gradients the reference does not have (SH degree 1-3 colour, 6-DoF pose) against central
  finite differences, in the style of gradcheck.hpp:105-148;
* oracle B (fp32 twin) against oracle A (fp64): projection, culling, the alpha-ellipse tile rect;
* key-list invariants (sorted, ranges cover the list, every pair's tile inside its rect);
* the deterministic expf / logf used by both the kernels and the twin.
"""
import math

import numpy as np
import pytest

from paper_2511_16144_b200 import scenes
from tests.ref_scenes import make_grad_scene
from tests.test_oracle_reference import gradcheck


def test_mt19937_64_standard_value(oracle):
    """[rand.predef]: the 10000th invocation of a default-constructed mt19937_64 is 9981545732273789042."""
    r = oracle.Rng(5489)
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042


def test_rng_transforms(oracle):
    """random.hpp:19-21 uniform = (u64 >> 11) * 2^-53; normal is Box-Muller with a cached spare."""
    a, b = oracle.Rng(7), oracle.Rng(7)
    for _ in range(100):
        assert a.uniform() == (b.next_u64() >> 11) * 2.0 ** -53
    r = oracle.Rng(11)
    xs = np.array([r.normal() for _ in range(20000)])
    assert abs(xs.mean()) < 0.03 and abs(xs.std() - 1.0) < 0.03


@pytest.mark.parametrize("deg", [1, 2, 3])
def test_sh_and_pose_gradcheck(oracle, deg):
    scene, cam, cfg, w_rgb, w_depth, w_feat = make_grad_scene(oracle, 12, 16, 8, 101, sh_degree=deg)
    cam = oracle.perturb_pose(cam, np.array([0.05, -0.03, 0.02, 0.02, 0.01, -0.05]))
    worst = gradcheck(oracle, scene, cam, cfg, w_rgb, w_depth, w_feat, pose=True)
    assert worst[0] < 1e-3, worst


def test_pose_gradcheck_sh0_rotated_camera(oracle):
    scene, cam, cfg, w_rgb, w_depth, w_feat = make_grad_scene(oracle, 10, 16, 4, 7)
    cam = oracle.perturb_pose(cam, np.array([0.2, 0.1, -0.15, 0.05, -0.02, 0.03]))
    worst = gradcheck(oracle, scene, cam, cfg, w_rgb, w_depth, w_feat, pose=True)
    assert worst[0] < 1e-3, worst


def test_se3_exp_compose(oracle):
    """geometry.cpp:22-41: exp(0,0,pi/2, 0,0,0) rotates (1,0,0) to (0,1,0) (SPEC.md core-geometry)."""
    cam = dict(q=[1.0, 0, 0, 0], t=[0.0, 0, 0], fx=1, fy=1, cx=0, cy=0, width=1, height=1)
    c2 = oracle.perturb_pose(cam, np.array([0, 0, math.pi / 2, 0, 0, 0]))
    w, x, y, z = c2["q"]
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    assert np.allclose(R @ [1, 0, 0], [0, 1, 0], atol=1e-12)


def test_fp32_twin_matches_fp64_projection(oracle):
    scene, cams, info = scenes.make_config("c0")
    cam = cams[0]
    pre = oracle.preprocess_f32(scene, cam)
    vis32 = pre["visible"].astype(bool)
    n = scene["pos"].shape[0]
    agree = 0
    for i in range(0, n, 50):
        p = oracle.project_gaussian(scene, i, cam)
        if p is None:
            continue
        agree += 1
        if not vis32[i]:
            continue  # culled by the alpha box only (opacity below 1/255 or empty box)
        assert pre["u"][i] == pytest.approx(p["u"], rel=1e-5, abs=1e-4)
        assert pre["v"][i] == pytest.approx(p["v"], rel=1e-5, abs=1e-4)
        assert pre["depth"][i] == pytest.approx(p["depth"], rel=1e-6)
        assert pre["radius"][i] == pytest.approx(p["radius"], rel=1e-4)
        assert pre["conic"][i, 0] == pytest.approx(p["conic"][0, 0], rel=1e-4)
        # the tile rect is the reference pixel rect intersected with the alpha box
        r = p["radius"]
        assert pre["bbox"][i, 0] >= max(0, math.floor(p["u"] - r)) - 1
        assert pre["bbox"][i, 1] <= min(cam["width"] - 1, math.ceil(p["u"] + r)) + 1
    assert agree > 100


def test_alpha_box_preserves_images(oracle):
    """Injecting the twin's (alpha-box-clipped) records reproduces the plain fp64 render."""
    scene, cams, info = scenes.make_config("c0", n=4000)
    cam = cams[0]
    pre = oracle.preprocess_f32(scene, cam)
    a = oracle.render(scene, cam)
    b = oracle.render(scene, cam, inject=pre)
    assert a.num_contributions == b.num_contributions
    assert np.abs(a.rgb - b.rgb).max() < 1e-5
    assert np.abs(a.feat - b.feat).max() < 1e-5


def test_key_list_invariants(oracle):
    scene, cams, info = scenes.make_config("c0")
    cam = cams[0]
    pre = oracle.preprocess_f32(scene, cam)
    keys, vals, ranges = oracle.bin_f32(pre, cam["width"], cam["height"])
    assert np.all(np.diff(keys.astype(np.float64)) >= 0) or np.all(keys[1:] >= keys[:-1])
    tiles_x = (cam["width"] + 15) // 16
    assert ranges[:, 1].max() == len(keys)
    t = (keys >> np.uint64(32)).astype(np.int64)
    for ti in range(ranges.shape[0]):
        b, e = ranges[ti]
        assert np.all(t[b:e] == ti)
    bb = pre["bbox"][vals]
    tx, ty = t % tiles_x, t // tiles_x
    assert np.all(tx >= bb[:, 0] // 16) and np.all(tx <= bb[:, 1] // 16)
    assert np.all(ty >= bb[:, 2] // 16) and np.all(ty <= bb[:, 3] // 16)
    # depth ties broken by map index (renderer.cpp:114-117)
    same = keys[1:] == keys[:-1]
    assert np.all(vals[1:][same] > vals[:-1][same])


def test_deterministic_exp_log_accuracy(oracle):
    xs = np.linspace(-30, 30, 2001).astype(np.float32)
    e = np.array([oracle.expf32(x) for x in xs], dtype=np.float64)
    assert np.max(np.abs(e / np.exp(xs.astype(np.float64)) - 1)) < 3e-7
    ys = np.exp(np.linspace(0, 25, 1001)).astype(np.float32)
    lg = np.array([oracle.lib().orc_logf_export(float(y)) for y in ys], dtype=np.float64)
    assert np.max(np.abs(lg - np.log(ys.astype(np.float64)))) < 5e-6
