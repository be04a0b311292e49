"""Pins oracle A against every renderer test of the reference.

Each test restates one TEST_CASE of proj/tests/test_renderer.cpp (cited per
test) with the same fixtures, thresholds and tolerances.  The reference itself
cannot be built here (no Eigen3 / libpng / doctest), so these
known-answer and property tests are what pin the restatement.
"""
import math

import numpy as np
import pytest

from tests.ref_scenes import MapBuilder, logit, make_grad_scene, rel_err, scene_loss, small_camera, splat_at


def _map1(p, scale, ol, color, d=4):
    mb = MapBuilder(d)
    splat_at(mb, p, scale, ol, color)
    return mb.scene()


def test_on_axis_projection(oracle):
    """test_renderer.cpp:38-49."""
    s = _map1([0, 0, 1], 0.1, 0.0, [1, 0, 0])
    p = oracle.project_gaussian(s, 0, small_camera())
    assert p is not None
    assert p["cov2d"][0, 0] == pytest.approx(100.3, rel=1e-9)
    assert p["cov2d"][1, 1] == pytest.approx(100.3, rel=1e-9)
    assert abs(p["cov2d"][0, 1]) < 1e-9
    assert p["depth"] == pytest.approx(1.0)


def test_behind_camera_culled(oracle):
    """test_renderer.cpp:51-57."""
    s = _map1([0, 0, -1], 0.1, 0.0, [1, 0, 0])
    assert oracle.project_gaussian(s, 0, small_camera()) is None


def test_doubling_fx_doubles_offset(oracle):
    """test_renderer.cpp:59-71."""
    s = _map1([0.2, 0.1, 1.5], 0.05, 0.0, [1, 0, 0])
    k = small_camera()
    p1 = oracle.project_gaussian(s, 0, k)
    k2 = dict(k, fx=k["fx"] * 2, fy=k["fy"] * 2)
    p2 = oracle.project_gaussian(s, 0, k2)
    assert (p2["u"] - k["cx"]) == pytest.approx(2 * (p1["u"] - k["cx"]), rel=1e-12)
    assert (p2["v"] - k["cy"]) == pytest.approx(2 * (p1["v"] - k["cy"]), rel=1e-12)


def test_empty_map_background(oracle):
    """test_renderer.cpp:73-80."""
    s = MapBuilder(4).scene()
    out = oracle.render(s, small_camera())
    for img in (out.rgb, out.acc, out.depth, out.feat):
        assert np.all(img == 0.0)


def test_single_opaque_splat(oracle):
    """test_renderer.cpp:82-93."""
    s = _map1([0, 0, 1.0], 0.2, logit(0.99), [1, 0, 0])
    out = oracle.render(s, small_camera())
    cy = cx = 31
    assert out.rgb[cy, cx, 0] == pytest.approx(0.99, rel=1e-3)
    assert out.rgb[cy, cx, 1] == 0.0
    assert out.depth[cy, cx] == pytest.approx(1.0, rel=1e-9)
    assert out.acc[cy, cx] == pytest.approx(0.99, rel=1e-3)


def test_two_coincident_splats(oracle):
    """test_renderer.cpp:95-106."""
    mb = MapBuilder(4)
    splat_at(mb, [0, 0, 1.0], 0.5, logit(0.5), [1, 0, 0])
    splat_at(mb, [0, 0, 1.0001], 0.5, logit(0.5), [0, 1, 0])
    out = oracle.render(mb.scene(), small_camera())
    assert out.rgb[31, 31, 0] == pytest.approx(0.5, rel=1e-3)
    assert out.rgb[31, 31, 1] == pytest.approx(0.25, rel=1e-3)


def _random_splats(oracle, seed, count, zlo, zhi, xy, slo, shi, olo, ohi):
    rng = oracle.Rng(seed)
    gs = []
    for _ in range(count):
        p = [rng.uniform(-xy, xy), rng.uniform(-xy, xy), rng.uniform(zlo, zhi)]
        sc = rng.uniform(slo, shi)
        ol = rng.uniform(olo, ohi)
        col = [rng.uniform(0, 1), rng.uniform(0, 1), rng.uniform(0, 1)]
        f = [rng.normal() for _ in range(8)]
        gs.append((p, sc, ol, col, f))
    return gs


def test_insertion_order_invariance(oracle):
    """test_renderer.cpp:108-131."""
    gs = _random_splats(oracle, 31, 12, 0.8, 2.0, 0.3, 0.03, 0.08, -1, 2)
    fwd, rev = MapBuilder(8), MapBuilder(8)
    for g in gs:
        splat_at(fwd, g[0], g[1], g[2], g[3], g[4])
    for g in reversed(gs):
        splat_at(rev, g[0], g[1], g[2], g[3], g[4])
    a = oracle.render(fwd.scene(), small_camera())
    b = oracle.render(rev.scene(), small_camera())
    assert np.max(np.abs(a.rgb - b.rgb)) < 1e-12


def test_bounded_outputs(oracle):
    """test_renderer.cpp:133-161."""
    gs = _random_splats(oracle, 32, 30, 0.6, 2.5, 0.4, 0.02, 0.1, -1, 3)
    mb = MapBuilder(8)
    max_norm = 0.0
    for g in gs:
        splat_at(mb, g[0], g[1], g[2], g[3], g[4])
        max_norm = max(max_norm, float(np.linalg.norm(g[4])))
    out = oracle.render(mb.scene(), small_camera())
    assert np.all(out.acc >= 0.0) and np.all(out.acc <= 1.0 + 1e-12)
    assert np.all(out.rgb <= 1.01) and np.all(out.rgb >= 0.0)
    assert np.all(np.linalg.norm(out.feat, axis=2) <= max_norm + 1e-9)
    assert out.num_contributions > 0


def test_zero_cotangent_zero_grads(oracle):
    """test_renderer.cpp:163-173."""
    s = _map1([0, 0, 1], 0.1, 0.5, [0.5, 0.5, 0.5])
    out = oracle.render(s, small_camera())
    g = oracle.render_backward(out, None, None, np.zeros((64, 64, 4)))
    assert np.max(np.abs(g["feature"])) == 0.0
    assert np.linalg.norm(g["position"][0]) == 0.0


def test_color_grad_equals_weight(oracle):
    """test_renderer.cpp:175-187."""
    s = _map1([0, 0, 1], 0.2, logit(0.8), [0.3, 0.3, 0.3])
    out = oracle.render(s, small_camera())
    g_rgb = np.zeros((64, 64, 3))
    g_rgb[31, 31, 0] = 1.0
    g = oracle.render_backward(out, g_rgb, None, None)
    assert g["sh"][0, 0, 0] == pytest.approx(out.acc[31, 31], rel=1e-12)
    assert g["sh"][0, 0, 1] == 0.0


def test_mismatched_cotangent_throws(oracle):
    """test_renderer.cpp:189-196 (std::invalid_argument -> ValueError)."""
    s = _map1([0, 0, 1], 0.1, 0.0, [1, 1, 1])
    out = oracle.render(s, small_camera())
    with pytest.raises(ValueError):
        oracle.render_backward(out, np.zeros((8, 8, 3)), None, None)


def gradcheck(oracle, scene, cam, cfg, w_rgb, w_depth, w_feat, h=1e-4, pose=False):
    """gradcheck.hpp:105-148 (+ EXT: SH coefficients and camera pose)."""
    out = oracle.render(scene, cam, cfg)
    g = oracle.render_backward(out, w_rgb, w_depth, w_feat, pose=pose)
    worst = (0.0, "")

    def central(arr, idx):
        saved = arr[idx]
        arr[idx] = saved + h
        up = scene_loss(oracle, scene, cam, cfg, w_rgb, w_depth, w_feat)
        arr[idx] = saved - h
        dn = scene_loss(oracle, scene, cam, cfg, w_rgb, w_depth, w_feat)
        arr[idx] = saved
        return (up - dn) / (2 * h)

    def upd(a, fd, grp):
        nonlocal worst
        e = rel_err(a, fd)
        if e > worst[0]:
            worst = (e, grp)

    n = scene["pos"].shape[0]
    K = scene["sh"].shape[1]
    for i in range(n):
        for a in range(3):
            upd(g["position"][i, a], central(scene["pos"], (i, a)), "position")
            upd(g["log_scale"][i, a], central(scene["log_s"], (i, a)), "log_scale")
            upd(g["sh"][i, 0, a], central(scene["sh"], (i, 0, a)), "color")
        # raw quaternion, storage (x,y,z,w); gradient order (w,x,y,z)
        for gi, si in ((0, 3), (1, 0), (2, 1), (3, 2)):
            upd(g["rotation"][i, gi], central(scene["rot"], (i, si)), "rotation")
        upd(g["opacity_logit"][i], central(scene["opac"], (i,)), "opacity")
        for c in range(scene["feat"].shape[0]):
            upd(g["feature"][c, i], central(scene["feat"], (c, i)), "feature")
        for k in range(1, K):
            for a in range(3):
                upd(g["sh"][i, k, a], central(scene["sh"], (i, k, a)), "sh")
    if pose:
        for a in range(6):
            xi = np.zeros(6)
            xi[a] = h
            up = scene_loss(oracle, scene, oracle.perturb_pose(cam, xi), cfg, w_rgb, w_depth, w_feat)
            xi[a] = -h
            dn = scene_loss(oracle, scene, oracle.perturb_pose(cam, xi), cfg, w_rgb, w_depth, w_feat)
            upd(g["pose"][a], (up - dn) / (2 * h), "pose")
    return worst


def test_gradcheck_seed101(oracle):
    """test_renderer.cpp:198-204: make_grad_scene(12, 16, 8, 101), max rel err < 1e-3."""
    scene, cam, cfg, w_rgb, w_depth, w_feat = make_grad_scene(oracle, 12, 16, 8, 101)
    worst = gradcheck(oracle, scene, cam, cfg, w_rgb, w_depth, w_feat)
    assert worst[0] < 1e-3, worst
