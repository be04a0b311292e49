"""Golden fixtures (tests/golden/, made by make_golden.py): the oracle must reproduce them exactly
(CPU), and the CUDA path within the parity tolerances of tests/parity.py (GPU)."""
import os

import numpy as np
import pytest

from tests.parity import GROUPS, grad_mismatch, image_mismatch

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(HERE, name)))


def scene_of(z):
    return {k[6:]: z[k] for k in z if k.startswith("scene_")}


def cam_of(z):
    fx, fy, cx, cy, w, h = z["cam_k"]
    return dict(q=z["cam_q"], t=z["cam_t"], fx=fx, fy=fy, cx=cx, cy=cy, width=int(w), height=int(h))


GRAD101_CAM = dict(q=[1.0, 0, 0, 0], t=[0.0, 0, 0], fx=1.4 * 16, fy=1.4 * 16, cx=7.5, cy=7.5, width=16, height=16)


def grad101_cfg(z):
    rs, skip, tmin = z["cfg"]
    return dict(radius_sigma=float(rs), alpha_skip=float(skip), transmittance_min=float(tmin))


def test_oracle_reproduces_grad101(oracle):
    z = load("grad101.npz")
    s = {k: v.astype(np.float64) for k, v in scene_of(z).items()}
    out = oracle.render(s, GRAD101_CAM, grad101_cfg(z))
    assert np.array_equal(out.rgb, z["rgb"]) and np.array_equal(out.feat, z["feat"])
    g = oracle.render_backward(out, z["w_rgb"], z["w_depth"], z["w_feat"])
    for k in GROUPS:
        assert np.array_equal(g[k], z[f"g_{k}"]), k


def test_oracle_reproduces_sh3_pose(oracle):
    z = load("sh3_pose.npz")
    out = oracle.render(scene_of(z), cam_of(z))
    assert np.array_equal(out.rgb, z["rgb"]) and np.array_equal(out.depth, z["depth"])
    g = oracle.render_backward(out, z["cot_rgb"], z["cot_depth"], z["cot_feat"], pose=True)
    for k in GROUPS + ("pose",):
        assert np.array_equal(g[k], z[f"g_{k}"]), k


@pytest.mark.gpu
def test_gpu_matches_golden_grad101():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_16144_b200 import renderer as R
    z = load("grad101.npz")
    dev = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).cuda() for k, v in scene_of(z).items()}
    out = R.render(dev, GRAD101_CAM, R.RenderConfig(**grad101_cfg(z)))
    for a, b in ((out.rgb, z["rgb"]), (out.depth, z["depth"]), (out.feat, z["feat"])):
        assert image_mismatch(a, b)[0] == 0.0
    g = R.render_backward(None, out, *(torch.from_numpy(z[k].astype(np.float32)).cuda()
                                       for k in ("w_rgb", "w_depth", "w_feat")))
    for k in GROUPS:
        assert grad_mismatch(g[k], z[f"g_{k}"])[0] == 0.0, k


@pytest.mark.gpu
def test_gpu_matches_golden_sh3_pose():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2511_16144_b200 import renderer as R
    z = load("sh3_pose.npz")
    dev = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).cuda() for k, v in scene_of(z).items()}
    out = R.render(dev, cam_of(z))
    for a, b in ((out.rgb, z["rgb"]), (out.depth, z["depth"]), (out.feat, z["feat"]), (out.acc, z["acc"])):
        frac, mx = image_mismatch(a, b)
        assert frac < 1e-3, mx
    g = R.render_backward(None, out, *(torch.from_numpy(z[k].astype(np.float32)).cuda()
                                       for k in ("cot_rgb", "cot_depth", "cot_feat")), pose=True)
    for k in GROUPS:
        frac, worst = grad_mismatch(g[k], z[f"g_{k}"])
        assert frac < 1e-3, (k, frac, worst)
    assert grad_mismatch(g["pose"], z["g_pose"], floor=0.0)[0] == 0.0
