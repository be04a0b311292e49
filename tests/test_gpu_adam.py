"""GPU Adam step on the resident map (lgs_adam_step, csrc/optim.cu) against the float32 numpy
restatement (oracle/adam.py), plus lgs_map_download and a short mapping loop
(render -> mapping loss -> backward -> Adam) that must reduce the loss."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import loss as OL  # noqa: E402
from oracle.adam import DEFAULT, AdamOracle  # noqa: E402
from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402

LR_KEY = {"pos": "lr_position", "rot": "lr_rotation", "log_s": "lr_log_scale", "opac": "lr_opacity",
          "sh": "lr_color", "feat": "lr_feature"}


def _dev(scene):
    return {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).cuda() for k, v in scene.items()}


@pytest.mark.parametrize("n", [5000, 4001])  # n % 4 != 0: rotation rows at float offset 3n
def test_map_download_round_trip(n):
    scene, _, _ = scenes.make_config("c1", n=n)
    dm = R.DeviceMap(_dev(scene))
    back = R.map_download(dm)
    for k, v in scene.items():
        assert np.array_equal(back[k], np.asarray(v, np.float32)), k
    dback = R.map_download(dm, device=True)
    for k, v in scene.items():
        assert np.array_equal(dback[k].cpu().numpy(), np.asarray(v, np.float32)), k


@pytest.mark.parametrize("name,n", [("c0", 4000), ("c0", 4001), ("c1", 20_000), ("c1", 20_003)])
def test_adam_steps_match_oracle(name, n):
    scene, cams, info = scenes.make_config(name, n=n)
    cam = cams[0]
    dm = R.DeviceMap(_dev(scene))
    opt = R.Adam(dm)
    ref = AdamOracle(scene)
    tg = {k: torch.from_numpy(v).cuda() for k, v in scenes.make_targets(cam, dm.d, info["depth_range"], 4).items()}
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    for it in range(3):
        out = R.render(dm, dict(cam, t=np.array([0.01 * it, 0.0, 0.0])), targets=tg)
        R.render_backward_l1(out, into=grads)
        host = {k: v.cpu().numpy() for k, v in grads.items() if k != "flat"}
        opt.step(grads)
        ref.step(host)
    torch.cuda.synchronize()
    assert opt.steps == 3
    got = R.map_download(dm)
    for k, lrk in LR_KEY.items():
        want = ref.p[k]
        tol = 1e-6 * np.abs(want) + 1e-3 * DEFAULT[lrk]
        bad = np.abs(got[k] - want) > tol
        assert not bad.any(), (k, float(np.abs(got[k] - want).max()))
    # the update really moved the parameters (by ~lr per step)
    assert np.abs(got["opac"] - scene["opac"]).max() > 1e-2


def test_adam_argument_errors():
    scene, _, _ = scenes.make_config("c0", n=1000)
    dm = R.DeviceMap(_dev(scene))
    opt = R.Adam(dm)
    host = R.alloc_grads(dm.n, dm.d, dm.K)  # host memory
    with pytest.raises(ValueError):
        opt.step(host)
    other = R.DeviceMap(_dev(scenes.make_config("c0", n=999)[0]))
    with pytest.raises(ValueError):
        opt.map = other
        opt.step(R.alloc_grads(other.n, other.d, other.K, device=0))
    with pytest.raises(TypeError):
        R.Adam(dm, lr_unknown=1.0)


def test_mapping_loop_reduces_loss():
    """render -> lgs_mapping_loss -> backward -> Adam, fitting a keyframe rendered from a perturbed
    copy of the map: l_total decreases (smoothed trace non-increasing)."""
    scene, cams, info = scenes.make_config("c0", n=3000)
    cam = cams[0]
    target = {k: np.array(v, np.float32, copy=True) for k, v in scene.items()}
    r = np.random.default_rng(0)
    target["sh"] = np.clip(target["sh"] + r.normal(0, 0.15, target["sh"].shape), 0, 1).astype(np.float32)
    target["opac"] = (target["opac"] + r.normal(0, 0.5, target["opac"].shape)).astype(np.float32)
    kf_out = R.render(_dev(target), cam)
    dec = scenes.make_decoder(32, 64, 16, 1)
    kf = {"rgb": kf_out.rgb.clone(), "depth": kf_out.depth.clone(),
          "feat_gt": torch.from_numpy(OL.decode(kf_out.feat.cpu().numpy(), *dec).astype(np.float32)).cuda()}
    dm = R.DeviceMap(_dev(scene))
    opt = R.Adam(dm)
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    losses = []
    for _ in range(40):
        out = R.render(dm, cam)
        losses.append(R.mapping_loss(out, kf, dec)["l_total"])
        R.render_backward_loss(out, into=grads)
        opt.step(grads)
    assert np.mean(losses[-5:]) < 0.8 * np.mean(losses[:5]), losses
