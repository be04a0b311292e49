"""Captured steps (lgs_plan_*: fused-L1 forward + backward in one CUDA graph) reproduce the eager
API: images bit-identical, gradients within the atomic-order bound of tests/parity.py, the pose
gradient within 1e-3; the capacity re-capture path (pair count outgrows the tile lists) and a
camera change give the eager results too."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402
from tests.parity import GROUPS, grad_mismatch  # noqa: E402


def _setup(n=30_000, name="c1"):
    scene, cams, info = scenes.make_config(name, n=n)
    cam = cams[0]
    ctx = R.Context(0)
    dm = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
    tg = {k: torch.from_numpy(v).cuda() for k, v in scenes.make_targets(cam, dm.d, info["depth_range"], 3).items()}
    return scene, cam, ctx, dm, tg


def _images(cam, d):
    H, W = cam["height"], cam["width"]
    return {"rgb": torch.zeros(H, W, 3, device="cuda"), "depth": torch.zeros(H, W, device="cuda"),
            "feat": torch.zeros(H, W, d, device="cuda"), "acc": torch.zeros(H, W, device="cuda")}


def _eager(dm, cam, tg):
    out = R.render(dm, cam, targets=tg)
    g = R.render_backward_l1(out, pose=True)
    torch.cuda.synchronize()
    return out, g


def _check(plan_grads, pose, imgs, out, g):
    assert torch.equal(imgs["rgb"], out.rgb) and torch.equal(imgs["feat"], out.feat)
    assert torch.equal(imgs["depth"], out.depth) and torch.equal(imgs["acc"], out.acc)
    for k in GROUPS:  # atomic accumulation order differs run to run (same allowance as the oracle tests)
        frac, worst = grad_mismatch(plan_grads[k], g[k])
        assert frac < 1e-3, (k, frac, worst)
    # the pose gradient sums every splat's contribution (the geometric accumulator slots are fp64,
    # so the atomic order moves it only in the last float digits)
    assert np.allclose(pose.numpy(), g["pose"], rtol=1e-4, atol=1e-5 * np.abs(g["pose"]).max())


def test_plan_matches_eager_and_replays():
    scene, cam, ctx, dm, tg = _setup()
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    imgs = _images(cam, dm.d)
    pose = torch.zeros(6, dtype=torch.float32, pin_memory=True)
    plan = R.Plan(dm, cam, tg, grads, images=imgs, pose_out=pose)
    assert plan.launches > 10
    out, g = _eager(dm, cam, tg)
    for _ in range(3):  # replays are stable, and every gradient row is written (zero rows included)
        grads["flat"].fill_(float("nan"))
        plan.run()
        pairs = plan.sync()
        assert not torch.isnan(grads["flat"]).any()
        _check(grads, pose, imgs, out, g)
    assert pairs == out.stats()["pairs"]
    assert plan.elapsed_ms() > 0.0


def test_plan_recaptures_when_pairs_outgrow_capacity():
    scene, cam, ctx, dm, tg = _setup()
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    imgs = _images(cam, dm.d)
    pose = torch.zeros(6, dtype=torch.float32, pin_memory=True)
    plan = R.Plan(dm, cam, tg, grads, images=imgs, pose_out=pose)
    p0 = plan.sync()
    bigger = dict(scene, log_s=(scene["log_s"] + 0.7).astype(np.float32))  # larger splats: more pairs
    dm.update({k: torch.from_numpy(v).cuda() for k, v in bigger.items()})
    plan.run()
    p1 = plan.sync()
    assert p1 > 1.25 * p0
    out, g = _eager(dm, cam, tg)
    _check(grads, pose, imgs, out, g)


def test_plan_set_camera():
    scene, cam, ctx, dm, tg = _setup()
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    imgs = _images(cam, dm.d)
    pose = torch.zeros(6, dtype=torch.float32, pin_memory=True)
    plan = R.Plan(dm, cam, tg, grads, images=imgs, pose_out=pose)
    cam2 = dict(cam, t=np.array([0.05, -0.02, 0.1]))
    plan.set_camera(cam2)
    plan.run()
    plan.sync()
    out, g = _eager(dm, cam2, tg)
    _check(grads, pose, imgs, out, g)


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c4"])
def test_plan_layered_second_pass_toggles(name):
    """The second pass of the depth-layered binning is a conditional node of the captured graph:
    a replay where tiles stay unsaturated (tiny, faint splats) runs it, a dense one skips it; both
    must reproduce the eager results."""
    scene, cam, ctx, dm, tg = _setup(n=20_000, name=name)
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    imgs = _images(cam, dm.d)
    pose = torch.zeros(6, dtype=torch.float32, pin_memory=True)
    plan = R.Plan(dm, cam, tg, grads, images=imgs, pose_out=pose)
    sparse = dict(scene, log_s=(scene["log_s"] - 0.5).astype(np.float32),
                  opac=(scene["opac"] - 2.0).astype(np.float32))
    for sc in (sparse, scene, sparse):
        dm.update({k: torch.from_numpy(v).cuda() for k, v in sc.items()})
        plan.run()
        plan.sync()
        out, g = _eager(dm, cam, tg)
        _check(grads, pose, imgs, out, g)


def test_eager_backward_overwrites_every_row():
    """The layered backward writes the chain's rows for the active Gaussians only and streams zeros
    into every other row: a gradient buffer full of NaN comes back equal to a fresh one."""
    scene, cam, ctx, dm, tg = _setup()
    out, g = _eager(dm, cam, tg)
    dirty = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    dirty["flat"].fill_(float("nan"))
    out2 = R.render(dm, cam, targets=tg)
    R.render_backward_l1(out2, into=dirty)
    torch.cuda.synchronize()
    assert not torch.isnan(dirty["flat"]).any()
    for k in GROUPS:
        frac, worst = grad_mismatch(dirty[k], g[k])
        assert frac < 1e-3, (k, frac, worst)


def test_speculative_plan_and_fallback():
    """A plan whose warm-up render saturated every tile on its layer-A list is captured without the
    second pass (lgs_plan_speculative).  Its replays match a plan captured with the pass and the
    eager step; a replay that leaves tiles unsaturated (faint splats) is detected, re-captured with
    the second pass and re-run inside sync(), and the results are again the eager ones."""
    scene, cams, info = scenes.make_config("c1", n=500_000)
    cam = cams[0]
    tg_np = scenes.make_targets(cam, scene["feat"].shape[0], info["depth_range"], 3)
    res = {}
    for spec in (True, False):
        ctx = R.Context(0, speculative_plans=spec)
        dm = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
        tg = {k: torch.from_numpy(v).cuda() for k, v in tg_np.items()}
        grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
        imgs = _images(cam, dm.d)
        pose = torch.zeros(6, dtype=torch.float32, pin_memory=True)
        plan = R.Plan(dm, cam, tg, grads, images=imgs, pose_out=pose)
        assert plan.speculative == spec
        plan.run()
        plan.sync()
        assert plan.recaptures == 0
        res[spec] = ({k: v.clone() for k, v in imgs.items()}, plan, dm, tg, grads, imgs, pose)
    for k in ("rgb", "depth", "feat", "acc"):
        assert torch.equal(res[True][0][k], res[False][0][k]), k
    _, plan, dm, tg, grads, imgs, pose = res[True]
    out, g = _eager(dm, cam, tg)
    _check(grads, pose, imgs, out, g)
    faint = dict(scene, opac=(scene["opac"] - 4.0).astype(np.float32))
    dm.update({k: torch.from_numpy(v).cuda() for k, v in faint.items()})
    plan.run()
    plan.sync()
    assert plan.recaptures == 1 and not plan.speculative
    out, g = _eager(dm, cam, tg)
    _check(grads, pose, imgs, out, g)
    dm.update({k: torch.from_numpy(v).cuda() for k, v in scene.items()})
    plan.run()
    plan.sync()
    assert plan.recaptures == 1
    out, g = _eager(dm, cam, tg)
    _check(grads, pose, imgs, out, g)


def test_speculative_accumulating_plans_miss_adds_nothing():
    """A two-plan batch on one gradient buffer (the same view twice): the writing plan captured with
    the second pass, the accumulating one speculative.  When the splats of one half of the image
    turn faint, that half's tiles stay unsaturated while the other half's finish and produce
    gradients: the speculative replay misses and its gradient chain must add nothing (a partial
    sum would stay under the re-run's), then sync_plans() re-runs it with the second pass -- the
    buffer holds exactly twice the eager gradients."""
    from paper_2511_16144_b200 import _lib
    scene, cams, info = scenes.make_config("c1", n=500_000)
    cam = cams[0]
    ctx = R.Context(0)
    dm = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
    tg = {k: torch.from_numpy(v).cuda() for k, v in scenes.make_targets(cam, dm.d, info["depth_range"], 3).items()}
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    poses = [torch.zeros(6, dtype=torch.float32, pin_memory=True) for _ in range(2)]
    plans = []
    for i in range(2):  # the writer with the second pass, the accumulating plan speculative
        _lib.load().lgs_ctx_set_option(ctx.h, _lib.LGS_OPT_SPECULATIVE_PLANS, i)
        plans.append(R.Plan(dm, cam, tg, grads, pose_out=poses[i], accumulate=i > 0))
    assert [p.speculative for p in plans] == [False, True]
    half = scene["opac"].copy()
    half[scene["pos"][:, 0] > 0] -= 4.0  # one half of the view faint: a partly unsaturated replay
    for sc, misses in ((scene, 0), (dict(scene, opac=half.astype(np.float32)), 1)):
        dm.update({k: torch.from_numpy(v).cuda() for k, v in sc.items()})
        for p in plans:
            p.run()
        R.sync_plans(plans)
        assert [p.recaptures for p in plans] == [0, misses]
        out, g = _eager(dm, cam, tg)
        for k in GROUPS:
            frac, worst = grad_mismatch(grads[k], 2.0 * g[k])
            assert frac < 1e-3, (k, frac, worst)
            # the gradient mass too: a partial sum left by the missed replay would add ~1/2 of it
            a = grads[k].detach().double().cpu().numpy() if hasattr(grads[k], "detach") else np.asarray(grads[k])
            b = 2.0 * np.asarray(g[k].detach().cpu().numpy() if hasattr(g[k], "detach") else g[k], dtype=np.float64)
            assert np.abs(a - b).sum() <= 1e-3 * np.abs(b).sum(), (k, np.abs(a - b).sum() / np.abs(b).sum())
        for pose in poses:
            assert np.allclose(pose.numpy(), g["pose"], rtol=1e-4, atol=1e-5 * np.abs(g["pose"]).max())


def test_sync_plans_reruns_the_batch_after_the_first_plan():
    """A batch whose first (writing) plan outgrows its tile lists while the accumulating plan does
    not: the first plan's re-run rewrites the buffer, so sync_plans runs the second again."""
    scene, cam, ctx, dm, tg = _setup()
    cam2 = dict(cam, t=np.array([0.05, 0.0, 0.0]))
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    poses = [torch.zeros(6, dtype=torch.float32, pin_memory=True) for _ in range(2)]
    bigger = dict(scene, log_s=(scene["log_s"] + 0.7).astype(np.float32))
    dev = lambda sc: {k: torch.from_numpy(v).cuda() for k, v in sc.items()}  # noqa: E731
    plans = [R.Plan(dm, cam, tg, grads, pose_out=poses[0])]
    dm.update(dev(bigger))  # the context's list capacity grows before the second plan captures
    R.render(dm, cam, targets=tg, ctx=ctx)
    torch.cuda.synchronize()
    dm.update(dev(scene))
    plans.append(R.Plan(dm, cam2, tg, grads, pose_out=poses[1], accumulate=True))
    for p in plans:
        p.run()
    R.sync_plans(plans)
    dm.update(dev(bigger))
    for p in plans:
        p.run()
    R.sync_plans(plans)
    assert [p.recaptures for p in plans] == [1, 0]
    _, g0 = _eager(dm, cam, tg)
    _, g1 = _eager(dm, cam2, tg)
    for k in GROUPS:
        frac, worst = grad_mismatch(grads[k], g0[k] + g1[k])
        assert frac < 1e-3, (k, frac, worst)
