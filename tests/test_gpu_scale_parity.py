"""Parity of the BENCHED step at the benched sizes.

The step bench.py times is a captured plan (lgs_plan: preprocess -> depth-layered binning -> the
fused forward+backward blend kernel with the L1 loss -> preprocess backward -> pose gradient).  Here
that exact step runs at the headline config (c1_500k: 640x480, 500k Gaussians, SH3, d=16), at
configs[1] (c1: 200k), at configs[2] (c2: 1200x680, 1M) and at configs[0] (c0: 160x120, 10k -- a
small view binned in one pass with complete lists, the fused kernel on every tile), and is
compared with oracle A -- the
fp64 restatement of renderer.cpp:94-356 -- run on the same fp32 projected records (oracle B,
bit-exact with the GPU's; test_gpu_parity.py) and fed the cotangents the kernel computed from its
own images (so an L1 sign at |render - target| ~ 0 cannot masquerade as a gradient error):

* images: |gpu - ref| <= 1e-5 + 1e-4 |ref| (north_star) for every pixel the fp32 decision twin does
  not flag; flagged pixels outside tolerance are counted and printed, unexplained ones must be 0;
* gradients (every group): |gpu - ref| <= 1e-3 (|ref| + 0.01 rms) for every component whose
  Gaussian is not flagged; same accounting;
* pose gradient: within 1e-3 of the oracle's, relative to its largest component;
* complete tile key lists, sorted order and ranges at c1_500k: bit-exact vs oracle B.
"""
import numpy as np
import pytest

from tests.parity import GROUPS, explain_grad, explain_image, l1_cotangents_f32, to_np

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402


def run_bench_step(name, target_seed=7):
    """bench.py's timed step (run_ours): a Plan on its own stream, replayed after warm-up."""
    scene, cams, info = scenes.make_config(name)
    cam = cams[0]
    d, K, n = scene["feat"].shape[0], scene["sh"].shape[1], scene["pos"].shape[0]
    tg = scenes.make_targets(cam, d, info["depth_range"], target_seed)
    stream = torch.cuda.Stream()
    ctx = R.Context(0, stream=stream.cuda_stream)
    H, W = cam["height"], cam["width"]
    with torch.cuda.stream(stream):
        dmap = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
        dtg = {k: torch.from_numpy(v).cuda() for k, v in tg.items()}
        grads = R.alloc_grads(n, d, K, device=0)
        imgs = {"rgb": torch.empty(H, W, 3, device="cuda"), "depth": torch.empty(H, W, device="cuda"),
                "feat": torch.empty(H, W, d, device="cuda"), "acc": torch.empty(H, W, device="cuda")}
        pose = torch.zeros(6, dtype=torch.float32, pin_memory=True)
        plan = R.Plan(dmap, cam, dtg, grads, images=imgs, pose_out=pose)
        for _ in range(3):
            plan.run()
            plan.sync()
        grads["flat"].fill_(float("nan"))  # every row (zero rows included) must be rewritten
        imgs["rgb"].fill_(float("nan"))
        plan.run()
        plan.sync()
    torch.cuda.synchronize()
    out = {k: to_np(v) for k, v in imgs.items()}
    g = {k: to_np(grads[k]) for k in GROUPS}
    g["pose"] = pose.numpy().astype(np.float64)
    return scene, cam, tg, out, g


@pytest.mark.parametrize("name", ["c1_500k", "c1", "c2", "c0"])
def test_benched_plan_matches_oracle_at_scale(oracle, name):
    scene, cam, tg, out, g = run_bench_step(name)
    for k in GROUPS:
        assert np.isfinite(g[k]).all(), f"{k}: rows left unwritten"
    pre = oracle.preprocess_f32(scene, cam)
    ref = oracle.render(scene, cam, inject=pre)
    pix_flag, g_flag = ref.flags()
    report = {"config": name, "flagged_pixels": int(((pix_flag & 3) != 0).sum()),
              "flagged_gaussians": int((g_flag != 0).sum()), "contributions": ref.num_contributions}
    for key, r in (("rgb", ref.rgb), ("depth", ref.depth), ("feat", ref.feat), ("acc", ref.acc)):
        report[key] = explain_image(out[key], r, pix_flag)
    cot = l1_cotangents_f32(out["rgb"], out["depth"], out["feat"], tg)
    gref = oracle.render_backward(ref, *cot, pose=True)
    for k in GROUPS:
        report[k] = explain_grad(g[k], gref[k], g_flag, rows_last=(k == "feature"))
    pe = np.abs(g["pose"] - gref["pose"]) / np.abs(gref["pose"]).max()
    report["pose"] = {"gpu": g["pose"].tolist(), "ref": gref["pose"].tolist(), "max_err": float(pe.max())}
    print("\nscale parity", report)
    for key in ("rgb", "depth", "feat", "acc") + GROUPS:
        assert report[key]["unexplained"] == 0, (key, report[key])
    assert pe.max() <= 1e-3, report["pose"]


def test_complete_lists_bit_exact_at_headline(oracle):
    scene, cams, info = scenes.make_config("c1_500k")
    cam = cams[0]
    ctx = R.Context(0, full_lists=True)
    o = R.render({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, cam, ctx=ctx)
    torch.cuda.synchronize()
    keys, vals, ranges = o.tile_keys()
    op = oracle.preprocess_f32(scene, cam)
    okeys, ovals, oranges = oracle.bin_f32(op, cam["width"], cam["height"])
    print(f"\nc1_500k complete lists: {okeys.size} pairs")
    assert keys.shape == okeys.shape
    assert np.array_equal(keys, okeys), "tile key lists differ"
    assert np.array_equal(vals, ovals), "sorted order differs"
    assert np.array_equal(ranges, oranges), "tile ranges differ"
