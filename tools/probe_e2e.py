"""Probe: one host thread's end-to-end step (host-mapped map, host targets, host gradients in delta
mode) per config: wall ms per step, the render's host_rows / listed / active, and the same with the
whole map copied.  Usage: python tools/probe_e2e.py c4 [c2 ...]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import pinned_like  # noqa: E402
from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402

for name in sys.argv[1:]:
    scene, cams, info = scenes.make_config(name)
    cam = cams[8 if name == "c4" else 0]
    hs = {k: pinned_like(v) for k, v in scene.items()}
    tg = {k: pinned_like(v) for k, v in scenes.make_targets(cam, scene["feat"].shape[0], info["depth_range"], 7).items()}
    n, d, K = scene["pos"].shape[0], scene["feat"].shape[0], scene["sh"].shape[1]
    H, W = cam["height"], cam["width"]
    img = {"rgb": pinned_like(np.zeros((H, W, 3), np.float32)), "depth": pinned_like(np.zeros((H, W), np.float32)),
           "feat": pinned_like(np.zeros((H, W, d), np.float32)), "acc": pinned_like(np.zeros((H, W), np.float32))}
    for mapped in (True, False):
        ctx = R.Context(0, stream="own", host_grad_delta=True)
        grads = R.alloc_grads(n, d, K, flat=pinned_like(np.zeros(n * (11 + 3 * K + d), np.float32)))
        ts = []
        for it in range(8):
            t0 = time.perf_counter()
            out = R.render(hs, cam, targets=tg, ctx=ctx, out=img, host_mapped=mapped)
            t1 = time.perf_counter()
            R.render_backward_l1(out, pose=True, into=grads)
            t2 = time.perf_counter()
            out.l1_loss()
            t3 = time.perf_counter()
            ts.append((t1 - t0, t2 - t1, t3 - t2))
        st = out.stats()
        ctx.profile(True)
        ctx.phase_times(reset=True)
        t0 = time.perf_counter()
        out = R.render(hs, cam, targets=tg, ctx=ctx, out=img, host_mapped=mapped)
        R.render_backward_l1(out, pose=True, into=grads)
        torch.cuda.synchronize()
        ph = ctx.phase_times()
        ctx.profile(False)
        print("   profiled step ms %.2f phases %s" % ((time.perf_counter() - t0) * 1e3, ph))
        a = np.array(ts[3:]) * 1e3
        print(name, "mapped" if mapped else "copied", "render/bwd/loss ms", a.mean(0).round(2), "total", a.sum(1).mean().round(2),
              {k: st.get(k) for k in ("host_rows", "listed", "active", "pairs", "layer_a")}, "layer_div", ctx.layer_div)
