"""Layered vs complete tile lists on one config: where do gradients differ? (debug tool)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60000
scene, cams, info = scenes.make_config(name, n=n)
cam = cams[0]
tg = scenes.make_targets(cam, scene["feat"].shape[0], info["depth_range"], 3)
ds = {k: torch.from_numpy(v).cuda() for k, v in scene.items()}
dtg = {k: torch.from_numpy(v).cuda() for k, v in tg.items()}
res = []
for full in (False, True, True):
    ctx = R.Context(0, full_lists=full)
    out = R.render(ds, cam, targets=dtg, ctx=ctx)
    g = R.render_backward_l1(out, pose=True)
    torch.cuda.synchronize()
    res.append((out, g))
for k in ("position", "rotation", "log_scale", "opacity_logit", "sh", "feature", "pose"):
    a = res[0][1][k]
    b = res[1][1][k]
    c = res[2][1][k]
    a, b, c = [x if isinstance(x, np.ndarray) else x.cpu().numpy() for x in (a, b, c)]
    d1 = np.abs(a - b)
    d2 = np.abs(c - b)
    print(k, "layered-full max", d1.max(), "full-full max", d2.max(), "scale", np.abs(b).max(),
          "n>1e-3rel", int((d1 > 1e-3 * (np.abs(b) + 1e-2 * np.abs(b).max())).sum()))
lo, fo = res[0][0], res[1][0]
print("stats layered", lo.stats(), "full", fo.stats())
ft1, nc1 = lo.pixel_state()
ft2, nc2 = fo.pixel_state()
print("final_t equal", np.array_equal(ft1, ft2), "n_contrib equal", np.array_equal(nc1, nc2))
print("cot equal", all(np.array_equal(x, y) for x, y in zip(lo.cotangents(), fo.cotangents())))
lk, lv, lr = lo.tile_keys()
fk, fv, fr = fo.tile_keys()
bad = 0
for t in range(lr.shape[0]):
    a = lv[lr[t, 0]:lr[t, 1]]
    b = fv[fr[t, 0]:fr[t, 1]]
    if not np.array_equal(a, b[:a.size]):
        bad += 1
print("non-prefix tiles", bad)
