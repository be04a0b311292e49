import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from bench import pinned_like
from paper_2511_16144_b200 import renderer as R, scenes
scene, cams, info = scenes.make_config("c4"); cam = cams[8]
hs = {k: pinned_like(v) for k, v in scene.items()}
tg = {k: pinned_like(v) for k, v in scenes.make_targets(cam, 16, info["depth_range"], 7).items()}
H, W = cam["height"], cam["width"]
img = {"rgb": pinned_like(np.zeros((H, W, 3), np.float32)), "depth": pinned_like(np.zeros((H, W), np.float32)),
       "feat": pinned_like(np.zeros((H, W, 16), np.float32)), "acc": pinned_like(np.zeros((H, W), np.float32))}
ctx = R.Context(0, stream="own")
for i in range(12):
    t = time.perf_counter()
    R.render(hs, cam, targets=tg, ctx=ctx, out=img, host_mapped=True)
    print("render ms %.2f" % ((time.perf_counter() - t) * 1e3), file=sys.stderr)
