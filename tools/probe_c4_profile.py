import cProfile, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from bench import pinned_like
from paper_2511_16144_b200 import renderer as R, scenes
scene, cams, info = scenes.make_config("c4"); cam = cams[8]
hs = {k: pinned_like(v) for k, v in scene.items()}
tg = {k: pinned_like(v) for k, v in scenes.make_targets(cam, 16, info["depth_range"], 7).items()}
x = torch.empty(900 << 20, dtype=torch.uint8, pin_memory=True); y = torch.empty_like(x, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize(); print("pinned H2D GB/s", 0.9e9 * 1.048 / (time.perf_counter() - t) / 1e9)
H, W = cam["height"], cam["width"]
img = {"rgb": pinned_like(np.zeros((H, W, 3), np.float32)), "depth": pinned_like(np.zeros((H, W), np.float32)),
       "feat": pinned_like(np.zeros((H, W, 16), np.float32)), "acc": pinned_like(np.zeros((H, W), np.float32))}
ctx = R.Context(0, stream="own")
for _ in range(3): R.render(hs, cam, targets=tg, ctx=ctx, out=img, host_mapped=True)
pr = cProfile.Profile(); pr.enable()
for _ in range(3): R.render(hs, cam, targets=tg, ctx=ctx, out=img, host_mapped=True)
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
