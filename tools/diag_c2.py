"""Diagnostic: c2 images through eager full lists / eager layered / plan vs oracle A (injected)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_16144_b200 import renderer as R, scenes
from oracle import oracle as orc
from tests.test_gpu_scale_parity import run_bench_step

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
scene, cams, info = scenes.make_config(name, n=n)
cam = cams[0]
dev = {k: torch.from_numpy(v).cuda() for k, v in scene.items()}
full = R.render(dev, cam, ctx=R.Context(0, full_lists=True))
lay = R.render(dev, cam, ctx=R.Context(0))
torch.cuda.synchronize()
pre = orc.preprocess_f32(scene, cam)
gp = full.projected()
for k in ("u", "v", "depth", "conic", "opacity", "color"):
    vis = pre["visible"].astype(bool)
    a = gp[k][vis]; b = pre[k][vis]
    print("proj", k, "ndiff", int((a != b).sum()), "maxdiff", float(np.abs(a - b).max()))
ref = orc.render(scene, cam, inject=pre)
def md(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else a
    return float(np.abs(a.astype(np.float64) - b).max())
for key in ("rgb", "feat", "depth", "acc"):
    print(key, "full-ref", md(getattr(full, key), getattr(ref, key)), "lay-ref", md(getattr(lay, key), getattr(ref, key)),
          "full-lay", md(getattr(full, key), getattr(lay, key).detach().cpu().numpy().astype(np.float64)))
err = np.abs(full.rgb.cpu().numpy() - ref.rgb).max(axis=2)
y, x = np.unravel_index(np.argmax(err), err.shape)
print("worst pixel", y, x, err[y, x], "gpu", full.rgb.cpu().numpy()[y, x], "ref", ref.rgb[y, x], "acc", ref.acc[y, x])
print("contrib count ref", ref.contrib_counts()[y, x])
print("stats", full.stats(), lay.stats())
