"""Plan (fused step) vs eager gradients vs eager-vs-eager noise (debug tool): python tools/diag_plan.py c4"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402
from tests.parity import GROUPS, grad_mismatch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
scene, cams, info = scenes.make_config(name, n=20000)
cam = cams[0]
ctx = R.Context(0)
dm = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
tg = {k: torch.from_numpy(v).cuda() for k, v in scenes.make_targets(cam, dm.d, info["depth_range"], 3).items()}
for label, sc in (("dense", scene), ("sparse", dict(scene, log_s=(scene["log_s"] - 0.5).astype(np.float32),
                                                     opac=(scene["opac"] - 2.0).astype(np.float32)))):
    dm.update({k: torch.from_numpy(v).cuda() for k, v in sc.items()})
    runs = []
    for _ in range(2):
        out = R.render(dm, cam, targets=tg)
        runs.append(R.render_backward_l1(out, pose=True))
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    H, W = cam["height"], cam["width"]
    imgs = {"rgb": torch.zeros(H, W, 3, device="cuda"), "depth": torch.zeros(H, W, device="cuda"),
            "feat": torch.zeros(H, W, dm.d, device="cuda"), "acc": torch.zeros(H, W, device="cuda")}
    pose = torch.zeros(6, dtype=torch.float32, pin_memory=True)
    plan = R.Plan(dm, cam, tg, grads, images=imgs, pose_out=pose)
    plan.run()
    plan.sync()
    torch.cuda.synchronize()
    st = out.stats()
    print(label, "listed", st["listed"], "pairs", st["pairs"])
    for k in GROUPS:
        f1, w1 = grad_mismatch(runs[1][k], runs[0][k])
        f2, w2 = grad_mismatch(grads[k], runs[0][k])
        print(f"  {k:14s} eager-eager frac {f1:.2e} worst {w1:.2e} | plan-eager frac {f2:.2e} worst {w2:.2e}")
    print("  pose eager", runs[0]["pose"], "eager2", runs[1]["pose"], "plan", pose.numpy())
