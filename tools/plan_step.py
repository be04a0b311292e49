"""A few replays of the captured fused step (lgs_plan) on a small config, for compute-sanitizer:
python tools/plan_step.py [config] [n] [replays]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c0"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else None
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    scene, cams, info = scenes.make_config(cfg, n=n)
    cam = cams[0]
    d = scene["feat"].shape[0]
    tg = scenes.make_targets(cam, d, info["depth_range"], 7)
    ctx = R.Context(0)
    dmap = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
    dtg = {k: torch.from_numpy(v).cuda() for k, v in tg.items()}
    grads = R.alloc_grads(dmap.n, dmap.d, dmap.K, device=0)
    H, W = cam["height"], cam["width"]
    imgs = {"rgb": torch.empty(H, W, 3, device="cuda"), "depth": torch.empty(H, W, device="cuda"),
            "feat": torch.empty(H, W, d, device="cuda"), "acc": torch.empty(H, W, device="cuda")}
    pose = torch.zeros(6, dtype=torch.float32, pin_memory=True)
    plan = R.Plan(dmap, cam, dtg, grads, images=imgs, pose_out=pose)
    for _ in range(reps):
        plan.run()
        plan.sync()
    torch.cuda.synchronize()
    print("plan ok", plan.launches, float(grads["flat"].abs().sum()), pose.tolist())


if __name__ == "__main__":
    main()
