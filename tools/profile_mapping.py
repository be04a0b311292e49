"""One mapping iteration at the headline config for ncu (python tools/profile_mapping.py [iters]):
render -> lgs_mapping_loss (SSIM + L1, masked depth, 16->64->32 decoder) -> backward -> Adam."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    scene, cams, info = scenes.make_config("c1_500k")
    cam = cams[0]
    H, W = cam["height"], cam["width"]
    ctx = R.Context(0)
    dm = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
    r = np.random.default_rng(11)
    kf = {"rgb": torch.from_numpy(r.uniform(0, 1, (H, W, 3)).astype(np.float32)).cuda(),
          "depth": torch.from_numpy(r.uniform(0.5, 6, (H, W)).astype(np.float32)).cuda(),
          "feat_gt": torch.from_numpy(r.normal(0, 0.5, (H, W, 32)).astype(np.float32)).cuda()}
    dec = tuple(torch.from_numpy(x).cuda() for x in scenes.make_decoder(32, 64, dm.d, 1))
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    opt = R.Adam(dm)
    ctx.profile(True)
    for _ in range(iters):
        out = R.render(dm, cam, ctx=ctx)
        br = R.mapping_loss(out, kf, dec)
        R.render_backward_loss(out, into=grads)
        opt.step(grads)
    torch.cuda.synchronize()
    for k, (ms, n) in ctx.phase_times().items():
        if n:
            print(f"{k:18s} {ms / n:8.4f} ms x{n}")
    print("loss", br)


if __name__ == "__main__":
    main()
