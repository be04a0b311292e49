"""Per-phase device times after warm-up (python tools/ab_phases.py [config] [steps]): for A/B runs of
kernel variants selected by environment knobs.  5 untimed warm-up steps, then `steps` profiled
steps with a 512 MiB L2 flush before each; prints the mean per phase."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1_500k"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    scene, cams, info = scenes.make_config(cfg)
    cam = cams[0]
    tg = scenes.make_targets(cam, scene["feat"].shape[0], info["depth_range"], 7)
    stream = torch.cuda.Stream()
    ctx = R.Context(0, stream=stream.cuda_stream)
    with torch.cuda.stream(stream):
        dm = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
        dtg = {k: torch.from_numpy(v).cuda() for k, v in tg.items()}
        grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
        for k in range(5 + steps):
            if k == 5:
                torch.cuda.synchronize()
                ctx.profile(True)
            flush.fill_(float(k))
            out = R.render(dm, cam, targets=dtg, ctx=ctx)
            R.render_backward_l1(out, into=grads)
        torch.cuda.synchronize()
    tot = 0.0
    for k, (ms, n) in ctx.phase_times().items():
        if n:
            print(f"{k:18s} {ms / steps:8.4f} ms")
            tot += ms / steps
    print(f"{'sum':18s} {tot:8.4f} ms")


if __name__ == "__main__":
    main()
