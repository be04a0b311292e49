"""One headline fwd+bwd step for ncu / compute-sanitizer (python tools/profile_step.py [config] [steps] [view]).

Runs `steps` identical steps of bench.py's workload (fused L1, pose gradient) on cuda:0 and
prints per-phase times and work counters, so an ncu capture of the same command can be matched
to the phases."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1_500k"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    scene, cams, info = scenes.make_config(cfg)
    cam = cams[int(sys.argv[3]) if len(sys.argv) > 3 else (8 if cfg == "c4" else 0)]  # bench.py default_view
    d = scene["feat"].shape[0]
    tg = scenes.make_targets(cam, d, info["depth_range"], 7)
    stream = torch.cuda.Stream()
    # FUSED=1: the fused forward+backward kernel of the captured step, uncaptured (LGS_OPT_FUSED_EAGER)
    ctx = R.Context(0, stream=stream.cuda_stream, fused_eager=os.environ.get("FUSED", "0") == "1")
    with torch.cuda.stream(stream):
        dmap = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
        dtg = {k: torch.from_numpy(v).cuda() for k, v in tg.items()}
        grads = R.alloc_grads(dmap.n, dmap.d, dmap.K, device=0)
        ctx.profile(True)
        for _ in range(steps):
            out = R.render(dmap, cam, targets=dtg, ctx=ctx)
            R.render_backward_l1(out, pose=True, into=grads)
    torch.cuda.synchronize()
    for k, (ms, n) in ctx.phase_times().items():
        if n:
            print(f"{k:18s} {ms / n:8.4f} ms x{n}")
    print("stats", out.stats(), "launches", ctx.launches)
    if os.environ.get("FUSED", "0") != "1":  # the fused kernel keeps no work counters / pixel tape
        print("work", out.work())
        ft, nc = out.pixel_state()
        H, W = cam["height"], cam["width"]
        pad = np.zeros(((H + 15) // 16 * 16, (W + 15) // 16 * 16), nc.dtype)
        pad[:H, :W] = nc
        tiles = pad.reshape(pad.shape[0] // 16, 16, pad.shape[1] // 16, 16).max(axis=(1, 3))
        print("sum over tiles of max n_contrib:", int(tiles.sum()), "mean:", float(tiles.mean()))


if __name__ == "__main__":
    main()
