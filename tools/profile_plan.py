"""The bench's captured step for ncu launch lists (python tools/profile_plan.py [config] [replays]).

Creates the plan (one eager warm-up step inside), then replays it `replays` times; with
`ncu --metrics gpu__time_duration.sum` the replayed kernels give the per-kernel split of exactly
the step bench.py times.  Prints the plan's own per-replay device time."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1_500k"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    scene, cams, info = scenes.make_config(cfg)
    cam = cams[0]
    stream = torch.cuda.Stream()
    ctx = R.Context(0, stream=stream.cuda_stream)
    with torch.cuda.stream(stream):
        dm = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
        tg = {k: torch.from_numpy(v).cuda()
              for k, v in scenes.make_targets(cam, dm.d, info["depth_range"], 7).items()}
        grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
        pose = torch.zeros(6, dtype=torch.float32, pin_memory=True)
        plan = R.Plan(dm, cam, tg, grads, pose_out=pose)
        ms = []
        for _ in range(reps):
            plan.run()
            plan.sync()
            ms.append(plan.elapsed_ms())
    print("plan launches", plan.launches, "ms per replay", [round(x, 4) for x in ms])
    with torch.cuda.stream(stream):
        plan.set_profiling(True)
        plan.run()
        plan.sync()
    print("phases of a profiling replay (ms):", {k: round(v, 4) for k, v in plan.phase_times().items()},
          "total", round(plan.elapsed_ms(), 4))


if __name__ == "__main__":
    main()
