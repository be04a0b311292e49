"""Probe: per-view plan status and replay time of the c3 multi-view batch (speculative or not,
device ms per replay, phase times of a profiling copy).  Usage: python tools/probe_c3.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402

scene, cams, info = scenes.make_config("c3")
n, d, K = scene["pos"].shape[0], scene["feat"].shape[0], scene["sh"].shape[1]
ctx = R.Context(0)
dmap = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
tgs = [{k: torch.from_numpy(v).cuda() for k, v in scenes.make_targets(c, d, info["depth_range"], 50 + v).items()}
       for v, c in enumerate(cams)]
grads = R.alloc_grads(n, d, K, device=0)
for acc in (False, True):
    for v, c in enumerate(cams[:3]):
        p = R.Plan(dmap, c, tgs[v], grads, accumulate=acc)
        ts = []
        for _ in range(5):
            p.run()
            p.sync()
            ts.append(p.elapsed_ms())
        out = R.render(dmap, c, targets=tgs[v], ctx=ctx)
        st = out.stats()
        p.set_profiling(True)
        p.run()
        p.sync()
        print(f"view {v} accumulate={acc} speculative={p.speculative} ms={min(ts):.4f} layer_div={ctx.layer_div} "
              f"pairs={st['pairs']} listed={st['listed']} phases={ {k: round(x, 4) for k, x in p.phase_times().items()} }")
