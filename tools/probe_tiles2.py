"""Probe (experiment build -DLGS_EXP_TILEPROF only): resident fused-blend CTAs per SM in three
launch settings -- a writing plan (side branch: zero rows + tile order), an accumulating plan (no
side branch), an uncaptured fused render -- at c1_500k."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_16144_b200 import _lib  # noqa: E402
from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402

scene, cams, info = scenes.make_config("c1_500k")
cam = cams[0]
nt = ((cam["width"] + 15) // 16) * ((cam["height"] + 15) // 16)
L = _lib.load()
L.lgs_exp_tile_prof.argtypes = [C.c_void_p, C.c_int]


def resident(tag):
    buf = np.zeros((nt, 6), dtype=np.uint64)
    L.lgs_exp_tile_prof(buf.ctypes.data, nt)
    p = buf.astype(np.int64)
    st, en = (p[:, 0] - p[:, 0].min()) / 1e3, (p[:, 1] - p[:, 0].min()) / 1e3
    ts = np.linspace(0, en.max(), 9)[1:-1]
    print(tag, "span %.1f us" % en.max(), "active tiles:", [int(((st <= t) & (en > t)).sum()) for t in ts])


for mode in ("plan", "plan_acc", "eager"):
    ctx = R.Context(0, fused_eager=(mode == "eager"))
    dm = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
    tg = {k: torch.from_numpy(v).cuda() for k, v in scenes.make_targets(cam, dm.d, info["depth_range"], 7).items()}
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    if mode == "eager":
        for _ in range(4):
            out = R.render(dm, cam, targets=tg, ctx=ctx)
            torch.cuda.synchronize()
    else:
        plan = R.Plan(dm, cam, tg, grads, accumulate=(mode == "plan_acc"))
        for _ in range(4):
            plan.run()
            plan.sync()
    resident(mode)
