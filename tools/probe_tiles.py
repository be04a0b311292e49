"""Probe (experiment build -DLGS_EXP_TILEPROF only): per-tile start / end (globaltimer), cycles,
SM, list length and consumed prefix of the fused blend in a captured replay, saved to
gpurun_out/tiles_<config>.npz.  Usage: python tools/probe_tiles.py c1_500k [c2 ...]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_16144_b200 import _lib  # noqa: E402
from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402

for name in sys.argv[1:]:
    scene, cams, info = scenes.make_config(name)
    cam = cams[8 if name == "c4" else 0]
    ctx = R.Context(0)
    dm = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
    tg = {k: torch.from_numpy(v).cuda() for k, v in scenes.make_targets(cam, dm.d, info["depth_range"], 7).items()}
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    plan = R.Plan(dm, cam, tg, grads)
    for _ in range(6):
        plan.run()
        plan.sync()
    nt = ((cam["width"] + 15) // 16) * ((cam["height"] + 15) // 16)
    buf = np.zeros((nt, 6), dtype=np.uint64)
    L = _lib.load()
    L.lgs_exp_tile_prof.argtypes = [C.c_void_p, C.c_int]
    rc = L.lgs_exp_tile_prof(buf.ctypes.data, nt)
    np.savez(f"gpurun_out/tiles_{name}.npz", prof=buf, ms=plan.elapsed_ms())
    print(name, rc, nt, plan.elapsed_ms())
