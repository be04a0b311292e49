import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2511_16144_b200 import renderer as R, scenes
scene, cams, info = scenes.make_config("c1_500k")
cam = cams[0]
tg = scenes.make_targets(cam, 16, info["depth_range"], 7)
stream = torch.cuda.Stream()
ctx = R.Context(0, stream=stream.cuda_stream)
with torch.cuda.stream(stream):
    dm = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
    dtg = {k: torch.from_numpy(v).cuda() for k, v in tg.items()}
    grads = R.alloc_grads(dm.n, dm.d, dm.K, device=0)
    pose = torch.zeros(6, dtype=torch.float32, pin_memory=True)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    rows = []
    for k in range(30):
        flush.fill_(float(k))
        t0 = time.perf_counter()
        out = R.render(dm, cam, targets=dtg, ctx=ctx)
        t1 = time.perf_counter()
        R.render_backward_loss_async(out, into=grads, pose_out=pose)
        t2 = time.perf_counter()
        stream.synchronize()
        t3 = time.perf_counter()
        del out
        t4 = time.perf_counter()
        rows.append((1e3*(t1-t0), 1e3*(t2-t1), 1e3*(t3-t2), 1e3*(t4-t3)))
    # no-flush variant: pure host enqueue rate
    for r in rows[5:15]:
        print("render %.3f  bwd %.3f  wait %.3f  del %.3f" % r)
