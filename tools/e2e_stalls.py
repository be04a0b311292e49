"""Per-step wall times of bench.py's e2e workers (3 host threads, own contexts): where do the
occasional multi-ms steps come from?  python tools/e2e_stalls.py [threads] [steps]"""
import os, sys, threading, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2511_16144_b200 import renderer as R, scenes

def pinned(a):
    t = torch.empty(a.shape, dtype=torch.float32, pin_memory=True); t.numpy()[...] = a; return t.numpy()

nth = int(sys.argv[1]) if len(sys.argv) > 1 else 3
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
scene, cams, info = scenes.make_config("c1_500k")
cam = cams[0]
tg = scenes.make_targets(cam, 16, info["depth_range"], 7)
hs = {k: pinned(v) for k, v in scene.items()}
htg = {k: pinned(v) for k, v in tg.items()}
n, d, K = scene["pos"].shape[0], 16, scene["sh"].shape[1]
H, W = cam["height"], cam["width"]

class Worker:
    def __init__(self):
        self.img = {"rgb": pinned(np.zeros((H, W, 3), np.float32)), "depth": pinned(np.zeros((H, W), np.float32)),
                    "feat": pinned(np.zeros((H, W, d), np.float32)), "acc": pinned(np.zeros((H, W), np.float32))}
        self.flat = pinned(np.zeros(n * (11 + 3 * K + d), np.float32))
        self.grads = R.alloc_grads(n, d, K, flat=self.flat)
        self.ctx = R.Context(0, stream="own", host_grad_delta=os.environ.get("DELTA", "1") == "1")
        self.t = []
    def step(self):
        t0 = time.perf_counter()
        out = R.render(hs, cam, targets=htg, ctx=self.ctx, out=self.img, host_mapped=os.environ.get("MAPPED", "1") == "1")
        t1 = time.perf_counter()
        R.render_backward_l1(out, pose=True, into=self.grads)
        t2 = time.perf_counter()
        out.l1_loss()
        t3 = time.perf_counter()
        self.t.append((t1 - t0, t2 - t1, t3 - t2))

ws = [Worker() for _ in range(nth)]
for w in ws:
    w.step(); w.step(); w.t.clear()
torch.cuda.synchronize()
import gc, os
if os.environ.get("NOGC"):
    gc.collect()
    gc.disable()
ths = [threading.Thread(target=lambda w=w: [w.step() for _ in range(steps)]) for w in ws]
t0 = time.perf_counter()
for t in ths: t.start()
for t in ths: t.join()
dt = time.perf_counter() - t0
print(f"{nth} threads: {nth * steps / dt:.1f} it/s")
for i, w in enumerate(ws):
    a = np.array(w.t) * 1e3
    print(i, "render ms p50/max", np.percentile(a[:, 0], 50).round(2), a[:, 0].max().round(1),
          "bwd", np.percentile(a[:, 1], 50).round(2), a[:, 1].max().round(1), "loss", a[:, 2].max().round(2))
    slow = np.nonzero(a.sum(1) > 10)[0]
    print("   slow steps", slow.tolist()[:10], a[slow].round(1).tolist()[:4])
