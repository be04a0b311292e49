"""Host-side timing of the e2e leg (bench.py run_e2e): per-call wall times of one thread's step
(render with a host-mapped map + host images, backward into host gradients, loss readback), and
the per-step time with 1..4 concurrent threads.  python tools/e2e_timing.py"""
import os
import sys
import threading
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_16144_b200 import renderer as R, scenes  # noqa: E402


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


MAPPED = os.environ.get("E2E_MAPPED", "1") != "0"
scene, cams, info = scenes.make_config("c1_500k")
cam = cams[0]
tg = scenes.make_targets(cam, 16, info["depth_range"], 7)
hs = {k: pinned(v) for k, v in scene.items()}
ht = {k: pinned(v) for k, v in tg.items()}
H, W, n, K, d = cam["height"], cam["width"], scene["pos"].shape[0], 16, 16


class Worker:
    def __init__(self):
        self.ctx = R.Context(0, stream="own")
        self.img = {"rgb": pinned(np.zeros((H, W, 3))), "depth": pinned(np.zeros((H, W))),
                    "feat": pinned(np.zeros((H, W, d))), "acc": pinned(np.zeros((H, W)))}
        self.flat = pinned(np.zeros(n * (11 + 3 * K + d)))
        self.grads = R.alloc_grads(n, d, K, flat=self.flat)

    def step(self, t=None):
        t0 = time.perf_counter()
        out = R.render(hs, cam, targets=ht, ctx=self.ctx, out=self.img, host_mapped=MAPPED)
        t1 = time.perf_counter()
        R.render_backward_l1(out, pose=True, into=self.grads)
        t2 = time.perf_counter()
        out.l1_loss()
        t3 = time.perf_counter()
        del out
        t4 = time.perf_counter()
        if t is not None:
            t.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3))


ws = [Worker() for _ in range(4)]
for w in ws:
    w.step()
    w.step()
torch.cuda.synchronize()
rows = []
for _ in range(10):
    ws[0].step(rows)
print("1 thread, ms per call: render %.2f  backward %.2f  loss %.2f  free %.2f" %
      tuple(1e3 * np.median([r[i] for r in rows]) for i in range(4)))
for nt in (1, 2, 3, 4):
    steps = 10

    def loop(w):
        for _ in range(steps):
            w.step()

    ths = [threading.Thread(target=loop, args=(w,)) for w in ws[:nt]]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{nt} threads: {1e3 * dt / (steps * nt):.2f} ms per step")
