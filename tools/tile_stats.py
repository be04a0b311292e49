"""Per-tile work distribution of the headline workload (python tools/tile_stats.py [config]).

Prints, per 16x16 tile, the list length and the backward's traversal length (max n_contrib), and
the makespan a longest-first list scheduler reaches on the blend kernels' persistent grid, to see
whether the blend kernels are bound by their longest tiles."""
import heapq
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402


def lpt(costs, slots):
    h = [0.0] * slots
    for c in sorted(costs, reverse=True):
        t = heapq.heappop(h)
        heapq.heappush(h, t + c)
    return max(h)


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1_500k"
    scene, cams, info = scenes.make_config(cfg)
    cam = cams[0]
    dev = {k: torch.from_numpy(v).cuda() for k, v in scene.items()}
    out = R.render(dev, cam)
    torch.cuda.synchronize()
    _, _, ranges = out.tile_keys()
    ft, nc = out.pixel_state()
    H, W = cam["height"], cam["width"]
    ty, tx = (H + 15) // 16, (W + 15) // 16
    ncp = np.zeros((ty * 16, tx * 16), np.int64)
    ncp[:H, :W] = nc.reshape(H, W)
    tmax = ncp.reshape(ty, 16, tx, 16).max(axis=(1, 3)).ravel()
    tsum = ncp.reshape(ty, 16, tx, 16).sum(axis=(1, 3)).ravel()
    ranges = np.asarray(ranges).reshape(-1, 2)
    lens = (ranges[:, 1] - ranges[:, 0]).astype(np.int64)
    ftp = np.zeros((ty * 16, tx * 16), np.float32)
    ftp[:H, :W] = ft
    open_tile = (ftp.reshape(ty, 16, tx, 16).max(axis=(1, 3)).ravel() >= 1e-4)
    fwd = np.where(open_tile, lens, np.minimum(lens, tmax + 1))
    print("fwd traversal mean %.1f pct %s (tiles never saturating: %d)" % (
        fwd.mean(), np.percentile(fwd, [50, 90, 99, 100]).astype(int).tolist(), int(open_tile.sum())))
    pct = [50, 90, 99, 100]
    print("tiles", len(lens))
    print("list length   mean %.0f pct %s" % (lens.mean(), np.percentile(lens, pct).astype(int).tolist()))
    print("max n_contrib mean %.1f pct %s" % (tmax.mean(), np.percentile(tmax, pct).astype(int).tolist()))
    print("sum n_contrib mean %.0f pct %s" % (tsum.mean(), np.percentile(tsum, pct).astype(int).tolist()))
    for slots in (148 * 4, 148 * 5, 148 * 8):
        for name, c in (("max_nc", tmax.astype(float) + 1), ("sum_nc", tsum.astype(float) + 1),
                        ("fwd", fwd.astype(float) + 1)):
            ms = lpt(c, slots)
            print(f"slots {slots} cost {name}: LPT makespan / mean load = {ms / (c.sum() / slots):.3f}"
                  f"  (longest tile / mean load = {c.max() / (c.sum() / slots):.3f})")


if __name__ == "__main__":
    main()
