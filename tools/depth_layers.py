"""How deep into the global depth order each tile's blending actually goes
(python tools/depth_layers.py [config]).

For a cut at depth-order rank R (the R nearest visible Gaussians), prints the share of tile pairs
the nearest R Gaussians own and the share of tiles whose every pixel saturates (T < T_min) on
Gaussians of rank < R -- i.e. how much of the binning a depth-layered pipeline would skip."""
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
    scene, cams, info = scenes.make_config(cfg)
    cam = cams[0]
    out = R.render({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, cam)
    torch.cuda.synchronize()
    keys, vals, ranges = out.tile_keys()
    ft, nc = out.pixel_state()
    pr = out.projected()
    vis = pr["visible"].astype(bool)
    n = vis.shape[0]
    depth = pr["depth"].astype(np.float32).view(np.uint32)
    idx = np.nonzero(vis)[0]
    order = idx[np.lexsort((idx, depth[idx]))]
    rank = np.full(n, -1, np.int64)
    rank[order] = np.arange(order.size)
    V = order.size
    H, W = cam["height"], cam["width"]
    ty, tx = (H + 15) // 16, (W + 15) // 16
    ranges = np.asarray(ranges).reshape(-1, 2)
    # per tile: rank of the deepest Gaussian any of its pixels uses, and whether all pixels saturate
    ncp = np.zeros((ty * 16, tx * 16), np.int64)
    ncp[:H, :W] = nc.reshape(H, W)
    ftp = np.ones((ty * 16, tx * 16), np.float32)
    ftp[:H, :W] = ft.reshape(H, W)
    tmax = ncp.reshape(ty, 16, tx, 16).max(axis=(1, 3)).ravel()
    sat = (ftp.reshape(ty, 16, tx, 16) < 1e-4).all(axis=(1, 3)).ravel()
    need = np.full(tmax.size, V, np.int64)
    for t in range(tmax.size):
        b, e = ranges[t]
        if tmax[t] > 0 and sat[t]:
            need[t] = rank[vals[b + tmax[t] - 1]] + 1
        elif e == b:
            need[t] = 0
    tiles_per = np.zeros(V, np.int64)
    np.add.at(tiles_per, rank[vals], 1)
    cum_pairs = np.cumsum(tiles_per)
    P = cum_pairs[-1]
    print(f"visible {V}, pairs {P}, tiles {tmax.size}, saturating tiles {int(sat.sum())}")
    for frac in (0.005, 0.01, 0.02, 0.05, 0.1, 0.2, 0.5):
        Rk = max(1, int(frac * V))
        done = float((need <= Rk).mean())
        print(f"cut at {100 * frac:5.1f}% of visible (rank {Rk:7d}, depth {np.frombuffer(depth[order[Rk - 1]].tobytes(), np.float32)[0]:.3f}):"
              f" pairs {100 * cum_pairs[Rk - 1] / P:5.1f}%  tiles done {100 * done:5.1f}%")
    print("tile need-rank percentiles (% of V):", np.percentile(need / V * 100, [50, 90, 99, 100]).round(2).tolist())


if __name__ == "__main__":
    main()
