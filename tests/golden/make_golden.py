"""Regenerates the golden fixtures in this directory from oracle A (python tests/golden/make_golden.py).

The reference ships no golden vectors and cannot be built here, so these fixtures
pin the *restatement*: they were produced by oracle A after it passed every reference renderer test
(tests/test_oracle_reference.py), and tests/test_golden.py checks that the oracle (CPU) and the
CUDA path (GPU) still reproduce them.

  grad101.npz   the reference gradcheck scene make_grad_scene(12, 16, 8, 101)
                (gradcheck.hpp:31-78): images and all gradients for its fixed cotangent images.
  sh3_pose.npz  400 Gaussians, SH degree 3, d = 16, 64x48, rotated camera, L1 cotangents:
                images, gradients and the pose gradient (EXT features, parity unpinned by the
                reference).
  map_small.legomap  a 3-Gaussian LEGOMAP1 file (d = 4) written field by field with struct per
                proj/src/gaussian_map.cpp:196-218 (tests/test_map_io.py reads it through the C ABI).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as orc  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402
from tests.ref_scenes import make_grad_scene  # noqa: E402


def grad101():
    scene, cam, cfg, w_rgb, w_depth, w_feat = make_grad_scene(orc, 12, 16, 8, 101)
    s32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in scene.items()}
    out = orc.render(s32, cam, cfg)
    g = orc.render_backward(out, w_rgb, w_depth, w_feat)
    return dict(**{f"scene_{k}": np.asarray(v, np.float32) for k, v in scene.items()},
                w_rgb=w_rgb, w_depth=w_depth, w_feat=w_feat, rgb=out.rgb, depth=out.depth, feat=out.feat,
                acc=out.acc, **{f"g_{k}": v for k, v in g.items()},
                cfg=np.array([cfg.get("radius_sigma"), cfg.get("alpha_skip"), cfg.get("transmittance_min")]))


def sh3_pose():
    scene, cams, info = scenes.make_config("c1", n=400)
    base = dict(cams[0], width=64, height=48, fx=70.0, fy=70.0, cx=31.5, cy=23.5)
    cam = orc.perturb_pose(base, np.array([0.03, -0.02, 0.01, 0.05, -0.04, 0.2]))
    out = orc.render(scene, cam)
    tg = scenes.make_targets(cam, 16, info["depth_range"], 5)
    cot = scenes.l1_cotangents(out.rgb, out.depth, out.feat, tg)
    g = orc.render_backward(out, *cot, pose=True)
    return dict(**{f"scene_{k}": v for k, v in scene.items()}, cam_q=cam["q"], cam_t=cam["t"],
                cam_k=np.array([cam["fx"], cam["fy"], cam["cx"], cam["cy"], cam["width"], cam["height"]]),
                cot_rgb=cot[0], cot_depth=cot[1], cot_feat=cot[2], rgb=out.rgb, depth=out.depth, feat=out.feat,
                acc=out.acc, **{f"g_{k}": v for k, v in g.items()})


def map_small(path):
    import struct
    rows = [  # position, rotation (w, x, y, z), log-scale, opacity logit, colour, feature, anchor
        ((0.0, 0.0, 2.0), (1.0, 0.0, 0.0, 0.0), (-3.0, -3.0, -3.0), 0.0, (0.2, 0.4, 0.6), (1.0, 0.0, 0.0, 0.0), 0),
        ((1.5, -2.0, 3.25), (0.5, 0.5, 0.5, 0.5), (-2.5, -3.5, -4.0), 1.5, (1.0, 0.0, 0.5), (0.0, 1.0, 0.0, 0.0), 5),
        ((-1.0, 0.5, 4.0), (0.0, 0.0, 1.0, 0.0), (-1.0, -2.0, -3.0), -2.0, (0.1, 0.1, 0.1), (0.5, -0.5, 0.25, 1.0), 7),
    ]
    with open(path, "wb") as f:
        f.write(b"LEGOMAP1" + struct.pack("<IQ", 4, len(rows)))
        for p, q, s, o, c, ft, a in rows:
            f.write(struct.pack("<3f4f3ff3f4fQ", *p, *q, *s, o, *c, *ft, a))


if __name__ == "__main__":
    map_small(os.path.join(HERE, "map_small.legomap"))
    np.savez_compressed(os.path.join(HERE, "grad101.npz"), **grad101())
    np.savez_compressed(os.path.join(HERE, "sh3_pose.npz"), **sh3_pose())
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))
