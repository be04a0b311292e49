"""Regenerates the REFERENCE golden fixtures (python tests/golden/make_ref_golden.py).

Unlike make_golden.py (oracle A outputs), these come from the reference itself: its unmodified
renderer.cpp / geometry.cpp compiled by oracle/Makefile into oracle/_ref/liblgs_ref.so (against the
self-written Eigen subset in oracle/eigen_shim, since Eigen3 is absent here).  /root/reference does
not exist on the GPU box, so the GPU tests read these committed vectors instead of the library.

  ref_grad101.npz  the reference's own gradcheck scene make_grad_scene(12, 16, 8, 101)
                   (gradcheck.hpp:31-78), exactly as the reference build draws it, rounded to fp32:
                   lego::render images and lego::render_backward gradients for its weight images.
  ref_c0.npz       configs[0] (160x120, SH0, d = 16) at 4000 Gaussians (scenes.make_config("c0"),
                   fp32 inputs): lego::render images, and lego::render_backward gradients for the L1
                   cotangents of the reference's own images against the seed-7 targets, stored as
                   fp32 (the GPU bounds are 1e-4 / 1e-3); the depth order and contributor counts.
  ref_prune.npz    the SPEC's language-pruning sweep (Eq. 4) run on the reference's own KdTree3
                   (kdtree.hpp; oracle/ref_bridge.cpp ref_find_language_redundant) over
                   scenes.make_prune_scene(PRUNE_N, seed=11, coherent=c) for the PRUNE_CASES
                   (coherent, k, tau_dist, tau_sim): flags per case, bit-packed.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402

C0_N = 4000
PRUNE_N = 6000
PRUNE_CASES = [(True, 8, 0.02, 0.9), (False, 8, 0.02, 0.9), (True, 1, 0.02, 0.9), (True, 32, 0.05, 0.5),
               (False, 4, 0.03, 0.0), (True, 8, 0.02, -0.5)]


def ref_grad101():
    scene, cam, cfg, w_rgb, w_depth, w_feat = ref.grad_scene(12, 16, 8, 101)
    s32 = {k: np.asarray(v, np.float32).astype(np.float64) for k, v in scene.items()}
    out = ref.render(s32, cam, cfg)
    g = ref.render_backward(out, w_rgb, w_depth, w_feat)
    return dict(**{f"scene_{k}": np.asarray(v, np.float32) for k, v in scene.items()},
                w_rgb=w_rgb, w_depth=w_depth, w_feat=w_feat, rgb=out.rgb, depth=out.depth, feat=out.feat,
                acc=out.acc, **{f"g_{k}": v for k, v in g.items()},
                cfg=np.array([cfg["radius_sigma"], cfg["alpha_skip"], cfg["transmittance_min"]]))


def ref_c0():
    scene, cams, info = scenes.make_config("c0", n=C0_N)
    cam = cams[0]
    tg = scenes.make_targets(cam, scene["feat"].shape[0], info["depth_range"], 7)
    out = ref.render(scene, cam)
    cot = scenes.l1_cotangents(out.rgb, out.depth, out.feat, tg)
    g = ref.render_backward(out, *cot)
    f32 = lambda a: np.asarray(a, np.float32)  # noqa: E731 (fp32 storage: the GPU bounds are 1e-4 / 1e-3)
    return dict(rgb=f32(out.rgb), depth=f32(out.depth), feat=f32(out.feat), acc=f32(out.acc),
                **{f"g_{k}": f32(v) for k, v in g.items()},
                order=out.sorted_indices().astype(np.int32), contribs=out.contrib_counts().astype(np.int16))


def ref_prune():
    out = {"cases": np.array(PRUNE_CASES, np.float64)}
    for ci, (coh, k, td, ts) in enumerate(PRUNE_CASES):
        scene = scenes.make_prune_scene(PRUNE_N, seed=11, coherent=bool(coh))
        out[f"flags{ci}"] = np.packbits(ref.find_language_redundant(scene, int(k), td, ts))
    return out


def main():
    if not ref.available():
        raise SystemExit("oracle/_ref/liblgs_ref.so is not built (make -C oracle, needs /root/reference)")
    np.savez_compressed(os.path.join(HERE, "ref_grad101.npz"), **ref_grad101())
    np.savez_compressed(os.path.join(HERE, "ref_c0.npz"), **ref_c0())
    np.savez_compressed(os.path.join(HERE, "ref_prune.npz"), **ref_prune())


if __name__ == "__main__":
    main()
