"""Diagnostic: pose gradient of the tensor-core and SIMT backward kernels vs the fp64 oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as orc  # noqa: E402
from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 60000
    scene, cams, info = scenes.make_config(name, n=n)
    cam = cams[0]
    tg = scenes.make_targets(cam, 16, info["depth_range"], 13)
    pre = orc.preprocess_f32(scene, cam)
    ref = orc.render(scene, cam, inject=pre)
    cot = scenes.l1_cotangents(ref.rgb, ref.depth, ref.feat, tg)
    g_ref = orc.render_backward(ref, *cot, pose=True)
    print("oracle pose", g_ref["pose"])
    for impl in ("mma", "simt"):
        os.environ["LGS_BWD_IMPL"] = impl
        dev = {k: torch.from_numpy(v).cuda() for k, v in scene.items()}
        out = R.render(dev, cam)
        g = R.render_backward(None, out, *(torch.from_numpy(c.astype(np.float32)).cuda() for c in cot), pose=True)
        rel = np.abs(g["pose"] - g_ref["pose"]) / np.abs(g_ref["pose"])
        print(impl, g["pose"], "rel err", rel)
        for k in ("position", "rotation", "log_scale", "opacity_logit", "feature"):
            a = g[k].cpu().numpy().astype(np.float64).ravel()
            b = g_ref[k].ravel()
            rms = np.sqrt(np.mean(b * b))
            e = np.abs(a - b) / (np.abs(b) + 0.01 * rms)
            print("   ", k, "max err", float(e.max()), "frac>1e-3", float((e > 1e-3).mean()))


if __name__ == "__main__":
    main()
