import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2511_16144_b200 import renderer as R, scenes
for name in ("c1_500k", "c1", "c2", "c0"):
    scene, cams, info = scenes.make_config(name)
    cam = cams[0]
    ds = {k: torch.from_numpy(v).cuda() for k, v in scene.items()}
    lo = R.render(ds, cam, ctx=R.Context(0)); fo = R.render(ds, cam, ctx=R.Context(0, full_lists=True))
    torch.cuda.synchronize()
    _, _, lr = lo.tile_keys(); _, _, fr = fo.tile_keys()
    ll = lr[:, 1] - lr[:, 0]; fl = fr[:, 1] - fr[:, 0]
    print(name, "tiles", len(ll), "complete-list tiles (pass 2 or layer A covers all)", int((ll == fl).sum()),
          "of which nonempty", int(((ll == fl) & (fl > 0)).sum()), "stats", lo.stats())
