"""Wall time of the GPU language-pruning sweep on a cluttered 500k map vs a 500k map with random
features (no candidates: the spatial hash + candidate pass alone).  python tools/prune_timing.py"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2511_16144_b200 import pruning as P  # noqa: E402
from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402

for name, s in (("cluttered", scenes.make_prune_scene(500_000, seed=9, objects=600, extent=6.0)),
                ("random-features", scenes.make_config("c1_500k")[0])):
    dm = R.DeviceMap(s)
    P.find_language_redundant(dm)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        P.find_language_redundant(dm)
        ts.append(1e3 * (time.perf_counter() - t0))
    print(name, f"{min(ts):.2f} ms", P.prune_stats(dm))
