"""GPU side of the map-file path (lgs_map_load / lgs_map_save) and the insertion coverage mask
(lgs_coverage_mask) against the float32 oracle rule (oracle/loss.py coverage_mask)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import loss as OL  # noqa: E402
from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402
from tests.test_map_io import py_write  # noqa: E402


def _sh0_scene(n=3000):
    scene, cams, info = scenes.make_config("c0", n=n)
    q = scene["rot"].astype(np.float64)
    scene["rot"] = (q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32)
    return scene, cams[0], info


@pytest.mark.parametrize("n", [3000, 3001])  # n % 4 != 0: the download staging
def test_map_load_renders_like_the_scene(tmp_path, n):
    scene, cam, _ = _sh0_scene(n)
    p = str(tmp_path / "m.legomap")
    py_write(p, scene, np.zeros(scene["pos"].shape[0], np.uint64))
    dm = R.map_load(p)
    a = R.render(dm, cam)
    back, _ = R.map_file_read(p)
    b = R.render({k: torch.from_numpy(v).cuda() for k, v in back.items()}, cam)
    torch.cuda.synchronize()
    assert torch.equal(a.rgb, b.rgb) and torch.equal(a.feat, b.feat) and torch.equal(a.depth, b.depth)
    q = str(tmp_path / "m2.legomap")
    R.map_save(dm, q, anchors=np.arange(dm.n, dtype=np.uint64))
    again, anchors = R.map_file_read(q)
    assert list(anchors[:3]) == [0, 1, 2]
    for k in back:
        assert np.array_equal(again[k], back[k]), k


def test_coverage_mask_matches_rule():
    scene, cam, info = _sh0_scene(6000)
    out = R.render({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, cam)
    H, W = cam["height"], cam["width"]
    r = np.random.default_rng(2)
    depth = out.depth.cpu().numpy()
    meas = (depth * r.choice([1.0, 1.02, 1.2], size=(H, W))).astype(np.float32)
    meas[r.uniform(size=(H, W)) < 0.1] = 0.0
    meas[0, :5] = np.nan
    want = OL.coverage_mask(out.acc.cpu().numpy(), depth, meas)
    mask, cnt = R.coverage_mask(out, meas)              # host depth -> host mask
    dmask, dcnt = R.coverage_mask(out, torch.from_numpy(meas).cuda())  # device in / out
    assert np.array_equal(mask, want) and cnt == int(want.sum())
    assert np.array_equal(dmask.cpu().numpy(), want) and dcnt == cnt
    assert 0 < cnt < H * W
    with pytest.raises(ValueError):
        R.coverage_mask(out, meas[:, :-1])
