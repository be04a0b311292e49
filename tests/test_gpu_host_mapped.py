"""LGS_MEM_HOST_MAPPED maps (include/lgs.h): a page-locked host scene whose SH rows and features
are read in place for just the listed Gaussians renders exactly like a device map -- bitwise
images, gradients within the atomic-order bound -- with the depth-layered binning (lazy colour and
feature fetch) and with complete lists (every feature gathered); after a render of the same host
map that listed many of its Gaussians the next one copies the SH / feature blocks in bulk instead
(same results); Adam and download refuse such a map, and pageable memory is rejected."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402
from paper_2511_16144_b200._lib import LgsError  # noqa: E402
from tests.parity import GROUPS, grad_mismatch  # noqa: E402


def _pinned(a):
    t = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


@pytest.mark.parametrize("full", [False, True])
@pytest.mark.parametrize("name,n", [("c1", 40_000), ("c0", None)])
def test_host_mapped_renders_like_device_map(name, n, full):
    scene, cams, info = scenes.make_config(name, n=n)
    cam = cams[0]
    tg = scenes.make_targets(cam, scene["feat"].shape[0], info["depth_range"], 3)
    ctx = R.Context(0, full_lists=full)
    dtg = {k: torch.from_numpy(v).cuda() for k, v in tg.items()}
    dev = R.render({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, cam, targets=dtg, ctx=ctx)
    gd = R.render_backward_l1(dev, pose=True)
    hs = {k: _pinned(v) for k, v in scene.items()}
    htg = {k: _pinned(v) for k, v in tg.items()}
    host = R.render(hs, cam, targets=htg, ctx=ctx, host_mapped=True)
    assert host._map.host_mapped
    gh = R.render_backward_l1(host, pose=True)
    torch.cuda.synchronize()
    for k in ("rgb", "depth", "feat", "acc"):
        assert np.array_equal(getattr(host, k), getattr(dev, k).cpu().numpy()), k
    for k in GROUPS:
        frac, worst = grad_mismatch(gh[k], gd[k])
        assert frac < 1e-3, (k, frac, worst)
    assert np.allclose(gh["pose"], gd["pose"], rtol=1e-4, atol=1e-5 * np.abs(gd["pose"]).max())


def test_host_mapped_bulk_copy_policy():
    # c1 at 200k: 139 of 1200 tiles take the second layered pass and ~20% of the Gaussians get
    # listed, so the second render of the same host map is done from a bulk copy (host_rows == 0);
    # c1_500k-like saturation (few listed) stays zero-copy
    scene, cams, info = scenes.make_config("c1")
    cam = cams[0]
    tg = scenes.make_targets(cam, scene["feat"].shape[0], info["depth_range"], 3)
    hs = {k: _pinned(v) for k, v in scene.items()}
    htg = {k: _pinned(v) for k, v in tg.items()}
    ctx = R.Context(0)
    outs, grads = [], []
    for _ in range(3):
        o = R.render(hs, cam, targets=htg, ctx=ctx, host_mapped=True)
        grads.append(R.render_backward_l1(o, pose=True))
        outs.append(o)
    st = [o.stats() for o in outs]
    print("\nhost rows per render", [x["host_rows"] for x in st], "active", st[0]["active"])
    assert st[0]["host_rows"] == st[0]["active"] > scene["pos"].shape[0] // 64
    assert st[1]["host_rows"] == 0 and st[2]["host_rows"] == 0
    for o in outs[1:]:
        for k in ("rgb", "depth", "feat", "acc"):
            assert np.array_equal(getattr(o, k), getattr(outs[0], k)), k
    for g in grads[1:]:
        for k in GROUPS:
            frac, worst = grad_mismatch(g[k], grads[0][k])
            assert frac < 1e-3, (k, frac, worst)
    small, scams, _ = scenes.make_config("c1_500k")
    hsm = {k: _pinned(v) for k, v in small.items()}
    # (the first render after c1 starts from c1's tile-list capacity and lists more: its count may
    # select one bulk render; the policy settles on zero-copy from the next count on)
    rs = [R.render(hsm, scams[0], ctx=ctx, host_mapped=True).stats() for _ in range(3)]
    assert rs[2]["host_rows"] == rs[2]["active"] == 2547, rs


def test_host_mapped_rejections():
    scene, cams, _ = scenes.make_config("c0", n=2000)
    ctx = R.Context(0)
    with pytest.raises(LgsError, match="page-locked"):  # pageable numpy arrays
        R.DeviceMap({k: np.ascontiguousarray(v) for k, v in scene.items()}, ctx, host_mapped=True)
    dm = R.DeviceMap({k: _pinned(v) for k, v in scene.items()}, ctx, host_mapped=True)
    with pytest.raises(LgsError, match="HOST_MAPPED"):
        R.Adam(dm)
