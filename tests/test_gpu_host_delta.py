"""Host-gradient delta mode (LGS_OPT_HOST_GRAD_DELTA): host MapGradients buffers reused across
backwards are rewritten row-sparse, yet hold the dense gradient after every call -- also when the
nonzero rows move between calls (different views) and rows nonzero before become zero.  (Compared
with a dense backward of a separate render: same nonzero rows, values within the atomic-order
bound.)"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402
from tests.parity import GROUPS, grad_mismatch  # noqa: E402


def _row_nonzero(g, n):
    nz = np.zeros(n, bool)
    for k in GROUPS:
        a = g[k]
        nz |= (a != 0).reshape(-1, n).any(axis=0) if k == "feature" else (a.reshape(n, -1) != 0).any(axis=1)
    return nz


def test_delta_host_grads_equal_dense():
    scene, cams, info = scenes.make_config("c3", n=200_000)
    d, K, n = scene["feat"].shape[0], scene["sh"].shape[1], scene["pos"].shape[0]
    dense_ctx = R.Context(0, stream="own")
    delta_ctx = R.Context(0, stream="own", host_grad_delta=True)
    host = R.alloc_grads(n, d, K)  # numpy: host buffers, reused by every delta backward
    moved = []
    for step, v in enumerate([0, 3, 3, 5, 0]):
        cam = cams[v]
        tg = scenes.make_targets(cam, d, info["depth_range"], 100 + step)
        ref = R.alloc_grads(n, d, K)
        out = R.render(scene, cam, targets=tg, ctx=dense_ctx)
        R.render_backward_l1(out, into=ref)
        b0 = delta_ctx.transfer_bytes()[1]
        out2 = R.render(scene, cam, targets=tg, ctx=delta_ctx)
        b1 = delta_ctx.transfer_bytes()[1]
        R.render_backward_l1(out2, into=host)
        moved.append(delta_ctx.transfer_bytes()[1] - b1)
        # the same rows nonzero (stale rows of an earlier view would show here) and the values within
        # the atomic-order bound of tests/parity.py (two separate backwards)
        assert np.array_equal(_row_nonzero(host, n), _row_nonzero(ref, n)), f"step {step}: nonzero rows differ"
        for k in GROUPS:
            frac, worst = grad_mismatch(host[k], ref[k])
            assert frac < 1e-3, (step, k, frac, worst)
        assert b1 > b0  # the images came back
    dense_bytes = host["flat"].nbytes
    assert moved[0] >= dense_bytes  # the first call writes densely
    assert max(moved[1:]) < dense_bytes / 20, moved  # then only the nonzero rows
