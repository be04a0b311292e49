"""Tensor-core backward (blend_bwd_mma.cu): pins the mma.sync TF32 fragment layouts and checks that
the tensor-core kernel and the SIMT shuffle-reduction kernel produce the same gradients."""
import os

import numpy as np
import pytest

from tests.parity import GROUPS, grad_mismatch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2511_16144_b200 import _lib  # noqa: E402
from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402


@pytest.mark.parametrize("split", [0, 1])
def test_mma_fragment_layout(split):
    rng = np.random.default_rng(3)
    a = rng.standard_normal((16, 8)).astype(np.float32)
    b = rng.standard_normal((8, 8)).astype(np.float32)
    d = np.zeros((16, 8), np.float32)
    _lib.check(_lib.load().lgs_debug_mma_selftest(0, a.ctypes.data, b.ctypes.data, d.ctypes.data, split))
    ref = a.astype(np.float64) @ b.astype(np.float64)
    err = np.abs(d - ref).max() / np.abs(ref).max()
    # plain TF32 (10-bit mantissa) vs the 3xTF32 split (~fp32)
    assert err < (2e-3 if split == 0 else 2e-6), err


def _grads(impl, scene, cam, tg):
    os.environ["LGS_BWD_IMPL"] = impl  # "mma" opts into the tensor-core kernel
    try:
        dev = {k: torch.from_numpy(v).cuda() for k, v in scene.items()}
        out = R.render(dev, cam, targets={k: torch.from_numpy(v).cuda() for k, v in tg.items()})
        return R.render_backward_l1(out, pose=True)
    finally:
        os.environ.pop("LGS_BWD_IMPL", None)


@pytest.mark.parametrize("name,n", [("c0", None), ("c1", 50_000), ("c4", 60_000)])
def test_mma_backward_matches_simt(name, n):
    scene, cams, info = scenes.make_config(name, n=n)
    cam = cams[0]
    tg = scenes.make_targets(cam, 16, info["depth_range"], 13)
    g_mma = _grads("mma", scene, cam, tg)
    g_simt = _grads("simt", scene, cam, tg)
    for k in GROUPS:
        frac, worst = grad_mismatch(g_mma[k], g_simt[k])
        assert frac < 1e-3, (k, frac, worst)  # same allowance as the oracle parity tests
    # the pose gradient sums every Gaussian; near-zero components carry cancellation noise
    # (L1 cotangents: every Gaussian's term is O(1) while the sum is small), so compare as a 6-vector
    a, b = (np.asarray(g["pose"], np.float64) for g in (g_mma, g_simt))
    assert np.linalg.norm(a - b) <= 1e-2 * np.linalg.norm(b), (a, b)
