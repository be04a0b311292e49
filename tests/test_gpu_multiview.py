"""Multi-view mapping step on the GPU through the library's own NCCL communicator (lgs_comm_*).

Only one GPU is available to the tests, so the communicator runs at world size 1 (NCCL refuses two
ranks on one device); the sharding and the sum across ranks are covered at world size 2 by the gloo
tests (test_multiview_gloo.py).  Here: the all-reduce path is wired through the C ABI, leaves a
1-rank sum unchanged, handles split attribute buffers, and a MultiViewStep equals the sum of its
per-view gradients."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2511_16144_b200 import multiview  # noqa: E402
from paper_2511_16144_b200 import renderer as R  # noqa: E402
from paper_2511_16144_b200 import scenes  # noqa: E402
from tests.parity import GROUPS, grad_mismatch  # noqa: E402


def _setup(nviews=3, n=20_000):
    scene, cams, info = scenes.make_config("c3", n=n)
    cams = cams[:nviews]
    ctx = R.Context(0)
    dmap = R.DeviceMap({k: torch.from_numpy(v).cuda() for k, v in scene.items()}, ctx)
    tgs = [{k: torch.from_numpy(v).cuda() for k, v in scenes.make_targets(c, dmap.d, info["depth_range"], 50 + i).items()}
           for i, c in enumerate(cams)]
    return ctx, dmap, cams, tgs


def test_native_comm_world1_step_equals_sum_of_views():
    ctx, dmap, cams, tgs = _setup()
    comm = multiview.NativeComm(ctx, world=1, rank=0)
    grads = R.alloc_grads(dmap.n, dmap.d, dmap.K, device=0)
    step = multiview.MultiViewStep(range(len(cams)), multiview.rasterizer_view_grads(dmap, cams, tgs, ctx=ctx), grads,
                                   comm=comm)
    step.step()
    torch.cuda.synchronize()
    ref = R.alloc_grads(dmap.n, dmap.d, dmap.K, device=0)
    for v in range(len(cams)):
        out = R.render(dmap, cams[v], targets=tgs[v], ctx=ctx)
        ref["flat"] += R.render_backward_l1(out)["flat"]
    torch.cuda.synchronize()
    assert ref["flat"].abs().max().item() > 0
    # atomic accumulation order differs between runs: the 1e-3 gradient bound of tests/parity.py,
    # with the same allowance for cancellation-dominated components as the oracle parity test
    for k in GROUPS:
        frac, worst = grad_mismatch(grads[k], ref[k])
        assert frac < 1e-3, (k, frac, worst)
    comm.close()


def test_native_comm_allreduce_grads_split_buffers():
    ctx, dmap, cams, tgs = _setup(nviews=1)
    comm = multiview.NativeComm(ctx, world=1, rank=0)
    out = R.render(dmap, cams[0], targets=tgs[0], ctx=ctx)
    g = R.render_backward_l1(out)
    split = {k: g[k].clone() for k in ("position", "rotation", "log_scale", "opacity_logit", "sh", "feature")}
    comm.all_reduce_grads(dmap, split)  # six separate buffers: one grouped NCCL launch
    comm.all_reduce_grads(dmap, g)      # one flat buffer: one call
    torch.cuda.synchronize()
    for k, v in split.items():
        assert torch.equal(v, g[k]), k
    comm.close()
    with pytest.raises(ValueError):
        comm2 = multiview.NativeComm.__new__(multiview.NativeComm)
        comm2.ctx = ctx
        comm2.all_reduce(g["flat"])  # lgs_comm_destroy'd context: LGS_EINVAL


def test_sparse_gradient_exchange_world1():
    """lgs_allreduce_grads_sparse at world size 1: the scan / pack / zero / add kernels run (the
    rows of the only rank) and must reproduce the gradient bit for bit; the row count is the number
    of Gaussians with a nonzero gradient (a few thousand with the depth-layered binning)."""
    ctx, dmap, cams, tgs = _setup(nviews=2)
    comm = multiview.NativeComm(ctx, world=1, rank=0)
    grads = R.alloc_grads(dmap.n, dmap.d, dmap.K, device=0)
    for v in range(2):
        out = R.render(dmap, cams[v], targets=tgs[v], ctx=ctx)
        R.render_backward_l1(out, into=grads, accumulate=v > 0)
    torch.cuda.synchronize()
    before = grads["flat"].clone()
    nz_rows = 0
    for k in ("position", "rotation", "log_scale", "opacity_logit", "sh"):
        g = grads[k].reshape(dmap.n, -1)
        nz = g.ne(0).any(dim=1)
        nz_rows = nz if isinstance(nz_rows, int) else nz_rows | nz
    nz_rows = nz_rows | grads["feature"].reshape(-1, dmap.n).ne(0).any(dim=0)
    rows = comm.all_reduce_grads_sparse(dmap, grads)
    torch.cuda.synchronize()
    assert rows == int(nz_rows.sum().item())
    assert 0 < rows < dmap.n
    assert torch.equal(grads["flat"], before)
    comm.close()
