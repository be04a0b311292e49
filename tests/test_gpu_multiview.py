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


def _simulated_exchange(dmap, grads_list, cap=0):
    import ctypes as C
    from paper_2511_16144_b200 import _lib
    structs = [R._grads_struct(g, False) for g in grads_list]
    arr = (C.POINTER(_lib.LgsMapGrads) * len(structs))(*[C.pointer(s) for s in structs])
    rows, ovf = C.c_int64(), C.c_int32()
    st = _lib.load().lgs_debug_sparse_reduce_simulated(dmap.ctx.h, dmap.h, arr, len(structs), cap, C.byref(rows),
                                                       C.byref(ovf))
    return (st, rows.value, ovf.value) if cap else (st, rows.value)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sparse_exchange_simulated_ranks_equals_dense_sum(world):
    """The world > 1 path of lgs_allreduce_grads_sparse (scan, count all-gather, pack, record
    all-gather, zero + rank-ordered add) over `world` ranks simulated on one GPU: every rank ends with
    the dense sum over ranks -- bit for bit the fp32 sum taken in rank order -- and all ranks are
    identical.  Each rank holds real per-view gradients (different c3 views), so rows overlap
    partially across ranks."""
    # the full c3 map: its views saturate on a few thousand Gaussians (sparse rows)
    ctx, dmap, cams, tgs = _setup(nviews=world if world <= 8 else 8, n=500_000)
    per_rank = []
    for r in range(world):
        g = R.alloc_grads(dmap.n, dmap.d, dmap.K, device=0)
        out = R.render(dmap, cams[r % len(cams)], targets=tgs[r % len(cams)], ctx=ctx)
        R.render_backward_l1(out, into=g)
        per_rank.append(g)
    torch.cuda.synchronize()
    dense = torch.zeros_like(per_rank[0]["flat"])
    for g in per_rank:  # ((0 + g0) + g1) + ...: the exchange's order
        dense = dense + g["flat"]
    st, rows = _simulated_exchange(dmap, per_rank)
    torch.cuda.synchronize()
    assert st == 0, st
    assert rows > 1
    for g in per_rank:
        assert torch.equal(g["flat"], dense)


def _per_rank_grads(world, n=500_000):
    ctx, dmap, cams, tgs = _setup(nviews=min(world, 8), n=n)
    per_rank = []
    for r in range(world):
        g = R.alloc_grads(dmap.n, dmap.d, dmap.K, device=0)
        out = R.render(dmap, cams[r % len(cams)], targets=tgs[r % len(cams)], ctx=ctx)
        R.render_backward_l1(out, into=g)
        per_rank.append(g)
    torch.cuda.synchronize()
    return dmap, per_rank


def test_sparse_exchange_capacity_speculative():
    """The host-wait-free form (lgs_allreduce_grads_sparse_async): record blocks of a fixed capacity.
    With room for every rank's rows it equals the exact exchange bit for bit; when a rank has more
    rows than the capacity the kernels see it in the gathered counts and change nothing (each rank
    keeps its own gradient), reporting the overflow and the largest count for the exact re-run."""
    world = 4
    dmap, per_rank = _per_rank_grads(world)
    before = [g["flat"].clone() for g in per_rank]
    dense = torch.zeros_like(before[0])
    for b in before:
        dense = dense + b
    st, rows, ovf = _simulated_exchange(dmap, per_rank, cap=8)  # far too small
    torch.cuda.synchronize()
    assert st == 0 and ovf == 1 and rows > 8
    for g, b in zip(per_rank, before):
        assert torch.equal(g["flat"], b)
    st, rows2, ovf = _simulated_exchange(dmap, per_rank, cap=rows + rows // 4)
    torch.cuda.synchronize()
    assert st == 0 and ovf == 0 and rows2 == rows
    for g in per_rank:
        assert torch.equal(g["flat"], dense)


def test_sparse_exchange_simulated_refuses_dense_rows():
    ctx, dmap, cams, tgs = _setup(nviews=1, n=4_000)
    per_rank = [R.alloc_grads(dmap.n, dmap.d, dmap.K, device=0) for _ in range(2)]
    for g in per_rank:
        g["flat"].fill_(1.0)  # every row nonzero: the real exchange takes the dense all-reduce
    st, rows = _simulated_exchange(dmap, per_rank)
    assert st == 1 and rows == -1
