"""Multi-view data-parallel mapping step (multiview.py) on CPU: world size 2 over gloo.

Each rank owns a subset of the views, accumulates their gradients into one flat buffer and the
buffer is all-reduced once; the result must equal the single-process sum over all views.  The
per-view gradients here come from the oracle (CPU) so the sharding and reduction logic is tested
without a GPU; on the GPU the same MultiViewStep runs with rasterizer_view_grads and NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_16144_b200 import multiview, scenes


def test_assign_views_round_robin_and_lpt():
    assert multiview.assign_views(8, 2, 0) == [0, 2, 4, 6]
    assert multiview.assign_views(8, 2, 1) == [1, 3, 5, 7]
    costs = [10, 1, 1, 1, 1, 1, 1, 4]
    owned = [multiview.assign_views(8, 2, r, costs) for r in range(2)]
    assert sorted(owned[0] + owned[1]) == list(range(8))
    loads = [sum(costs[v] for v in o) for o in owned]
    assert max(loads) == 10  # the heavy view alone on one rank, everything else on the other
    with pytest.raises(ValueError):
        multiview.assign_views(8, 2, 2)


def _views():
    scene, cams, info = scenes.make_config("c3", n=600)
    small = []
    for c in cams[:4]:
        small.append(dict(c, width=48, height=36, fx=43.3, fy=43.3, cx=23.5, cy=17.5))
    return scene, small, info


def _oracle_view_grads(scene, cams, info):
    from oracle import oracle as orc
    from paper_2511_16144_b200.renderer import alloc_grads  # noqa: F401  (layout helper only)

    def fn(v, grads, accumulate):
        out = orc.render(scene, cams[v])
        tg = scenes.make_targets(cams[v], 16, info["depth_range"], 100 + v)
        g = orc.render_backward(out, *scenes.l1_cotangents(out.rgb, out.depth, out.feat, tg))
        for k in ("position", "rotation", "log_scale", "opacity_logit", "sh", "feature"):
            grads[k] += torch.from_numpy(g[k].astype(np.float32))

    return fn


def _flat_grads(n, d, K):
    from paper_2511_16144_b200.renderer import alloc_grads
    return alloc_grads(n, d, K, flat=torch.zeros(n * (11 + 3 * K + d)))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene, cams, info = _views()
    n, d, K = scene["pos"].shape[0], scene["feat"].shape[0], scene["sh"].shape[1]
    grads = _flat_grads(n, d, K)
    step = multiview.MultiViewStep(multiview.assign_views(len(cams), world, rank), _oracle_view_grads(scene, cams, info),
                                   grads)
    g = step.step()
    q.put((rank, g["flat"].numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_allreduce_equals_single_process_sum():
    scene, cams, info = _views()
    n, d, K = scene["pos"].shape[0], scene["feat"].shape[0], scene["sh"].shape[1]
    ref = _flat_grads(n, d, K)
    fn = _oracle_view_grads(scene, cams, info)
    for v in range(len(cams)):
        fn(v, ref, True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = ref["flat"].numpy()
    scale = float(np.abs(want).max())
    for r in range(2):
        # fp32 sums in a different order (v0+v2, v1+v3, then the all-reduce): rounding only
        assert np.allclose(res[r], want, rtol=1e-5, atol=1e-6 * scale)
    assert np.array_equal(res[0], res[1])


def _sparse_worker(rank, world, port, q, caps=(0,)):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for cap in caps:
        dense = _sparse_rank_grads(rank)
        maxc = multiview.sparse_all_reduce_host(dense, cap=cap)
        out.append((dense.copy(), maxc))
    q.put((rank, out[0][0], out[0][1]) if len(caps) == 1 else (rank, out))
    dist.barrier()
    dist.destroy_process_group()


def _sparse_rank_grads(rank, n=5000, R=75):
    """a rank's view gradient with the layered binning's shape: a few hundred nonzero rows,
    overlapping between ranks"""
    rng = np.random.default_rng(100 + rank)
    g = np.zeros((n, R), np.float32)
    rows = np.unique(np.concatenate([rng.choice(n, 300, replace=False), np.arange(40)]))
    g[rows] = rng.standard_normal((rows.size, R)).astype(np.float32)
    return g


def test_sparse_gradient_exchange_equals_dense_sum():
    """lgs_allreduce_grads_sparse's exchange (nonzero rows as (index, row) records, merged in rank
    order) restated over gloo at world size 3: equal to the dense sum, bitwise identical on every
    rank, and the same as the single-process merge (multiview.sparse_sum_reference)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sparse_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, dense, maxc = q.get(timeout=300)
        res[r] = (dense, maxc)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    per_rank = [_sparse_rank_grads(r) for r in range(world)]
    want = np.sum(per_rank, axis=0, dtype=np.float64)
    merged = multiview.sparse_sum_reference(per_rank)
    for r in range(world):
        dense, maxc = res[r]
        assert maxc == max(int(np.any(g != 0, axis=1).sum()) for g in per_rank)
        assert np.array_equal(dense, res[0][0])
        assert np.array_equal(dense, merged)
        assert np.allclose(dense, want, rtol=1e-5, atol=1e-6)


def test_sparse_exchange_capacity_overflow_changes_nothing():
    """The capacity-speculative form (lgs_allreduce_grads_sparse_async) at world size 3: a capacity
    below some rank's row count leaves every rank's gradient as it was and reports the count; a
    sufficient capacity gives the exact exchange's result."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    caps = (50, 1000)
    procs = [ctx.Process(target=_sparse_worker, args=(r, world, port, q, caps)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out = q.get(timeout=300)
        res[r] = out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    per_rank = [_sparse_rank_grads(r) for r in range(world)]
    rows = max(int(np.any(g != 0, axis=1).sum()) for g in per_rank)
    merged = multiview.sparse_sum_reference(per_rank)
    for r in range(world):
        (d_small, m_small), (d_big, m_big) = res[r]
        assert m_small == -rows and np.array_equal(d_small, per_rank[r])
        assert m_big == rows and np.array_equal(d_big, merged)
