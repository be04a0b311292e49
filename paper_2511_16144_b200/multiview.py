"""Multi-keyframe mapping batches sharded one view per GPU (BASELINE configs 3-4).

The Gaussian map is replicated on every rank; each rank renders its views forward + backward and
accumulates the per-Gaussian fp32 gradients of all of its views into ONE flat buffer
(lgs_map_grads with accumulate = 1); a single all-reduce (sum) over NCCL / NVLink then produces
the batch gradient on every rank.  The gradient is a sum over pixels of all views, so any
partition of the views is valid and the same all-reduce sums it.

The reference has no multi-view or distributed path at all (it is single-threaded CPU code,
SURVEY.md §2 "Parallelism strategies"); this module is the B200-side extension named in
BASELINE.json configs 3-4.
"""
from __future__ import annotations

from typing import Callable, Sequence


def assign_views(n_views: int, world: int, rank: int, costs: Sequence[float] | None = None) -> list[int]:
    """Views owned by ``rank``.  Without costs: round-robin.  With per-view cost estimates (e.g. the
    pair counts P of a previous step): deterministic longest-processing-time-first greedy, which
    bounds the slowest rank at 4/3 of optimal -- the imbalance, not the all-reduce, is what limits
    8-GPU efficiency on the multi-view configs (SURVEY.md §7 hard part 7)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if costs is None:
        return [v for v in range(n_views) if v % world == rank]
    if len(costs) != n_views:
        raise ValueError("one cost per view")
    order = sorted(range(n_views), key=lambda v: (-float(costs[v]), v))
    load = [0.0] * world
    owner = [0] * n_views
    for v in order:
        r = min(range(world), key=lambda q: (load[q], q))
        owner[v] = r
        load[r] += float(costs[v])
    return [v for v in range(n_views) if owner[v] == rank]


class NativeComm:
    """The library's own NCCL communicator on a rasterizer context (lgs_comm_* in include/lgs.h).

    The 128-byte NCCL id made by rank 0 is shipped to the other ranks over the process group
    (``torch.distributed`` with any backend -- gloo here, nccl on the box -- is only the bootstrap);
    the gradient all-reduce itself is enqueued by liblgs.so on the context's stream, so a mapping
    step (render -> backward -> all-reduce) never leaves the C ABI."""

    def __init__(self, ctx, group=None, world: int | None = None, rank: int | None = None):
        import ctypes as C

        from . import _lib

        self.ctx = ctx
        L = _lib.load()
        if world is None:
            import torch.distributed as dist

            world, rank = dist.get_world_size(group), dist.get_rank(group)
            cid = _lib.LgsCommId()
            payload = [None]
            if rank == 0:
                _lib.check(L.lgs_comm_unique_id(C.byref(cid)))
                payload = [bytes(cid.bytes)]
            dist.broadcast_object_list(payload, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            C.memmove(cid.bytes, payload[0], 128)
        else:  # single process (world 1) or an id exchanged by the caller
            cid = _lib.LgsCommId()
            _lib.check(L.lgs_comm_unique_id(C.byref(cid)))
        _lib.check(L.lgs_comm_init(ctx.h, int(world), int(rank or 0), C.byref(cid)))
        self.world, self.rank = int(world), int(rank or 0)

    def all_reduce(self, flat):
        """In-place fp32 sum over ranks of a contiguous CUDA tensor, on the context's stream."""
        from . import _lib

        assert flat.is_cuda and flat.dtype.is_floating_point and flat.is_contiguous()
        _lib.check(_lib.load().lgs_allreduce_f32(self.ctx.h, flat.data_ptr(), flat.numel()))

    def all_reduce_grads(self, dmap, grads):
        from . import _lib
        from .renderer import _grads_struct

        gs = _grads_struct(grads, False)
        _lib.check(_lib.load().lgs_allreduce_grads(self.ctx.h, dmap.h, gs))

    def all_reduce_grads_sparse(self, dmap, grads) -> int:
        """lgs_allreduce_grads_sparse: the dense sum, exchanging only the nonzero rows.  Returns the
        largest per-rank row count (-1: fell back to the dense all-reduce)."""
        import ctypes as C

        from . import _lib
        from .renderer import _grads_struct

        gs = _grads_struct(grads, False)
        rows = C.c_int64()
        _lib.check(_lib.load().lgs_allreduce_grads_sparse(self.ctx.h, dmap.h, C.byref(gs), C.byref(rows)))
        return rows.value

    def all_reduce_grads_sparse_async(self, dmap, grads):
        """lgs_allreduce_grads_sparse_async: the same sum enqueued without a host wait (capacity-sized
        row blocks); call ``wait_grads_sparse`` after the step."""
        from . import _lib
        from .renderer import _grads_struct

        self._pending = _grads_struct(grads, False)
        _lib.check(_lib.load().lgs_allreduce_grads_sparse_async(self.ctx.h, dmap.h, self._pending))

    def wait_grads_sparse(self, dmap, grads) -> int:
        """Completes an async sparse exchange (re-running it exactly if a rank outgrew the capacity);
        returns the largest per-rank row count."""
        import ctypes as C

        from . import _lib
        from .renderer import _grads_struct

        gs = getattr(self, "_pending", None) or _grads_struct(grads, False)
        rows = C.c_int64()
        _lib.check(_lib.load().lgs_allreduce_grads_sparse_wait(self.ctx.h, dmap.h, gs, C.byref(rows)))
        self._pending = None
        return rows.value

    def set_timeout(self, ms: int):
        """Bound the host waits inside collectives (lgs_comm_set_timeout)."""
        from . import _lib

        _lib.check(_lib.load().lgs_comm_set_timeout(self.ctx.h, int(ms)))

    def close(self):
        from . import _lib

        if getattr(self, "ctx", None) is not None:
            _lib.check(_lib.load().lgs_comm_destroy(self.ctx.h))
            self.ctx = None


class MultiViewStep:
    """One data-parallel mapping step: local views fwd+bwd into a flat gradient, then all-reduce.

    ``view_grads(view, grads, accumulate)`` renders one view and adds its gradients into ``grads``
    (the rasterizer path below, or any callable with that contract -- the CPU gloo tests plug in
    the oracle to exercise the sharding / reduction logic without a GPU).
    """

    def __init__(self, views: Sequence[int], view_grads: Callable, grads: dict, group=None, comm=None):
        self.views = list(views)
        self.view_grads = view_grads
        self.grads = grads
        self.group = group
        self.comm = comm  # NativeComm: the library's NCCL all-reduce; None: torch.distributed

    def step(self):
        import torch.distributed as dist

        flat = self.grads["flat"]
        flat.zero_()
        for v in self.views:
            self.view_grads(v, self.grads, True)
        if self.comm is not None:
            self.comm.all_reduce(flat)
        elif dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group)
        return self.grads


def rasterizer_view_grads(dmap, cams, targets, ctx=None, pose_out: dict | None = None):
    """view_grads callable backed by the sm_100a rasterizer (fused L1 loss per view)."""
    from . import renderer as R

    def fn(v, grads, accumulate):
        out = R.render(dmap, cams[v], targets=targets[v], ctx=ctx)
        g = R.render_backward_l1(out, pose=pose_out is not None, into=grads, accumulate=accumulate)
        if pose_out is not None:
            pose_out[v] = g.pop("pose")
        return out

    return fn


def sparse_sum_reference(rows_per_rank):
    """Host restatement of lgs_allreduce_grads_sparse's merge (sparse_reduce.cu) for tests: given,
    per rank, a dense [N][R] gradient, every rank's nonzero rows are zeroed and then re-added rank
    by rank in rank order.  Returns the merged dense array (equal to the plain sum)."""
    import numpy as np

    out = np.array(rows_per_rank[0], dtype=np.float32, copy=True)
    lists = [np.nonzero(np.any(g != 0, axis=1))[0] for g in rows_per_rank]
    for idx in lists:
        out[idx] = 0.0
    for g, idx in zip(rows_per_rank, lists):
        out[idx] = out[idx] + g[idx]
    return out


def sparse_all_reduce_host(dense, group=None, cap=0):
    """lgs_allreduce_grads_sparse's exchange over torch.distributed on host arrays (any backend;
    the gloo tests run it): nonzero rows of a [N][R] float32 array are all-gathered as (index,
    row) records and merged like sparse_sum_reference (listed rows zeroed, ranks added in rank
    order), in place.  Returns the largest per-rank row count.  cap > 0: the capacity-speculative
    form (lgs_allreduce_grads_sparse_async): record blocks of ``cap`` rows; if any rank has more
    rows, nothing is merged and -(largest count) is returned."""
    import numpy as np
    import torch
    import torch.distributed as dist

    idx = np.nonzero(np.any(dense != 0, axis=1))[0]
    world = dist.get_world_size(group)
    cnt = torch.tensor([idx.size], dtype=torch.int64)
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    maxc = int(max(c.item() for c in counts))
    block = cap if cap > 0 else maxc
    rec = torch.zeros(block, dense.shape[1] + 1, dtype=torch.float32)
    k = min(idx.size, block)  # the pack kernel writes at most `block` records
    rec[:k, 0] = torch.from_numpy(idx[:k].astype(np.int32).view(np.float32))
    rec[:k, 1:] = torch.from_numpy(dense[idx[:k]])
    recs = [torch.zeros_like(rec) for _ in range(world)]
    dist.all_gather(recs, rec, group=group)
    if maxc > block:  # some rank overflowed the capacity: every rank keeps its own gradient
        return -maxc
    lists = [r[:int(c.item()), 0].numpy().view(np.int32) for r, c in zip(recs, counts)]
    for li in lists:
        dense[li] = 0.0
    for r, c, li in zip(recs, counts, lists):
        dense[li] += r[:int(c.item()), 1:].numpy()
    return maxc
