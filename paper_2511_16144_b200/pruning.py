"""Map pruning on the resident map: the SPEC's [MODULE] pruning over lgs_prune*.

The reference ships only a placeholder (proj/src/pruning.cpp:1); the operations, defaults and
invariants here are the SPEC's:

* ``find_language_redundant(map, cfg)`` -- Eq. 4: Gaussians in ascending ID; a
  live G_i queries its ``k_neighbors`` nearest live neighbours (the reference KD-tree's order,
  kdtree.hpp:36-55) and marks each G_j closer than ``tau_dist`` with cos(f_i, f_j) > ``tau_sim``;
  marked Gaussians are dead at once (greedy, order-deterministic).  Runs on the GPU as exact
  parallel dependency rounds (csrc/prune.cu).
* ``find_geometric(map, cfg)`` -- SPEC.md:496-503: opacity < ``alpha_min`` or max(exp(s)) >
  ``scale_max``.
* ``prune(map, cfg, adam=None, ids=None)`` -- SPEC.md:505-509: deletes the union, compacts the Adam
  moments with it, survivors keep their order (and their IDs: ``ids`` are filtered alongside).

IDs are the map's row indices unless ``ids`` (the caller's stable IDs, one per row) is given.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import LGS_MEM_HOST, check
from .renderer import Adam, DeviceMap


@dataclass
class PruneConfig:
    """SPEC.md:475-478 (PruneConfig): defaults K = 8, tau_dist 0.02 m, tau_sim 0.9, alpha_min 0.05,
    scale_max 0.5 m, every 200 mapping iterations (``period``: the caller's schedule)."""
    k_neighbors: int = 8
    tau_dist: float = 0.02
    tau_sim: float = 0.9
    alpha_min: float = 0.05
    scale_max: float = 0.5
    period: int = 200

    def __post_init__(self):
        # SPEC.md:477 invariants (the library checks them again and raises ValueError)
        if not (-1.0 < self.tau_sim <= 1.0):
            raise ValueError("tau_sim must be in (-1, 1]")
        if not self.tau_dist > 0:
            raise ValueError("tau_dist must be > 0")
        if self.period < 1:
            raise ValueError("period must be >= 1")

    def c(self) -> _lib.LgsPruneConfig:
        return _lib.LgsPruneConfig(int(self.k_neighbors), float(self.tau_dist), float(self.tau_sim),
                                   float(self.alpha_min), float(self.scale_max))


@dataclass
class PruneReport:
    """the two removal sets (IDs) and the survivor count."""
    removed_language: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    removed_geometric: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    kept: int = 0
    surviving_ids: np.ndarray | None = None


def _flags_call(fn, dmap: DeviceMap, cfg: PruneConfig | None) -> np.ndarray:
    cfg = cfg or PruneConfig()
    flags = np.zeros(max(dmap.n, 1), np.uint8)
    count = C.c_int64()
    check(fn(dmap.ctx.h, dmap.h, C.byref(cfg.c()), flags.ctypes.data, LGS_MEM_HOST, C.byref(count)))
    return np.flatnonzero(flags[:dmap.n]).astype(np.int64)


def find_language_redundant(dmap: DeviceMap, cfg: PruneConfig | None = None) -> np.ndarray:
    """Row indices the Eq. 4 sweep marks, ascending."""
    return _flags_call(_lib.load().lgs_find_language_redundant, dmap, cfg)


def find_geometric(dmap: DeviceMap, cfg: PruneConfig | None = None) -> np.ndarray:
    """Row indices failing the geometric criteria, ascending."""
    return _flags_call(_lib.load().lgs_find_geometric, dmap, cfg)


def prune_stats(dmap: DeviceMap) -> dict:
    """Work of the last language sweep on the map's context: candidates (Gaussians with a similar
    neighbour inside tau_dist) and the dependency rounds the GPU sweep took."""
    cand, rounds = C.c_int64(), C.c_int64()
    check(_lib.load().lgs_prune_stats(dmap.ctx.h, C.byref(cand), C.byref(rounds)))
    return {"candidates": int(cand.value), "rounds": int(rounds.value)}


def prune(dmap: DeviceMap, cfg: PruneConfig | None = None, adam: Adam | None = None, ids=None) -> PruneReport:
    """Delete the union of both rules from the map (and the Adam moments).  Renders and plans made
    on the map before are invalid afterwards (the library refuses them)."""
    cfg = cfg or PruneConfig()
    n = dmap.n
    ids = np.arange(n, dtype=np.int64) if ids is None else np.asarray(ids, np.int64)
    if ids.shape != (n,):
        raise ValueError(f"ids must have one entry per Gaussian ({n})")
    fl = np.zeros(max(n, 1), np.uint8)
    fg = np.zeros(max(n, 1), np.uint8)
    kept = C.c_int64()
    if adam is not None and adam.map is not dmap:
        raise ValueError("adam belongs to another map")
    check(_lib.load().lgs_prune(dmap.ctx.h, dmap.h, adam.h if adam is not None else None, C.byref(cfg.c()),
                                fl.ctypes.data, fg.ctypes.data, LGS_MEM_HOST, C.byref(kept)))
    fl, fg = fl[:n].astype(bool), fg[:n].astype(bool)
    dmap.n = int(kept.value)
    return PruneReport(removed_language=ids[fl], removed_geometric=ids[fg], kept=int(kept.value),
                       surviving_ids=ids[~(fl | fg)])
