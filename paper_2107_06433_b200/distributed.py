"""Multi-GPU Sinkhorn-WMD: document columns sharded over ranks, one gather.

One process per GPU (``torch.distributed``; NCCL over NVLink/NVSwitch on the
B200 box, gloo on CPU for the tests).  The shard split is the reference's
``column_blocks`` (sparse.py:261-276): contiguous, nnz-balanced column ranges
that never split a column.  Columns are independent (test_acceptance.py:
212-222), so each rank runs the whole Sinkhorn loop on its block with the
embedding table (and hence K) replicated, and there is no data-path
collective until the end:

* one all-gather of the per-rank distance blocks (padded to equal length);
* one small all-gather of each rank's earliest degeneracy event, so every
  rank raises the same error the single-process solve would;
* with ``tol`` set, one 2-double all-reduce(MAX) per iteration (the global
  max-norm change and an any-failed flag), keeping ``converged`` and
  ``iterations_run`` global (solver.py:179-183).

Per-column arithmetic does not depend on the shard, so the gathered result is
bitwise identical for every world size.
"""

from __future__ import annotations

import time
from typing import Callable, Protocol

import numpy as np
import torch
import torch.distributed as dist

from .kernels import DegeneracyError, select_nonzero
from .solver import (DegEvent, ShardResult, SinkhornWorkspace, SolverConfig, SolverResult,
                     phase_timings)
from .sparse import SparseVector, column_blocks

__all__ = ["ShardSolver", "DeviceShardSolver", "shard_bounds", "sinkhorn_wmd_sharded",
           "merge_events"]


class ShardSolver(Protocol):
    def __call__(self, sel: np.ndarray, weights: np.ndarray, c0: int, c1: int,
                 config: SolverConfig, allreduce_max: Callable | None) -> ShardResult: ...


def shard_bounds(corpus, world: int) -> np.ndarray:
    """Column boundaries of the ``world`` shards (column_blocks semantics)."""
    if hasattr(corpus, "csc_compact"):
        col_ptr = corpus.csc_compact()[0]
    else:
        col_ptr = corpus.csc_index()[0]
    return column_blocks(col_ptr, world)


class DeviceShardSolver:
    """The GPU shard solver: this rank's column block resident on its device."""

    def __init__(self, corpus, embeddings, workspace: SinkhornWorkspace | None = None,
                 dev: torch.device | None = None):
        from .device import DeviceCorpus, DeviceEmbeddings, device

        self.corpus = corpus
        self.dev = dev or device()
        self.de = DeviceEmbeddings.of(embeddings, self.dev)
        self.ws = workspace or SinkhornWorkspace()
        self._blocks: dict[tuple[int, int], object] = {}

    def __call__(self, sel, weights, c0, c1, config, allreduce_max):
        from .device import DeviceCorpus
        from .solver import solve_on_device

        blk = self._blocks.get((c0, c1))
        if blk is None:
            if (c0, c1) == (0, self.corpus.n_cols):
                blk = DeviceCorpus.of(self.corpus, self.dev)
            else:   # upload only this rank's column block
                if hasattr(self.corpus, "csc_compact"):
                    cp, rows, vals = self.corpus.csc_compact()
                else:
                    cp, rows, _, vals = self.corpus.csc_index()
                blk = DeviceCorpus(self.corpus.n_rows, cp[c0: c1 + 1], rows, vals, self.dev,
                                   col_offset=c0, n_key=self.corpus.n_cols)
            self._blocks[(c0, c1)] = blk
        return solve_on_device(sel, weights, blk, self.de, config, self.ws,
                               allreduce_max=allreduce_max)


def merge_events(events: list[DegEvent | None]) -> DegEvent | None:
    """The event the single-process solve would raise: earliest code, then the
    reference's ordering inside one check ((i, j) row-major for zero
    denominators, (value, flat index) for the nonpositive-iterate check)."""
    live = [e for e in events if e is not None]
    if not live:
        return None
    return min(live, key=lambda e: (e.code, e.key))


def _comm_device(group) -> torch.device:
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def sinkhorn_wmd_sharded(query, corpus, embeddings, config: SolverConfig,
                         solver: ShardSolver | None = None, group=None) -> SolverResult:
    """``sinkhorn_wmd`` over all ranks of ``group``; every rank returns the full result."""
    t_start = time.perf_counter()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if isinstance(query, SparseVector):
        query = query.to_dense()
    query = np.asarray(query, dtype=np.float64)
    if query.shape != (corpus.n_rows,) or tuple(embeddings.shape)[0] != corpus.n_rows:
        raise ValueError(
            f"shape mismatch: query {query.shape}, embeddings "
            f"{tuple(embeddings.shape)}, corpus rows {corpus.n_rows}")
    t0 = time.perf_counter()
    sel, weights = select_nonzero(query)
    t_select = time.perf_counter() - t0
    bounds = shard_bounds(corpus, world)
    c0, c1 = int(bounds[rank]), int(bounds[rank + 1])
    if solver is None:
        solver = DeviceShardSolver(corpus, embeddings)
    cdev = _comm_device(group)

    def allreduce_max(v: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return t.cpu().numpy()

    res = solver(sel, weights, c0, c1, config, allreduce_max if config.tol is not None else None)

    # one gather of the distance blocks (padded to the largest block)
    width = int(np.max(np.diff(bounds))) if world else 0
    mine = torch.zeros(width + 1, dtype=torch.float64)
    mine[: c1 - c0] = torch.from_numpy(np.ascontiguousarray(res.wmd[: c1 - c0]))
    # the last slot carries this rank's iteration count (equal on all ranks)
    mine[width] = float(res.iterations)
    mine = mine.to(cdev)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)

    # one gather of the degeneracy events
    ev = res.event
    enc = np.full(4, np.inf)
    if ev is not None:
        enc[:] = [ev.code, *[float(k) for k in ev.key], rank]
    etens = torch.from_numpy(enc).to(cdev)
    eparts = [torch.empty_like(etens) for _ in range(world)]
    dist.all_gather(eparts, etens, group=group)
    evs = []
    for p in eparts:
        e = p.cpu().numpy()
        if np.isfinite(e[0]):
            evs.append(e)
    if evs:
        best = min(evs, key=lambda e: (e[0], e[1], e[2]))
        # the owning rank's message text; every rank reconstructs it
        code, k0, k1 = int(best[0]), best[1], best[2]
        if code % 2 == 0:
            msg = f"nonpositive iterate entry {float(k0)} at flat index {int(k1)}"
        else:
            msg = f"zero denominator at nonzero ({int(k0)}, {int(k1)})"
        raise DegeneracyError(msg)

    wmd = np.empty(corpus.n_cols, dtype=np.float64)
    for r, p in enumerate(parts):
        a, b = int(bounds[r]), int(bounds[r + 1])
        wmd[a:b] = p[: b - a].cpu().numpy()
    timings = phase_timings({"select": t_select, "total": time.perf_counter() - t_start},
                            res.timings)
    return SolverResult(wmd=wmd, iterations_run=res.iterations, converged=res.converged,
                        timings=timings)
