"""Multi-GPU Sinkhorn-WMD: document columns sharded over ranks, one gather.

One process per GPU (``torch.distributed``; NCCL over NVLink/NVSwitch on the
B200 box, gloo on CPU for the tests).  The shard split is the reference's
``column_blocks`` (sparse.py:261-276): contiguous, nnz-balanced column ranges
that never split a column.  Columns are independent (test_acceptance.py:
212-222), so each rank runs the whole Sinkhorn loop on its block with the
embedding table (and hence K) replicated, and there is no data-path
collective until the end:

* one ``all_gather_into_tensor`` of equal per-rank slots — the distance
  block (padded to the widest block), the block's raw device error record,
  the iteration count and the converged flag.  On the GPU the solve writes
  its distances and error record straight into the slot, so nothing crosses
  PCIe before the gather and the result comes back in one device->host copy;
* only if some rank recorded a degeneracy, one more small all-gather of each
  rank's decoded earliest event, so every rank raises the same error the
  single-process solve would;
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
    """The GPU shard solver: this rank's column block resident on its device.

    ``__call__`` is the ShardSolver protocol (host result).  ``solve_into``
    is the device path ``sinkhorn_wmd_sharded`` uses: the solve writes its
    distances straight into the rank's slot of the gather buffer and the raw
    error record next to them, so nothing crosses PCIe before the gather.
    """

    def __init__(self, corpus, embeddings, workspace: SinkhornWorkspace | None = None,
                 dev: torch.device | None = None):
        from .device import DeviceEmbeddings, device

        self.corpus = corpus
        self.dev = dev or device()
        self.de = DeviceEmbeddings.of(embeddings, self.dev)
        self.ws = workspace or SinkhornWorkspace()
        self._blocks: dict[tuple[int, int], object] = {}

    def block(self, c0: int, c1: int):
        """This rank's column block, uploaded once (only its columns)."""
        from .device import DeviceCorpus

        blk = self._blocks.get((c0, c1))
        if blk is None:
            blk = DeviceCorpus.block_of(self.corpus, self.dev, c0, c1)
            self._blocks[(c0, c1)] = blk
        return blk

    def __call__(self, sel, weights, c0, c1, config, allreduce_max):
        from .solver import solve_on_device

        return solve_on_device(sel, weights, self.block(c0, c1), self.de, config, self.ws,
                               allreduce_max=allreduce_max)

    def solve_into(self, sel, weights, c0, c1, config, allreduce_max, slot: torch.Tensor,
                   query: np.ndarray | None = None):
        """Solve the block with ``slot[:c1-c0]`` (float64, on this device) as
        the distance buffer and the error record written to
        ``slot[width:width+4]`` (int64 bits).  Returns (iterations,
        converged, decode, spans) — ``decode(err_words)`` yields the block's
        DegEvent, ``spans(gathered_slot)`` the device phase times.

        tol unset and a dense float64 query: the native per-query runtime
        (one C call: select, one CUDA-graph launch, results left in the slot,
        phase stamps copied next to them) — nothing is synchronised before the
        caller's all-gather."""
        from .solver import QueryPlan, _device_spans, _Events, _native_plan

        dc = self.block(c0, c1)
        width = slot.numel() - _TAIL
        if (config.tol is None and query is not None and query.dtype == np.float64
                and query.ndim == 1 and query.flags.c_contiguous and dc.n_cols > 0):
            nplan = _native_plan(self.ws, dc, self.de, dc.device)
            err_view = slot[width: width + 4].view(torch.int64)
            rc = nplan.run_device(query, config, slot.data_ptr(), err_view.data_ptr())
            if rc == 0:
                n = dc.n_cols
                slot[width + 6: width + 9].view(torch.int64).copy_(
                    nplan.out_dev[n + 4: n + 7])

                def decode(_words):      # rare error path: replay to name the event exactly
                    qp = QueryPlan(sel, weights, dc, self.de, config, self.ws)
                    qp.enqueue_distances()
                    qp.enqueue_solve()
                    return qp.decode_event(qp.readback()[1])

                def spans(row):
                    st = np.asarray(row[width + 6: width + 9]).view(np.int64)
                    return {"distances": (st[1] - st[0]) * 1e-9, "precompute": 0.0,
                            "init": 0.0, "iterations": (st[2] - st[1]) * 1e-9, "final": 0.0}

                return config.max_iter, False, decode, spans
            if rc > 0:
                from . import _lib

                raise _lib.NativeError(f"swmd_plan_run_device: CUDA error {rc}")
            # rc < 0: outside the native fast path (argument errors were raised by
            # select_nonzero already): the general path below
        plan = QueryPlan(sel, weights, dc, self.de, config, self.ws)
        plan.wmd = slot[: c1 - c0]
        plan.err = slot[width: width + 4].view(torch.int64)
        ev = _Events(True)
        ev.mark("d0")
        plan.enqueue_distances()
        ev.mark("d1")
        if config.tol is None:
            plan.enqueue_solve()
            iterations, converged = config.max_iter, False
        else:
            iterations, converged = plan.run_tol(allreduce_max)
        ev.mark("i1")
        return iterations, converged, plan.decode_event, lambda _row: _device_spans(ev)


# per-rank gather slot: distances (padded to the widest block) | the block's
# error record (4 int64 words, swmd.h) | iterations run | converged | the
# native runtime's 3 device clock stamps (int64 bits; zero on other paths)
_TAIL = 9


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

    arm = allreduce_max if config.tol is not None else None

    # ONE all-gather of equal slots: [distances | error record | iterations | converged]
    width = int(np.max(np.diff(bounds))) if world else 0
    slot = torch.zeros(width + _TAIL, dtype=torch.float64, device=cdev)
    if isinstance(solver, DeviceShardSolver) and cdev.type == "cuda":
        iterations, converged, decode, spans = solver.solve_into(sel, weights, c0, c1, config,
                                                                 arm, slot, query=query)
    else:
        res = solver(sel, weights, c0, c1, config, arm)
        host = np.zeros(width + _TAIL, dtype=np.float64)
        host[: c1 - c0] = res.wmd[: c1 - c0]
        words = host[width: width + 4].view(np.int64)
        words[:] = _NO_EVENT
        if res.event is not None:
            words[0] = 0                      # "this block has an event"
        iterations, converged = res.iterations, res.converged
        decode = lambda _words, ev=res.event: ev   # noqa: E731
        spans = lambda _row, t=res.timings: t   # noqa: E731
        slot.copy_(torch.from_numpy(host))
    slot[width + 4] = float(iterations)
    slot[width + 5] = 1.0 if converged else 0.0
    gathered = torch.empty(world * (width + _TAIL), dtype=torch.float64, device=cdev)
    dist.all_gather_into_tensor(gathered, slot, group=group)
    allv = gathered.cpu().numpy().reshape(world, width + _TAIL)
    words_all = allv[:, width: width + 4].copy().view(np.int64)

    if any(_has_event(w) for w in words_all):
        # rare path: every rank decodes its own block's event, one more gather
        own = words_all[rank]
        ev = decode(own) if _has_event(own) else None
        enc = np.full(4, np.inf)
        if ev is not None:
            enc[:] = [ev.code, *[float(k) for k in ev.key], rank]
        etens = torch.from_numpy(enc).to(cdev)
        eparts = torch.empty(4 * world, dtype=torch.float64, device=cdev)
        dist.all_gather_into_tensor(eparts, etens, group=group)
        evs = [e for e in eparts.cpu().numpy().reshape(world, 4) if np.isfinite(e[0])]
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
    for r in range(world):
        a, b = int(bounds[r]), int(bounds[r + 1])
        wmd[a:b] = allv[r, : b - a]
    timings = phase_timings({"select": t_select, "total": time.perf_counter() - t_start},
                            spans(allv[rank]))
    return SolverResult(wmd=wmd, iterations_run=int(allv[0, width + 4]),
                        converged=bool(allv[0, width + 5]), timings=timings)


_NO_EVENT = (1 << 63) - 1


def _has_event(words: np.ndarray) -> bool:
    """Whether an error record holds an event the reference would raise
    (a zero denominator, or a nonpositive iterate not masked by NaN)."""
    from .solver import nonpositive_fires

    return int(words[0]) != _NO_EVENT or nonpositive_fires(words)
