"""The unfused comparator: the same Sinkhorn algorithm with the intermediate
stored, on the B200 (the reference's ``baseline.unfused_sparse_wmd``,
baseline.py:67-131).

Per iteration the reference calls the standalone sampled-quotient kernel
(``kernels.sddmm``) and the sparse product (``kernels.spmm``) in sequence,
materialising the quotient values ``w`` (one per nonzero) between them.  The
device version does the same with two launches per iteration
(``swmd_unfused_iterate_f64``): an SDDMM that writes ``w`` to HBM and an SpMM
that reads it back, so every iteration re-gathers the K rows twice and round
trips ``w`` and ``x`` through HBM — exactly what the fused persistent solve
(``swmd_solve_f64``) avoids.  ``bench.py`` times both on the same resident
inputs and reports their ratio as ``fusion_speedup`` (the paper's
fused-vs-unfused comparison, 1.15-2.22x on CPUs).

Signature, phase names and error behaviour follow the reference: the
function returns the distances (N,) as a numpy array, fills ``timings`` with
the seven phase keys when a dict is passed, raises
``DegeneracyError("nonpositive iterate entry")`` when an iterate entry is not
positive and ``DegeneracyError("zero denominator at nonzero (i, j)")`` for a
zero sampled denominator.
"""

from __future__ import annotations

import time

import numpy as np
import torch

from . import _lib
from .device import DeviceCorpus, DeviceEmbeddings, device
from .kernels import DegeneracyError, select_nonzero, zero_denominator_event
from .solver import (
    PHASES,
    QueryPlan,
    SinkhornWorkspace,
    SolverConfig,
    _default_ws,
    nonpositive_fires,
)

__all__ = ["unfused_sparse_wmd", "UnfusedPlan"]


def unfused_row_width(v_r: int) -> int:
    """Padded row width of the unfused kernels (their ldk and ldx), 0 if unsupported."""
    return int(_lib.lib().swmd_unfused_row_width(int(v_r)))


class UnfusedPlan:
    """Device state of the unfused comparator for one query on one corpus.

    ``enqueue_distances`` builds K and K*M (the fused path's cost build, with
    the unfused kernels' padded row width), ``enqueue_iteration`` launches one
    SDDMM + SpMM pair, ``enqueue_final`` the distance pass.  Nothing
    synchronises the host, so a whole solve can be captured in a CUDA graph.
    """

    def __init__(self, sel: np.ndarray | None, weights: np.ndarray | None, dc: DeviceCorpus,
                 de: DeviceEmbeddings, config: SolverConfig, ws: SinkhornWorkspace,
                 staged_v_r: int | None = None):
        v_r = int(sel.size) if staged_v_r is None else int(staged_v_r)
        width = unfused_row_width(v_r)
        if width == 0:
            raise ValueError(f"the device unfused comparator supports v_r <= 64, got {v_r}")
        self.qp = QueryPlan(sel, weights, dc, de, config, ws, staged_v_r=staged_v_r, ldk=width)
        self.dc, self.config, self.v_r, self.ld = dc, config, v_r, width
        dws = self.qp.dws
        n = dc.n_cols * width
        self.x = (dws.flat("unf_x_a", n), dws.flat("unf_x_b", n))
        self.w = dws.flat("unf_w", max(1, dc.nnz))
        self.cur = None

    @property
    def err(self) -> torch.Tensor:
        return self.qp.err

    @property
    def wmd(self) -> torch.Tensor:
        return self.qp.wmd

    def enqueue_distances(self) -> None:
        self.qp.enqueue_distances()   # also resets the error record
        self.cur = None

    def enqueue_iteration(self, t: int) -> None:
        qp, dc = self.qp, self.dc
        nxt = self.x[t % 2]
        _lib.call("swmd_unfused_iterate_f64", dc.col_ptr.data_ptr(), dc.rows.data_ptr(),
                  dc.vals.data_ptr(), dc.n_cols, qp.K.data_ptr(), qp.r_dev.data_ptr(), self.v_r,
                  self.ld, self.cur.data_ptr() if self.cur is not None else None, nxt.data_ptr(),
                  self.ld, self.w.data_ptr(), t, dc.col_offset, dc.n_key, qp.err.data_ptr(),
                  qp.stream)
        self.cur = nxt

    def enqueue_final(self, t_final: int) -> None:
        qp, dc = self.qp, self.dc
        _lib.call("swmd_unfused_final_f64", dc.col_ptr.data_ptr(), dc.rows.data_ptr(),
                  dc.vals.data_ptr(), dc.n_cols, qp.K.data_ptr(), qp.KM.data_ptr(), self.v_r,
                  self.ld, self.cur.data_ptr() if self.cur is not None else None, self.ld,
                  qp.wmd.data_ptr(), t_final, dc.col_offset, dc.n_key, qp.err.data_ptr(),
                  qp.stream)

    def enqueue_solve(self) -> None:
        """tol unset: max_iter iterations and the final pass, no host sync."""
        self.cur = None   # x = 1/v_r (init_x) at the first iteration of every solve
        for t in range(self.config.max_iter):
            self.enqueue_iteration(t)
        self.enqueue_final(self.config.max_iter)

    def run_tol(self) -> tuple[int, bool]:
        """tol set: the reference's early exit (baseline.py:119-121) — the
        max-norm change is read back after every iteration.  Returns
        (iterations run, failed); the final pass is left to the caller."""
        host = self.qp.ws.pinned("unf_err_host", _lib.ERR_WORDS, torch.int64)
        t_done = 0
        self.cur = None
        for t in range(self.config.max_iter):
            self.qp.err[2].zero_()
            self.enqueue_iteration(t)
            host.copy_(self.qp.err)
            torch.cuda.current_stream(self.qp.dev).synchronize()
            he = host.numpy()
            t_done = t + 1
            if he[0] != _lib.NO_EVENT or nonpositive_fires(he):
                return t_done, True
            if float(he[2:3].view(np.float64)[0]) < self.config.tol:
                break
        return t_done, False


def _raise_first_event(he: np.ndarray, n_key: int) -> None:
    """The first failing check in the reference's order (event codes: swmd.h)."""
    zd = zero_denominator_event(he, n_key)
    code_nonpos = int(he[1]) if nonpositive_fires(he) else None
    if code_nonpos is not None and (zd is None or code_nonpos < zd[0]):
        raise DegeneracyError("nonpositive iterate entry")
    if zd is not None:
        raise DegeneracyError(f"zero denominator at nonzero ({zd[1]}, {zd[2]})")


def unfused_sparse_wmd(query, corpus, embeddings, config: SolverConfig,
                       timings: dict[str, float] | None = None) -> np.ndarray:
    """Same algorithm as the fused solver with ``w`` stored between an SDDMM
    and an SpMM launch every iteration (baseline.py:67-131).  Pass a dict as
    ``timings`` to receive per-phase durations under the fused solver's phase
    names (device phases from CUDA events)."""
    record = timings if timings is not None else {}
    t_start = time.perf_counter()
    t0 = time.perf_counter()
    sel, weights = select_nonzero(np.asarray(query, dtype=np.float64))
    record["select"] = time.perf_counter() - t0
    dev = device()
    if tuple(embeddings.shape)[0] != corpus.n_rows:
        raise ValueError(f"shape mismatch: embeddings {tuple(embeddings.shape)}, "
                         f"corpus rows {corpus.n_rows}")
    dc = DeviceCorpus.of(corpus, dev)
    de = DeviceEmbeddings.of(embeddings, dev)
    plan = UnfusedPlan(sel, weights, dc, de, config, _default_ws())
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    plan.enqueue_distances()
    ev[1].record()
    if config.tol is None:
        for t in range(config.max_iter):
            plan.enqueue_iteration(t)
        ev[2].record()
        plan.enqueue_final(config.max_iter)
    else:
        t_done, failed = plan.run_tol()
        ev[2].record()
        if not failed:
            plan.enqueue_final(t_done)
    ev[3].record()
    out = plan.qp.out.cpu().numpy()
    n = dc.n_cols
    he = out[n:]
    _raise_first_event(he, dc.n_key)
    wmd = out[:n].view(np.float64).copy()
    record["distances"] = ev[0].elapsed_time(ev[1]) / 1e3
    record["precompute"] = 0.0   # fused into the cost build
    record["init"] = 0.0         # x = 1/v_r is implicit in the first SDDMM
    record["iterations"] = ev[1].elapsed_time(ev[2]) / 1e3
    record["final"] = ev[2].elapsed_time(ev[3]) / 1e3
    record["total"] = time.perf_counter() - t_start
    for k in PHASES:
        record.setdefault(k, 0.0)
    return wmd
