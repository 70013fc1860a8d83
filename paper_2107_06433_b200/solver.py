"""Sinkhorn-WMD solver: the drop-in entry point, running on one B200.

``sinkhorn_wmd(query, corpus, embeddings, config, workspace=None)`` keeps the
reference's signature, result type, phase names and error behaviour
(solver.py:106-201).  What runs underneath:

1. ``select`` — positive entries of the query, on the host (the reference's
   numpy step, kernels.py:74-88); ``sel`` and ``r`` go to the device in one
   small copy.
2. ``distances`` — one launch of the fused cost/kernel build
   (swmd_cost_build_f64): M, K = exp(-lam M) and K*M for every vocabulary row
   that occurs in the corpus (rows that never occur are never read).
   ``precompute`` is fused into it and reports 0.
3. ``iterations`` — tol unset: ONE persistent launch (swmd_solve_f64) runs
   all max_iter iterations and the final type-2 pass per document column
   with x, u on chip (``init`` and ``final`` are fused and report 0);
   tol set: one launch per iteration with the max-norm change read back after
   each, as the reference does (solver.py:179-183), then a final launch.
4. One device->host copy returns the distances and the error record.

Per-phase times come from CUDA events on the solver's stream.
"""

from __future__ import annotations

import os
import threading
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import cuda_ok, DeviceCorpus, DeviceEmbeddings, DeviceWorkspace, device, stream_ptr
from .kernels import (
    COST_MODE_DIRECT,
    COST_MODE_GRAM,
    DegeneracyError,
    EmptyQueryError,
    raise_zero_denominator,
    select_nonzero,
    zero_denominator_event,
)
from .sparse import SparseVector

__all__ = [
    "SolverConfig",
    "SolverResult",
    "SinkhornWorkspace",
    "init_x",
    "update_u",
    "sinkhorn_wmd",
    "sinkhorn_wmd_batch",
    "sinkhorn_wmd_devices",
    "solve_on_device",
    "DegEvent",
    "ShardResult",
    "QueryPlan",
    "TopKResult",
    "sinkhorn_wmd_topk",
]

PHASES = ("select", "distances", "precompute", "init", "iterations", "final", "total")


@dataclass(frozen=True)
class SolverConfig:
    """Solver parameters (solver.py:22-46).

    ``workers`` and ``deterministic`` are accepted for compatibility; the GPU
    path is column-owned, so results are identical for every value.
    ``cost_mode`` selects the distance form: "gram" (default; fused
    ||e||^2+||q||^2-2e.q with an exact zero self-distance) or "direct" (the
    reference's difference form, bitwise-identical distances).
    ``precision="f32"`` selects the multi-query fp32 variant (BASELINE c4;
    batch.py): fp32 embeddings, kernel matrices and iterates, results within
    1e-4 of the fp64 reference.
    """

    lam: float = 10.0
    max_iter: int = 15
    tol: float | None = None
    workers: int = 1
    deterministic: bool = False
    cost_mode: str = "gram"
    precision: str = "f64"

    def __post_init__(self):
        if self.lam <= 0.0:
            raise ValueError(f"lam must be positive, got {self.lam}")
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {self.max_iter}")
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")
        if self.tol is not None and self.tol < 0.0:
            raise ValueError(f"tol must be nonnegative, got {self.tol}")
        if self.cost_mode not in ("gram", "direct"):
            raise ValueError(f"cost_mode must be 'gram' or 'direct', got {self.cost_mode!r}")
        if self.precision not in ("f64", "f32"):
            raise ValueError(f"precision must be 'f64' or 'f32', got {self.precision!r}")


@dataclass(frozen=True)
class SolverResult:
    """Distances of one query to every target document (solver.py:49-56)."""

    wmd: np.ndarray
    iterations_run: int
    converged: bool
    timings: dict[str, float]


class SinkhornWorkspace:
    """Reusable buffers (solver.py:59-81): host pools with the reference's
    ``matrix``/``vector`` views, plus grow-only device pools per GPU."""

    def __init__(self):
        self._pools: dict[str, np.ndarray] = {}
        self._device: dict[tuple, DeviceWorkspace] = {}
        self._pinned: dict[str, torch.Tensor] = {}

    def _flat(self, name: str, size: int) -> np.ndarray:
        pool = self._pools.get(name)
        if pool is None or pool.size < size:
            pool = np.empty(size, dtype=np.float64)
            self._pools[name] = pool
        return pool[:size]

    def matrix(self, name: str, n_rows: int, n_cols: int) -> np.ndarray:
        return self._flat(name, n_rows * n_cols).reshape(n_rows, n_cols)

    def vector(self, name: str, size: int) -> np.ndarray:
        return self._flat(name, size)

    def on(self, dev: torch.device) -> DeviceWorkspace:
        key = (dev.type, dev.index)
        ws = self._device.get(key)
        if ws is None:
            ws = DeviceWorkspace(dev)
            self._device[key] = ws
        return ws

    def pinned(self, name: str, n: int, dtype=torch.int64) -> torch.Tensor:
        p = self._pinned.get(name)
        if p is None or p.numel() < n or p.dtype != dtype:
            # pinned when a device exists (async H2D); plain host memory otherwise,
            # so argument errors still surface before the missing-device error
            p = torch.empty(max(n, 1), dtype=dtype, pin_memory=torch.cuda.is_available())
            self._pinned[name] = p
            self._pinned_np = {}
        return p[:n]

    def pinned_np(self, name: str, n: int) -> np.ndarray:
        """numpy view of a pinned int64 staging buffer (grow-only)."""
        t = self.pinned(name, n)
        cache = self.__dict__.setdefault("_pinned_np", {})
        arr = cache.get(name)
        if arr is None or arr.size < n:
            arr = self._pinned[name].numpy()
            cache[name] = arr
        return arr


try:
    _HOT_ROWS = max(0, int(os.environ.get("SWMD_CTA_HOT", "0") or 0))
except ValueError:
    _HOT_ROWS = 0


def init_x(v_r: int, n_docs: int) -> np.ndarray:
    """Uniform initial iterate 1/v_r, document-major (n_docs, v_r) (solver.py:84-92)."""
    if v_r < 1 or n_docs < 1:
        raise ValueError(f"need v_r >= 1 and n_docs >= 1, got ({v_r}, {n_docs})")
    return np.full((n_docs, v_r), 1.0 / v_r, dtype=np.float64)


def update_u(x: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    """Elementwise reciprocal with the positivity check (solver.py:95-103).

    Host numpy helper kept for API compatibility; the device path fuses this
    step into the iteration kernel.
    """
    x = np.asarray(x)
    if x.size and np.min(x) <= 0.0:
        flat = int(np.argmin(x))
        raise DegeneracyError(f"nonpositive iterate entry {x.flat[flat]} at flat index {flat}")
    return np.divide(1.0, x, out=out)


# ----------------------------------------------------------------------------------------

_ws_local = threading.local()


def _default_ws() -> SinkhornWorkspace:
    """The implicit workspace of ``workspace=None`` calls: one per host thread,
    so concurrent solver calls never share staging buffers or a native plan
    (the reference's contract: concurrent calls on distinct workspaces are
    safe)."""
    ws = getattr(_ws_local, "ws", None)
    if ws is None:
        ws = _ws_local.ws = SinkhornWorkspace()
    return ws


class _Events:
    """CUDA events on the solver stream (per-phase device timings)."""

    def __init__(self, enabled: bool):
        self.enabled = enabled
        self.ev: dict[str, torch.cuda.Event] = {}

    def mark(self, name: str):
        if self.enabled:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.ev[name] = e

    def span(self, a: str, b: str) -> float:
        if not self.enabled or a not in self.ev or b not in self.ev:
            return 0.0
        return self.ev[a].elapsed_time(self.ev[b]) / 1e3


def phase_timings(host: dict, device: dict) -> dict[str, float]:
    """The reference's per-phase ``timings`` dict (solver.py:131-194): the
    seven phase keys in order, host phases from ``host``, device phases from
    ``device`` (seconds; phases fused into another kernel report 0.0)."""
    d = {**device, **host}
    return {k: float(d.get(k, 0.0)) for k in PHASES}


def _device_spans(ev: _Events) -> dict[str, float]:
    """Device phase times once the stream has been synchronised."""
    return {"distances": ev.span("d0", "d1"), "precompute": 0.0, "init": 0.0,
            "iterations": ev.span("d1", "i1"), "final": 0.0}


def _nonpositive_entry(dc: DeviceCorpus, K, KM, r_dev, v_r: int, ldk: int, t_check: int,
                       ws: DeviceWorkspace) -> tuple[float, int]:
    """Re-derive what the reference's update_u reports (solver.py:95-103) — the
    value and first flat index of min x — for the check at iteration t_check,
    replaying the iterations with x stored.  Only runs on the error path."""
    dev = dc.device
    n = dc.n_cols * v_r
    xa = ws.flat("diag_x_a", n)
    xb = ws.flat("diag_x_b", n)
    err = ws.flat("diag_err", _lib.ERR_WORDS, torch.int64)
    counter = ws.flat("counter", 1, torch.int32)
    cur = None
    for t in range(t_check):
        nxt = (xa, xb)[t % 2]
        _lib.call("swmd_err_reset", err.data_ptr(), stream_ptr(dev))
        _lib.call("swmd_solve_f64", dc.col_ptr.data_ptr(), dc.rows.data_ptr(), dc.vals.data_ptr(),
                  dc.n_cols, dc.order.data_ptr(), K.data_ptr(), KM.data_ptr(), r_dev.data_ptr(),
                  v_r, ldk, t, t + 1, cur.data_ptr() if cur is not None else None,
                  nxt.data_ptr(), None, dc.col_offset, dc.n_key, _group(dc, v_r),
                  dc.max_len, err.data_ptr(), counter.data_ptr(), stream_ptr(dev))
        cur = nxt
    x = cur.view(dc.n_cols, v_r)
    # global flat index in the reference's (N, v_r) iterate
    flat_local = int(torch.argmin(x.reshape(-1)).item())
    val = float(x.reshape(-1)[flat_local].item())
    flat = (dc.col_offset * v_r) + flat_local
    return val, flat


def _group(dc: DeviceCorpus, v_r: int) -> int:
    return 32 if dc.mean_len > 64 else 16


def nonpositive_fires(he: np.ndarray) -> bool:
    """Whether the reference's update_u check (solver.py:95-103) fires for the
    event recorded in err[1]: not when a NaN entry was seen at the same or an
    earlier check (err[3]) — np.min propagates NaN and ``min(x) <= 0`` is
    then False."""
    if he[1] == _lib.NO_EVENT:
        return False
    return not (he[3] != _lib.NO_EVENT and int(he[3]) <= int(he[1]))


@dataclass(frozen=True)
class DegEvent:
    """The earliest degeneracy of a (shard's) solve: its event code (swmd.h),
    a key ordering simultaneous events the way the reference reports them
    ((i, j) of a zero denominator; (value, flat index) of a nonpositive
    iterate entry), and the reference's message."""

    code: int
    key: tuple
    message: str


@dataclass
class ShardResult:
    wmd: np.ndarray
    iterations: int
    converged: bool
    timings: dict
    event: DegEvent | None


class QueryPlan:
    """Device state of one query against one resident corpus (block).

    Construction uploads ``sel`` and ``r`` in one small copy and binds the
    workspace buffers; ``enqueue_distances`` / ``enqueue_solve`` only launch
    kernels (no host synchronisation), ``readback`` copies the distances and
    the error record back in one transfer.  bench.py times the enqueue calls
    alone for the device-resident figure.
    """

    def __init__(self, sel: np.ndarray | None, weights: np.ndarray | None, dc: DeviceCorpus,
                 de: DeviceEmbeddings, config: SolverConfig, ws: SinkhornWorkspace,
                 staged_v_r: int | None = None, ldk: int | None = None):
        self.dc, self.de, self.config, self.ws = dc, de, config, ws
        self.dev = dc.device
        self._stream = stream_ptr(self.dev)
        self.dws = dws = ws.on(self.dev)
        if staged_v_r is None:
            v_r = int(sel.size)
            stage = ws.pinned("qstage", 2 * v_r, torch.int64)
            stage_np = stage.numpy()
            stage_np[:v_r] = sel
            stage_np[v_r:] = np.ascontiguousarray(weights, dtype=np.float64).view(np.int64)
        else:   # (sel | weight bits) already in the pinned stage (native select)
            v_r = int(staged_v_r)
            stage = ws.pinned("qstage", 2 * v_r, torch.int64)
        self.v_r = v_r
        # K row stride = v_r rounded up to 4 (zero pad columns): 16-byte rows that
        # the fast v_r <= 32 kernel reads as whole pairs without masking
        self.ldk = ((v_r + 3) // 4) * 4 if v_r <= 32 else v_r + (v_r & 1)
        if ldk is not None:   # a caller-chosen padded width (the unfused comparator)
            self.ldk = int(ldk)
        V, N = dc.n_rows, dc.n_cols
        qdev = dws.flat("qdev", 2 * v_r, torch.int64)
        qdev.copy_(stage[: 2 * v_r], non_blocking=True)
        self.sel_dev = qdev[:v_r]
        self.r_dev = qdev[v_r:].view(torch.float64)
        self.K = dws.flat("kernel", V * self.ldk)
        self.KM = dws.flat("kernel_cost", V * self.ldk)
        self.out = dws.flat("out", N + _lib.ERR_WORDS, torch.int64)
        self.wmd = self.out[:N].view(torch.float64)
        self.err = self.out[N:]
        self.counter = dws.flat("counter", 1, torch.int32)
        self.mode = COST_MODE_GRAM if config.cost_mode == "gram" else COST_MODE_DIRECT
        self.norms = de.norms if self.mode == COST_MODE_GRAM else None
        self.use_list = dc.present_rows is not None and dc.n_present < V
        self.group = _group(dc, v_r)
        self.launches = 0

    @property
    def stream(self) -> int:
        return self._stream

    def enqueue_distances(self) -> None:
        dc, de = self.dc, self.de
        # the solve's error record and work counter are reset here, ahead of
        # the cost build (by the cost kernel itself on the compact path), so
        # enqueue_solve launches right behind it
        self._armed = True
        comp = dc.compact_rows(de) if self.mode == COST_MODE_GRAM else None
        if comp is not None:
            Ec, ldc = comp
            n_c = dc.n_present if self.use_list else dc.n_rows
            _lib.call("swmd_cost_build_compact_reset_f64", de.E.data_ptr(), de.ld, Ec.data_ptr(),
                      n_c, de.dim, ldc, dc.present_rows.data_ptr() if self.use_list else None,
                      self.sel_dev.data_ptr(), self.v_r, self.r_dev.data_ptr(),
                      float(self.config.lam), self.norms.data_ptr(), self.K.data_ptr(),
                      self.KM.data_ptr(), self.ldk, self.err.data_ptr(), self.counter.data_ptr(),
                      self.stream)
            self.launches += (self.ldk + 31) // 32
            return
        _lib.call("swmd_solve_reset", self.err.data_ptr(), self.counter.data_ptr(), self.stream)
        self.launches += 1
        _lib.call("swmd_cost_build_f64", de.E.data_ptr(), de.V, de.dim, de.ld,
                  self.sel_dev.data_ptr(), self.v_r, self.r_dev.data_ptr(),
                  float(self.config.lam), self.mode,
                  self.norms.data_ptr() if self.norms is not None else None,
                  dc.present_rows.data_ptr() if self.use_list else None,
                  dc.n_present if self.use_list else 0, None, self.K.data_ptr(), None,
                  self.KM.data_ptr(), self.ldk, self.stream)
        self.launches += (self.ldk + 31) // 32

    def _solve(self, t0: int, t1: int, x_in, x_out, wmd, reset_done: bool = False) -> None:
        dc = self.dc
        if 32 < self.v_r <= 256 and _HOT_ROWS > 0:
            # long queries, opt-in (SWMD_CTA_HOT=<rows>): the corpus's hot-row
            # index rides along (swmd.h: swmd_solve_hot_f64)
            slot, ids = dc.hot_index()
            _lib.call("swmd_solve_hot_f64", dc.col_ptr.data_ptr(), dc.rows.data_ptr(),
                      dc.vals.data_ptr(), dc.n_cols, dc.order.data_ptr(), self.K.data_ptr(),
                      self.KM.data_ptr(), self.r_dev.data_ptr(), self.v_r, self.ldk, t0, t1,
                      x_in.data_ptr() if x_in is not None else None,
                      x_out.data_ptr() if x_out is not None else None,
                      wmd.data_ptr() if wmd is not None else None, dc.col_offset, dc.n_key,
                      self.group, dc.max_len, self.err.data_ptr(), self.counter.data_ptr(),
                      self.stream, 1 if reset_done else 0,
                      slot.data_ptr() if slot is not None else None,
                      ids.data_ptr() if ids is not None else None,
                      int(ids.numel()) if ids is not None else 0)
            self.launches += 1
            return
        _lib.call("swmd_solve_f64_reset_done" if reset_done else "swmd_solve_f64",
                  dc.col_ptr.data_ptr(), dc.rows.data_ptr(),
                  dc.vals.data_ptr(), dc.n_cols, dc.order.data_ptr(), self.K.data_ptr(),
                  self.KM.data_ptr(), self.r_dev.data_ptr(), self.v_r, self.ldk, t0, t1,
                  x_in.data_ptr() if x_in is not None else None,
                  x_out.data_ptr() if x_out is not None else None,
                  wmd.data_ptr() if wmd is not None else None, dc.col_offset, dc.n_key,
                  self.group, dc.max_len, self.err.data_ptr(), self.counter.data_ptr(),
                  self.stream)
        self.launches += 1

    def enqueue_solve(self) -> None:
        """tol unset: the whole loop plus the final pass in one persistent launch."""
        if getattr(self, "_armed", False):
            self._armed = False
            self._solve(0, self.config.max_iter, None, None, self.wmd, reset_done=True)
            return
        _lib.call("swmd_err_reset", self.err.data_ptr(), self.stream)
        self.launches += 1
        self._solve(0, self.config.max_iter, None, None, self.wmd)

    # tol path, split so several plans (devices) can run it in lockstep
    def tol_begin(self) -> None:
        n = self.dc.n_cols * self.v_r
        self._tol_bufs = (self.dws.flat("x_a", n), self.dws.flat("x_b", n))
        self._tol_host = self.ws.pinned("err_host", _lib.ERR_WORDS, torch.int64)
        self._armed = False
        _lib.call("swmd_err_reset", self.err.data_ptr(), self.stream)
        self._cur = None

    def tol_launch(self, t: int) -> None:
        """Iteration t with x stored; the error record (max|dx| in err[2]) is
        copied to pinned host memory behind it."""
        nxt = self._tol_bufs[t % 2]
        self.err[2].zero_()
        self._solve(t, t + 1, self._cur, nxt, None)
        self._tol_host.copy_(self.err, non_blocking=True)
        self._cur = nxt

    def tol_read(self) -> tuple[bool, float]:
        """(failed, max|dx|) of the last launched iteration (synchronises)."""
        torch.cuda.synchronize(self.dev)
        he = self._tol_host.numpy()
        fail = he[0] != _lib.NO_EVENT or nonpositive_fires(he)
        return bool(fail), float(he[2:3].view(np.float64)[0])

    def tol_final(self, iterations: int) -> None:
        self._solve(iterations, iterations, self._cur, None, self.wmd)

    def run_tol(self, allreduce_max=None) -> tuple[int, bool]:
        """tol set: one launch per iteration, max|dx| read back after each
        (solver.py:170-183), then the final pass.  Returns (iterations, converged)."""
        cfg = self.config
        self.tol_begin()
        iterations, converged, failed = 0, False, False
        for t in range(cfg.max_iter):
            self.tol_launch(t)
            fail, delta = self.tol_read()
            iterations += 1
            if allreduce_max is not None:
                g = allreduce_max(np.array([delta, 1.0 if fail else 0.0]))
                delta, fail = float(g[0]), bool(g[1] > 0)
            if fail:
                failed = True      # decoded from the error record by the caller
                break
            if delta < cfg.tol:
                converged = True
                break
        if not failed:
            self.tol_final(iterations)
        return iterations, converged

    def readback(self) -> tuple[np.ndarray, np.ndarray]:
        N = self.dc.n_cols
        host = self.ws.pinned("out_host", N + _lib.ERR_WORDS, torch.int64)
        host.copy_(self.out, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        hn = host.numpy()
        return hn[:N].view(np.float64).copy(), hn[N:].copy()

    def decode_event(self, he: np.ndarray) -> DegEvent | None:
        """Earliest degeneracy in the error record (precedence: see swmd.h)."""
        dc = self.dc
        zd = zero_denominator_event(he, dc.n_key)
        code_zero = zd[0] if zd is not None else None
        code_nonpos = int(he[1]) if nonpositive_fires(he) else None
        if code_nonpos is not None and (code_zero is None or code_nonpos < code_zero):
            val, flat = _nonpositive_entry(dc, self.K, self.KM, self.r_dev, self.v_r, self.ldk,
                                           code_nonpos // 2, self.dws)
            return DegEvent(code_nonpos, (val, flat),
                            f"nonpositive iterate entry {val} at flat index {flat}")
        if zd is not None:
            code, i, j = zd
            if (i * dc.n_key + j) >= (1 << 47) - 1:
                return DegEvent(code, (float("inf"), 0),
                                "zero denominator at nonzero (index overflow)")
            return DegEvent(code, (i, j), f"zero denominator at nonzero ({i}, {j})")
        return None


def solve_on_device(sel: np.ndarray | None, weights: np.ndarray | None, dc: DeviceCorpus,
                    de: DeviceEmbeddings, config: SolverConfig, ws: SinkhornWorkspace,
                    timed: bool = True, allreduce_max=None,
                    staged_v_r: int | None = None) -> ShardResult:
    """Run phases 2-4 for one query on ``dc``'s device (all columns of ``dc``).

    ``allreduce_max`` (multi-GPU tol path) maps a float64 numpy vector to its
    element-wise max over ranks; it keeps the early exit global.
    """
    ev = _Events(timed)
    plan = QueryPlan(sel, weights, dc, de, config, ws, staged_v_r=staged_v_r)
    ev.mark("d0")
    plan.enqueue_distances()
    ev.mark("d1")
    if config.tol is None:
        plan.enqueue_solve()
        iterations, converged = config.max_iter, False
        ev.mark("i1")
    else:
        iterations, converged = plan.run_tol(allreduce_max)
        ev.mark("i1")
    wmd_host, he = plan.readback()
    event = plan.decode_event(he)
    return ShardResult(wmd_host, iterations, converged, _device_spans(ev), event)


def _is_sparse_vector(q) -> bool:
    """This package's SparseVector or the reference's (same attributes)."""
    return isinstance(q, SparseVector) or (
        not isinstance(q, np.ndarray) and hasattr(q, "indices") and hasattr(q, "values")
        and hasattr(q, "length") and hasattr(q, "to_dense"))


def select_native(query: np.ndarray, ws: SinkhornWorkspace) -> tuple[np.ndarray, np.ndarray]:
    """``select_nonzero`` (kernels.py:74-88) through the native scan
    (swmd_select_query): the same ``(sel, weights)``, errors and messages, at
    a fraction of numpy's cost on a dense 100k-word histogram."""
    v_r = _stage_query(query, query.shape[0], ws)
    st = ws.pinned_np("qstage", 2 * v_r)
    return st[:v_r].copy(), st[v_r: 2 * v_r].view(np.float64).copy()


def _stage_query(query, n_vocab: int, ws: SinkhornWorkspace) -> int:
    """select_nonzero (kernels.py:74-88) straight into the pinned H2D stage:
    writes (sel | weight bits) and returns v_r.  Same errors as the reference."""
    if isinstance(query, SparseVector):
        idx, val = query.indices, query.values
        v_r = int(idx.size)
        if v_r == 0:
            raise EmptyQueryError("query histogram has no positive entries")
        st = ws.pinned_np("qstage", 2 * v_r)
        st[:v_r] = idx
        st[v_r: 2 * v_r] = val.view(np.int64)
        return v_r
    q = np.asarray(query, dtype=np.float64)
    if q.ndim != 1:
        raise ValueError("query histogram must be 1-D")
    if not q.flags.c_contiguous:
        q = np.ascontiguousarray(q)
    cap = max(64, ws.__dict__.get("_qcap", 64))
    while True:
        st = ws.pinned_np("qstage", 2 * cap)
        cnt = _lib.lib().swmd_select_query(q.ctypes.data, q.size, st.ctypes.data, cap)
        if cnt == -2:
            raise ValueError("query histogram must be nonnegative")
        if cnt < 0:
            raise ValueError("query histogram could not be read")
        if cnt <= cap:
            break
        cap = int(cnt)
        ws.__dict__["_qcap"] = cap
    if cnt == 0:
        raise EmptyQueryError("query histogram has no positive entries")
    if cnt != cap:
        # weights were written right after the ids: already contiguous
        pass
    return int(cnt)


class NativePlan:
    """The native per-query runtime (swmd_plan_run) bound to one resident
    corpus and embedding table: buffers owned here, pointers handed to C once."""

    Q_CAP = 32

    def __init__(self, dc: DeviceCorpus, de: DeviceEmbeddings):
        dev = dc.device
        self.dc, self.de = dc, de
        V, N = dc.n_rows, dc.n_cols
        self.K = torch.empty(V * 32, dtype=torch.float64, device=dev)
        self.KM = torch.empty(V * 32, dtype=torch.float64, device=dev)
        self.qdev = torch.empty(2 * self.Q_CAP, dtype=torch.int64, device=dev)
        self.qhost = torch.empty(2 * self.Q_CAP, dtype=torch.int64, pin_memory=True)
        self.out_dev = torch.empty(N + _lib.ERR_WORDS + 3, dtype=torch.int64, device=dev)
        self.out_host = torch.empty(N + _lib.ERR_WORDS + 3, dtype=torch.int64, pin_memory=True)
        self.counter = torch.empty(1, dtype=torch.int32, device=dev)
        self.err = np.empty(_lib.ERR_WORDS, dtype=np.int64)
        self.times = np.zeros(6, dtype=np.float32)
        self.vr = np.zeros(1, dtype=np.int64)
        norms = de.norms
        pres = dc.present_rows
        desc = np.array([
            de.E.data_ptr(), de.V, de.dim, de.ld, norms.data_ptr(),
            dc.col_ptr.data_ptr(), dc.rows.data_ptr(), dc.vals.data_ptr(), N,
            dc.order.data_ptr(), pres.data_ptr() if pres is not None else 0, dc.n_present,
            dc.col_offset, dc.n_key, dc.max_len, _group(dc, 19),
            self.K.data_ptr(), self.KM.data_ptr(), V * 32,
            self.qdev.data_ptr(), self.qhost.data_ptr(), self.Q_CAP,
            self.out_dev.data_ptr(), self.out_host.data_ptr(), self.counter.data_ptr(),
            stream_ptr(dev), *self._compact(dc, de)], dtype=np.int64)
        import ctypes
        h = ctypes.c_void_p()
        _lib.call("swmd_plan_create", ctypes.byref(h), desc.ctypes.data, desc.size)
        self.handle = h
        self._args = (self.err.ctypes.data, self.times.ctypes.data, self.vr.ctypes.data)
        self._stream = stream_ptr(dev)

    def _compact(self, dc, de):
        comp = dc.compact_rows(de)
        if comp is None:
            return [0, 0, 0]
        self._Ec = comp[0]
        n_c = dc.n_present if (dc.present_rows is not None and dc.n_present < dc.n_rows) else dc.n_rows
        return [comp[0].data_ptr(), n_c, comp[1]]

    def __del__(self):
        try:
            _lib.lib().swmd_plan_destroy(self.handle)
        except Exception:
            pass

    def run_device(self, q: np.ndarray, config: SolverConfig, wmd_ptr: int, err_ptr: int) -> int:
        """Enqueue the query with results left in device buffers (no sync).
        Returns rc: 0 ok, -2/-3 argument errors, -4 general path."""
        mode = COST_MODE_GRAM if config.cost_mode == "gram" else COST_MODE_DIRECT
        return _lib.lib().swmd_plan_run_device(self.handle, q.ctypes.data, q.size,
                                               float(config.lam), int(config.max_iter), mode,
                                               wmd_ptr, err_ptr, self.vr.ctypes.data)

    def run_selected(self, indices: np.ndarray, values: np.ndarray, config: SolverConfig):
        """``run`` for an already-selected query (SparseVector): (rc, wmd)."""
        sel = np.ascontiguousarray(indices, dtype=np.int64)
        w = np.ascontiguousarray(values, dtype=np.float64)
        wmd = np.empty(self.dc.n_cols, dtype=np.float64)
        mode = COST_MODE_GRAM if config.cost_mode == "gram" else COST_MODE_DIRECT
        rc = _lib.lib().swmd_plan_run_selected(self.handle, sel.ctypes.data, w.ctypes.data,
                                               sel.size, float(config.lam), int(config.max_iter),
                                               mode, wmd.ctypes.data, self._args[0], self._args[1])
        return rc, wmd

    def run(self, q: np.ndarray, config: SolverConfig):
        """Returns (rc, wmd).  rc: 0 ok, -2/-3 argument errors, -4 general path."""
        wmd = np.empty(self.dc.n_cols, dtype=np.float64)
        mode = COST_MODE_GRAM if config.cost_mode == "gram" else COST_MODE_DIRECT
        rc = _lib.lib().swmd_plan_run(self.handle, q.ctypes.data, q.size, float(config.lam),
                                      int(config.max_iter), mode, wmd.ctypes.data, *self._args)
        return rc, wmd


def _native_plan(ws: SinkhornWorkspace, dc: DeviceCorpus, de: DeviceEmbeddings,
                 dev: torch.device) -> "NativePlan | None":
    key = (id(dc), id(de))
    cache = ws.__dict__.setdefault("_native_plans", {})
    plan = cache.get(key)
    if plan is None or plan.dc is not dc or plan.de is not de or plan._stream != stream_ptr(dev):
        plan = NativePlan(dc, de)
        cache.clear()          # one resident plan per workspace
        cache[key] = plan
    return plan


def sinkhorn_wmd(query, corpus, embeddings, config: SolverConfig,
                 workspace: SinkhornWorkspace | None = None) -> SolverResult:
    """Regularised transport distance of one query to every corpus column
    (solver.py:106-201), on the current CUDA device."""
    t_start = time.perf_counter()
    n_vocab = corpus.n_rows
    emb_shape = tuple(embeddings.shape)
    ws = workspace if workspace is not None else _default_ws()
    if _is_sparse_vector(query):
        # the reference's ingest hands queries over as SparseVector histograms
        # (ingest.py:175-197): already selected, so the native runtime takes
        # (ids, weights) directly — no densify, no scan of V entries
        if (config.tol is None and config.precision == "f64" and config.workers <= 1
                and int(query.length) == n_vocab and emb_shape[0] == n_vocab
                and corpus.n_cols > 0 and 0 < query.indices.size <= 32 and cuda_ok()):
            dev = device()
            dc = DeviceCorpus.of(corpus, dev)
            de = DeviceEmbeddings.of(embeddings, dev)
            plan = _native_plan(ws, dc, de, dev)
            rc, wmd = plan.run_selected(query.indices, query.values, config)
            if rc > 0:
                raise _lib.NativeError(f"swmd_plan_run_selected: CUDA error {rc}")
            if rc == 0 and plan.err[0] == _lib.NO_EVENT and plan.err[1] == _lib.NO_EVENT:
                t = plan.times
                timings = {"select": float(t[2]) / 1e3, "distances": float(t[0]) / 1e3,
                           "precompute": 0.0, "init": 0.0, "iterations": float(t[1]) / 1e3,
                           "final": 0.0, "total": time.perf_counter() - t_start}
                return SolverResult(wmd=wmd, iterations_run=config.max_iter, converged=False,
                                    timings=timings)
        query = query.to_dense()
    query = np.asarray(query, dtype=np.float64)
    if query.shape != (n_vocab,) or emb_shape[0] != n_vocab:
        raise ValueError(
            f"shape mismatch: query {query.shape}, embeddings "
            f"{emb_shape}, corpus rows {n_vocab}")
    if config.workers > 1 and config.precision == "f64" and corpus.n_cols > 1 and cuda_ok():
        n_dev = min(config.workers, torch.cuda.device_count())
        if n_dev > 1:   # workers -> GPUs: one column block per device
            devs = [torch.device("cuda", k) for k in range(n_dev)]
            return sinkhorn_wmd_devices(query, corpus, embeddings, config, devs, ws, t_start)
    if config.precision == "f32":
        from .batch import solve_batch_f32

        res = solve_batch_f32([query], corpus, embeddings, config, ws)[0]
        if isinstance(res, Exception):
            raise res
        return res
    if (config.tol is None and isinstance(query, np.ndarray) and query.dtype == np.float64
            and query.ndim == 1 and query.flags.c_contiguous and corpus.n_cols > 0
            and cuda_ok()):
        # native runtime: one C call does select -> H2D -> kernels -> D2H
        dev = device()
        dc = DeviceCorpus.of(corpus, dev)
        de = DeviceEmbeddings.of(embeddings, dev)
        plan = _native_plan(ws, dc, de, dev)
        rc, wmd = plan.run(query, config)
        if rc == -2:
            raise ValueError("query histogram must be nonnegative")
        if rc == -3:
            raise EmptyQueryError("query histogram has no positive entries")
        if rc > 0:
            raise _lib.NativeError(f"swmd_plan_run: CUDA error {rc}")
        if rc == 0 and plan.err[0] == _lib.NO_EVENT and plan.err[1] == _lib.NO_EVENT:
            t = plan.times
            timings = {"select": float(t[2]) / 1e3, "distances": float(t[0]) / 1e3,
                       "precompute": 0.0, "init": 0.0, "iterations": float(t[1]) / 1e3,
                       "final": 0.0, "total": time.perf_counter() - t_start}   # PHASES order
            return SolverResult(wmd=wmd, iterations_run=config.max_iter, converged=False,
                                timings=timings)
        # rc == -4 (outside the native fast path) or a degeneracy to decode:
        # the general path below reproduces the reference's error exactly
    t0 = time.perf_counter()
    v_r = _stage_query(query, n_vocab, ws)
    t_select = time.perf_counter() - t0
    dev = device()
    dc = DeviceCorpus.of(corpus, dev)
    de = DeviceEmbeddings.of(embeddings, dev)
    res = solve_on_device(None, None, dc, de, config, ws, staged_v_r=v_r)
    if res.event is not None:
        raise DegeneracyError(res.event.message)
    host = {"select": t_select, "total": time.perf_counter() - t_start}
    return SolverResult(wmd=res.wmd, iterations_run=res.iterations, converged=res.converged,
                        timings=phase_timings(host, res.timings))


def sinkhorn_wmd_devices(query, corpus, embeddings, config: SolverConfig,
                         devices: list[torch.device], workspace: SinkhornWorkspace | None = None,
                         t_start: float | None = None) -> SolverResult:
    """``sinkhorn_wmd`` with the document columns split over ``devices`` in
    this one process: the reference's ``workers`` (solver.py:35, threads over
    nnz-balanced column blocks, sparse.py:261-276) become GPUs.  Each device
    gets a contiguous column_blocks shard (uploaded once, cached on the
    corpus), builds K itself and runs the persistent solve on its own stream;
    the host enqueues every device before it waits on any, then reads each
    block back.  With ``tol`` the devices step in lockstep and share one
    global max|dx| (solver.py:179-183).  A device may appear more than once
    (one block per entry).  Results are bitwise those of the one-launch solve."""
    from .sparse import column_blocks

    t_start = time.perf_counter() if t_start is None else t_start
    ws = workspace if workspace is not None else _default_ws()
    t0 = time.perf_counter()
    sel, weights = select_nonzero(query)
    t_select = time.perf_counter() - t0
    col_ptr = corpus.csc_compact()[0] if hasattr(corpus, "csc_compact") else corpus.csc_index()[0]
    bounds = column_blocks(col_ptr, len(devices))
    shard_ws = ws.__dict__.setdefault("_shard_ws", {})
    plans, evs = [], []
    for k, dev in enumerate(devices):
        c0, c1 = int(bounds[k]), int(bounds[k + 1])
        if c1 <= c0:
            continue
        with torch.cuda.device(dev):
            sws = shard_ws.setdefault(k, SinkhornWorkspace())
            dc = DeviceCorpus.block_of(corpus, dev, c0, c1)
            de = DeviceEmbeddings.of(embeddings, dev)
            plan = QueryPlan(sel, weights, dc, de, config, sws)
            ev = _Events(True)
            ev.mark("d0")
            plan.enqueue_distances()
            ev.mark("d1")
            if config.tol is None:
                plan.enqueue_solve()
                ev.mark("i1")
            plans.append((c0, c1, plan))
            evs.append(ev)
    iterations, converged, failed = config.max_iter, False, False
    if config.tol is not None:
        for _, _, plan in plans:
            with torch.cuda.device(plan.dev):
                plan.tol_begin()
        iterations = 0
        for t in range(config.max_iter):
            for _, _, plan in plans:
                with torch.cuda.device(plan.dev):
                    plan.tol_launch(t)
            reads = [plan.tol_read() for _, _, plan in plans]
            iterations += 1
            if any(f for f, _ in reads):
                failed = True
                break
            if max(d for _, d in reads) < config.tol:   # NaN never converges (np.max)
                converged = True
                break
        for (_, _, plan), ev in zip(plans, evs):
            with torch.cuda.device(plan.dev):
                if not failed:
                    plan.tol_final(iterations)
                ev.mark("i1")
    wmd = np.empty(corpus.n_cols, dtype=np.float64)
    events = []
    for c0, c1, plan in plans:
        with torch.cuda.device(plan.dev):
            part, he = plan.readback()
            events.append(plan.decode_event(he))
        wmd[c0:c1] = part
    from .distributed import merge_events

    ev0 = merge_events(events)
    if ev0 is not None:
        raise DegeneracyError(ev0.message)
    spans = [_device_spans(e) for e in evs]
    dev_t = {k: max(sp[k] for sp in spans) for k in spans[0]} if spans else {}
    return SolverResult(wmd=wmd, iterations_run=iterations, converged=converged,
                        timings=phase_timings({"select": t_select,
                                               "total": time.perf_counter() - t_start}, dev_t))


@dataclass(frozen=True)
class TopKResult:
    """The k nearest documents of one query: ``indices`` ascending by distance,
    ties toward the lower document id (np.argsort(wmd, kind="stable")[:k]),
    and their distances ``wmd``."""

    indices: np.ndarray
    wmd: np.ndarray
    iterations_run: int
    converged: bool
    timings: dict[str, float]


def sinkhorn_wmd_topk(query, corpus, embeddings, config: SolverConfig, k: int,
                      workspace: SinkhornWorkspace | None = None) -> TopKResult:
    """``sinkhorn_wmd`` followed by a device top-k: only the k nearest
    documents cross PCIe (k <= 1024; fp64 path)."""
    t_start = time.perf_counter()
    if not 1 <= int(k) <= 1024:
        raise ValueError(f"k must be in [1, 1024], got {k}")
    if config.precision != "f64":
        raise ValueError("sinkhorn_wmd_topk runs the fp64 path")
    if isinstance(query, SparseVector):
        query = query.to_dense()
    query = np.asarray(query, dtype=np.float64)
    n_vocab = corpus.n_rows
    if query.shape != (n_vocab,) or tuple(embeddings.shape)[0] != n_vocab:
        raise ValueError(
            f"shape mismatch: query {query.shape}, embeddings "
            f"{tuple(embeddings.shape)}, corpus rows {n_vocab}")
    ws = workspace if workspace is not None else _default_ws()
    t0 = time.perf_counter()
    v_r = _stage_query(query, n_vocab, ws)
    t_select = time.perf_counter() - t0
    dev = device()
    dc = DeviceCorpus.of(corpus, dev)
    de = DeviceEmbeddings.of(embeddings, dev)
    ev = _Events(True)
    plan = QueryPlan(None, None, dc, de, config, ws, staged_v_r=v_r)
    ev.mark("d0")
    plan.enqueue_distances()
    ev.mark("d1")
    if config.tol is None:
        plan.enqueue_solve()
        iterations, converged = config.max_iter, False
    else:
        iterations, converged = plan.run_tol()
    ev.mark("i1")
    k = min(int(k), dc.n_cols)
    dws = plan.dws
    nb = int(_lib.lib().swmd_topk_scratch_bytes(dc.n_cols, k))
    scratch = dws.flat("topk_scratch", (nb + 7) // 8, torch.int64)
    res = dws.flat("topk_out", 2 * k, torch.int64)
    _lib.call("swmd_topk_f64", plan.wmd.data_ptr(), dc.n_cols, k, dc.col_offset,
              res.data_ptr(), res.data_ptr() + 8 * k, scratch.data_ptr(), nb, plan.stream)
    host = ws.pinned("topk_host", 2 * k + _lib.ERR_WORDS, torch.int64)
    host[: 2 * k].copy_(res, non_blocking=True)
    host[2 * k:].copy_(plan.err, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    hn = host.numpy()
    event = plan.decode_event(hn[2 * k:].copy())
    if event is not None:
        raise DegeneracyError(event.message)
    host_t = {"select": t_select, "total": time.perf_counter() - t_start}
    return TopKResult(indices=hn[:k].copy(), wmd=hn[k: 2 * k].view(np.float64).copy(),
                      iterations_run=iterations, converged=converged,
                      timings=phase_timings(host_t, _device_spans(ev)))


def sinkhorn_wmd_batch(queries, corpus, embeddings, config: SolverConfig,
                       workspace: SinkhornWorkspace | None = None) -> list:
    """Independent solves sharing one workspace; a failing query yields its
    exception instead of aborting the batch (solver.py:204-223)."""
    ws = workspace if workspace is not None else SinkhornWorkspace()
    if config.precision == "f32":
        from .batch import solve_batch_f32

        return solve_batch_f32(list(queries), corpus, embeddings, config, ws)
    results: list = []
    for q in queries:
        try:
            results.append(sinkhorn_wmd(q, corpus, embeddings, config, workspace=ws))
        except (ValueError, ArithmeticError) as exc:
            results.append(exc)
    return results
