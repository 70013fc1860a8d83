"""Operator surface of the hot path, backed by the sm_100a kernels.

Same names, signatures, error types and messages as the reference's
``sinkwmd.kernels`` (kernels.py:38-387): numpy arrays in, numpy arrays out,
outputs optionally written into caller buffers.  Every numeric operation runs
on the GPU through libswmd.so (include/swmd.h); there is no CPU fallback.

``workers`` / ``deterministic`` / ``partitions`` are accepted for
compatibility.  The device path is always column-owned (one warp per document
column, rows in increasing order), so results never depend on them; the
reference's argument checks (partitions rejected in deterministic mode,
counts refused in deterministic multi-worker mode) are kept, and ``counts``
receives the exact multiply-accumulate count 2*nnz*v_r split the way the
reference's workers would have split it (kernels.py:258-269).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .device import DeviceCorpus, device, stream_ptr
from .sparse import CsrMatrix, NnzPartition, nnz_partition

__all__ = [
    "EmptyQueryError",
    "DegeneracyError",
    "SinkhornMatrices",
    "select_nonzero",
    "euclidean_rows",
    "precompute",
    "sddmm",
    "spmm",
    "fused_iteration",
    "fused_final",
    "warmup",
    "COST_MODE_DIRECT",
    "COST_MODE_GRAM",
]

COST_MODE_DIRECT = 0   # reference operation order, bitwise-identical distances
COST_MODE_GRAM = 1     # ||e||^2 + ||q||^2 - 2 e.q with exact self-distance


class EmptyQueryError(ValueError):
    """A query histogram has no positive entries (kernels.py:38-39)."""


class DegeneracyError(ArithmeticError):
    """A sampled denominator is exactly zero, or an iterate entry is not
    positive (kernels.py:42-47, solver.py:95-103)."""


@dataclass(frozen=True)
class SinkhornMatrices:
    """Per-query matrices, each (V, v_r) (kernels.py:50-71)."""

    cost: np.ndarray
    kernel: np.ndarray
    kernel_over_r: np.ndarray
    kernel_cost: np.ndarray
    lam: float

    @property
    def v_r(self) -> int:
        return int(self.kernel.shape[1])


def select_nonzero(r_full) -> tuple[np.ndarray, np.ndarray]:
    """(sel, weights) of the positive entries, sel increasing (kernels.py:74-88)."""
    r_full = np.asarray(r_full, dtype=np.float64)
    if r_full.ndim != 1:
        raise ValueError("query histogram must be 1-D")
    if (r_full < 0.0).any():
        raise ValueError("query histogram must be nonnegative")
    sel = np.flatnonzero(r_full > 0.0)
    if sel.size == 0:
        raise EmptyQueryError("query histogram has no positive entries")
    return sel.astype(np.int64, copy=False), r_full[sel]


# -- error record ---------------------------------------------------------------

_KEY_BITS = 47
_KEY_MASK = (1 << _KEY_BITS) - 1


def new_err(dev: torch.device) -> torch.Tensor:
    err = torch.empty(_lib.ERR_WORDS, dtype=torch.int64, device=dev)
    _lib.call("swmd_err_reset", err.data_ptr(), stream_ptr(dev))
    return err


def zero_denominator_event(err_host: np.ndarray, n_key: int):
    """(code, i, j) of the recorded zero denominator, or None."""
    key = int(err_host[0])
    if key == _lib.NO_EVENT:
        return None
    code = key >> _KEY_BITS
    ij = key & _KEY_MASK
    i, j = divmod(ij, max(1, n_key))
    return code, int(i), int(j)


def raise_zero_denominator(i: int, j: int):
    raise DegeneracyError(f"zero denominator at nonzero ({i}, {j})")


def _check_err_single(err: torch.Tensor, n_key: int) -> None:
    ev = zero_denominator_event(err.cpu().numpy(), n_key)
    if ev is not None:
        raise_zero_denominator(ev[1], ev[2])


# -- helpers ----------------------------------------------------------------------

def _dev_f64(a, dev) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.detach().to(dev, torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def _check_shapes(corpus, kernel: np.ndarray, u: np.ndarray) -> None:
    """kernels.py:144-153."""
    v_r = kernel.shape[1]
    if kernel.shape[0] != corpus.n_rows:
        raise ValueError(f"kernel rows {kernel.shape[0]} != corpus rows {corpus.n_rows}")
    if u.shape != (corpus.n_cols, v_r):
        raise ValueError(
            f"iterate shape {u.shape} != (n_docs, v_r) = ({corpus.n_cols}, {v_r})")


def _reject_partitions_in_deterministic_mode(partitions) -> None:
    if partitions is not None:
        raise ValueError("explicit nonzero partitions require deterministic=False")


def _to_out(t: torch.Tensor, out: np.ndarray | None) -> np.ndarray:
    host = t.cpu().numpy()
    if out is None:
        return host
    out[...] = host
    return out


# -- operations -----------------------------------------------------------------------

def euclidean_rows(vecs, sel, out: np.ndarray | None = None, workers: int = 1,
                   mode: int = COST_MODE_DIRECT) -> np.ndarray:
    """out[i, a] = ||vecs[sel[a]] - vecs[i]|| on the GPU (kernels.py:91-111).

    The default mode keeps the reference's operation order, so the distances
    are bitwise identical to it.
    """
    vecs = np.ascontiguousarray(vecs, dtype=np.float64)
    sel = np.ascontiguousarray(sel, dtype=np.int64)
    if sel.size and (sel.min() < 0 or sel.max() >= vecs.shape[0]):
        raise IndexError("selected word ids out of bounds")
    V, dim = vecs.shape
    if out is None:
        out = np.empty((V, sel.size), dtype=np.float64)
    if sel.size == 0 or V == 0:
        return out
    dev = device()
    E = _dev_f64(vecs, dev)
    s = torch.from_numpy(sel).to(dev)
    w = torch.ones(sel.size, dtype=torch.float64, device=dev)
    cost = torch.empty((V, sel.size), dtype=torch.float64, device=dev)
    K = torch.empty_like(cost)
    norms = None
    if mode == COST_MODE_GRAM:
        norms = torch.empty(V, dtype=torch.float64, device=dev)
        _lib.call("swmd_row_norms_f64", E.data_ptr(), V, dim, dim, norms.data_ptr(), stream_ptr(dev))
    _lib.call("swmd_cost_build_f64", E.data_ptr(), V, dim, dim, s.data_ptr(), sel.size,
              w.data_ptr(), 1.0, mode, norms.data_ptr() if norms is not None else None,
              None, 0, cost.data_ptr(), K.data_ptr(), None, None, sel.size, stream_ptr(dev))
    return _to_out(cost, out)


def precompute(cost, weights, lam: float, buffers=None, workers: int = 1) -> SinkhornMatrices:
    """K = exp(-lam*cost), K/r, K*cost on the GPU (kernels.py:114-141)."""
    if lam <= 0.0:
        raise ValueError(f"lam must be positive, got {lam}")
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    if np.any(weights <= 0.0):
        raise ValueError("query weights must be strictly positive")
    cost = np.asarray(cost, dtype=np.float64)
    V, v_r = cost.shape
    if buffers is None:
        kernel, kor, kcost = (np.empty_like(cost) for _ in range(3))
    else:
        kernel, kor, kcost = buffers
    if V and v_r:
        dev = device()
        c = _dev_f64(cost, dev)
        w = _dev_f64(weights, dev)
        K, KoR, KM = (torch.empty_like(c) for _ in range(3))
        _lib.call("swmd_precompute_f64", c.data_ptr(), V, v_r, v_r, w.data_ptr(), float(lam),
                  K.data_ptr(), KoR.data_ptr(), KM.data_ptr(), stream_ptr(dev))
        _to_out(K, kernel)
        _to_out(KoR, kor)
        _to_out(KM, kcost)
    return SinkhornMatrices(cost, kernel, kor, kcost, float(lam))


def _counts_fill(corpus, counts: np.ndarray, v_r: int, workers: int,
                 partitions: Sequence[NnzPartition] | None) -> None:
    """The reference's MAC instrumentation (_jit.py:186-236): 2*v_r per nonzero."""
    if workers == 1 and partitions is None:
        counts[0] = 2 * corpus.nnz * v_r
        return
    parts = partitions if partitions is not None else nnz_partition(
        corpus.row_ptr, corpus.nnz, workers)
    if counts.shape[0] != len(parts):
        raise ValueError("counts must have one slot per worker")
    for k, p in enumerate(parts):
        counts[k] = 2 * p.size * v_r


def sddmm(corpus, kernel, u, workers: int = 1, partitions=None,
          out: np.ndarray | None = None) -> np.ndarray:
    """w[z] = c_z / (kernel[i,:] . u[j,:]) in CSR storage order (kernels.py:177-208)."""
    kernel = np.asarray(kernel, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    _check_shapes(corpus, kernel, u)
    if out is None:
        out = np.empty(corpus.nnz, dtype=np.float64)
    dc = DeviceCorpus.of(corpus)
    if corpus.nnz == 0:
        return out
    dev = dc.device
    pos = dc.ensure_pos()
    K, U = _dev_f64(kernel, dev), _dev_f64(u, dev)
    w = torch.empty(corpus.nnz, dtype=torch.float64, device=dev)
    err = new_err(dev)
    _lib.call("swmd_sddmm_f64", dc.col_ptr.data_ptr(), dc.rows.data_ptr(), pos.data_ptr(),
              dc.vals.data_ptr(), dc.n_cols, K.data_ptr(), kernel.shape[1], kernel.shape[1],
              U.data_ptr(), w.data_ptr(), corpus.n_cols, err.data_ptr(), stream_ptr(dev))
    _to_out(w, out)
    _check_err_single(err, corpus.n_cols)
    return out


def spmm(corpus, w_values, kernel_over_r, workers: int = 1, deterministic: bool = False,
         partitions=None, x_out: np.ndarray | None = None) -> np.ndarray:
    """x_out[j,a] += sum_i kernel_over_r[i,a] * w(i,j) (kernels.py:211-247)."""
    kor = np.asarray(kernel_over_r, dtype=np.float64)
    w_values = np.asarray(w_values, dtype=np.float64)
    v_r = kor.shape[1]
    if w_values.shape != (corpus.nnz,):
        raise ValueError(f"w has {w_values.shape[0]} values, corpus nnz is {corpus.nnz}")
    if x_out is None:
        x_out = np.zeros((corpus.n_cols, v_r), dtype=np.float64)
    if deterministic:
        _reject_partitions_in_deterministic_mode(partitions)
    dc = DeviceCorpus.of(corpus)
    if corpus.nnz == 0:
        return x_out
    dev = dc.device
    pos = dc.ensure_pos()
    R, W, X = _dev_f64(kor, dev), _dev_f64(w_values, dev), _dev_f64(x_out, dev)
    _lib.call("swmd_spmm_f64", dc.col_ptr.data_ptr(), dc.rows.data_ptr(), pos.data_ptr(),
              W.data_ptr(), dc.n_cols, R.data_ptr(), v_r, v_r, X.data_ptr(), stream_ptr(dev))
    return _to_out(X, x_out)


def fused_iteration(corpus, mats: SinkhornMatrices, u, x_out: np.ndarray, workers: int = 1,
                    deterministic: bool = False, partitions=None,
                    counts: np.ndarray | None = None) -> None:
    """One type-1 fused SDDMM-SpMM pass accumulating into x_out (kernels.py:250-310)."""
    u = np.asarray(u, dtype=np.float64)
    _check_shapes(corpus, mats.kernel, u)
    if x_out.shape != u.shape:
        raise ValueError(f"x_out shape {x_out.shape} != u shape {u.shape}")
    if deterministic:
        _reject_partitions_in_deterministic_mode(partitions)
    if counts is not None:
        if deterministic and workers > 1:
            raise ValueError("instrumentation is unavailable in deterministic mode")
        _counts_fill(corpus, counts, mats.v_r, workers, partitions)
    dc = DeviceCorpus.of(corpus)
    if corpus.nnz == 0:
        return
    dev = dc.device
    v_r = mats.v_r
    K, KoR = _dev_f64(mats.kernel, dev), _dev_f64(mats.kernel_over_r, dev)
    U, X = _dev_f64(u, dev), _dev_f64(x_out, dev)
    err = new_err(dev)
    _lib.call("swmd_fused_iteration_f64", dc.col_ptr.data_ptr(), dc.rows.data_ptr(),
              dc.vals.data_ptr(), dc.n_cols, K.data_ptr(), KoR.data_ptr(), v_r, v_r,
              U.data_ptr(), X.data_ptr(), corpus.n_cols, err.data_ptr(), stream_ptr(dev))
    _to_out(X, x_out)
    _check_err_single(err, corpus.n_cols)


def fused_final(corpus, mats: SinkhornMatrices, u, workers: int = 1,
                deterministic: bool = False, partitions=None,
                out: np.ndarray | None = None) -> np.ndarray:
    """Type-2 distance pass (kernels.py:313-354); out is zeroed then filled."""
    u = np.asarray(u, dtype=np.float64)
    _check_shapes(corpus, mats.kernel, u)
    if out is None:
        out = np.zeros(corpus.n_cols, dtype=np.float64)
    elif out.shape != (corpus.n_cols,):
        raise ValueError(f"out shape {out.shape} != ({corpus.n_cols},)")
    else:
        out[:] = 0.0
    if deterministic:
        _reject_partitions_in_deterministic_mode(partitions)
    dc = DeviceCorpus.of(corpus)
    if corpus.n_cols == 0:
        return out
    dev = dc.device
    v_r = mats.v_r
    K, KM, U = _dev_f64(mats.kernel, dev), _dev_f64(mats.kernel_cost, dev), _dev_f64(u, dev)
    wmd = torch.zeros(corpus.n_cols, dtype=torch.float64, device=dev)
    err = new_err(dev)
    _lib.call("swmd_fused_final_f64", dc.col_ptr.data_ptr(), dc.rows.data_ptr(),
              dc.vals.data_ptr(), dc.n_cols, K.data_ptr(), KM.data_ptr(), v_r, v_r,
              U.data_ptr(), wmd.data_ptr(), corpus.n_cols, err.data_ptr(), stream_ptr(dev))
    _to_out(wmd, out)
    _check_err_single(err, corpus.n_cols)
    return out


_warmed = False


def warmup() -> None:
    """Load the library and touch every kernel once on a 2x2 instance
    (kernels.py:357-387), so timed sections never pay first-launch cost."""
    global _warmed
    if _warmed:
        return
    _lib.lib()
    corpus = CsrMatrix(2, 2, np.array([0, 1, 3]), np.array([0, 0, 1]), np.array([0.5, 0.5, 1.0]))
    vecs = np.array([[0.0, 0.0], [1.0, 0.0]])
    sel, weights = select_nonzero(np.array([0.5, 0.5]))
    mats = precompute(euclidean_rows(vecs, sel), weights, 1.0)
    u = np.full((2, 2), 1.0)
    x = np.zeros((2, 2))
    fused_iteration(corpus, mats, u, x)
    fused_final(corpus, mats, u)
    w = sddmm(corpus, mats.kernel, u)
    spmm(corpus, w, mats.kernel_over_r)
    from .solver import SolverConfig, sinkhorn_wmd
    sinkhorn_wmd(np.array([0.5, 0.5]), corpus, vecs, SolverConfig(lam=1.0, max_iter=2))
    torch.cuda.synchronize()
    _warmed = True
