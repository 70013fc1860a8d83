"""Multi-query fp32 variant: a whole batch of queries in one cost-build launch.

BASELINE config c4 (64 queries, v_r in [8, 64], N=100k documents, fp32,
max_iter=20, tolerance 1e-4 vs the fp64 oracle).  The reference is fp64-only
and solves a batch one query at a time (``sinkhorn_wmd_batch``,
solver.py:204-223); this path keeps its contract — one ``SolverResult`` or
exception per query, a failing query never aborts the batch — and batches the
work the B200 way:

* the selected words of every query are concatenated and ONE fp32 GEMM
  (``swmd_cost_build_batch_f32``) builds K and K*M for all of them, reading
  the (fp32, resident) embedding table once per 64 output columns;
* each query's K block is a 16-byte-aligned column range of that matrix,
  zero-padded to v_r rounded to 8, and the fp32 solve kernel reads it in
  place (row stride = the batch width);
* queries of one padded width are solved GROUP (4) at a time in one
  persistent launch (``swmd_solve_group_f32``): a claimed column is solved
  for each query of the group in turn, so its CSC entries are fetched from
  HBM once per group instead of once per query;
* one device->host copy returns every query's distances and error record.
"""

from __future__ import annotations

import os
import time

import numpy as np
import torch

from . import _lib
from .device import DeviceCorpus, DeviceEmbeddings, device, stream_ptr
from .kernels import DegeneracyError, select_nonzero, zero_denominator_event
from .solver import nonpositive_fires
from .sparse import SparseVector

__all__ = ["solve_batch_f32"]

last_launches = 0   # kernels the last tol-unset batch launched (bench.py reports it)

_INT64_MAX = (1 << 63) - 1


def _block_width(v_r: int) -> int:
    return (v_r + 7) // 8 * 8 if v_r <= 64 else (v_r + 3) // 4 * 4


def _solve32(dc, K_ptr, KM_ptr, r_ptr, v_r, LD, t0, t1, x_in, x_out, wmd_ptr, err_ptr, counter, s):
    _lib.call("swmd_solve_f32", dc.col_ptr.data_ptr(), dc.rows.data_ptr(), dc.vals.data_ptr(),
              dc.n_cols, dc.order.data_ptr(), K_ptr, KM_ptr, r_ptr, v_r, LD, t0, t1,
              x_in, x_out, wmd_ptr, dc.col_offset, dc.n_key, dc.max_len, err_ptr,
              counter.data_ptr(), s)


# queries per group launch (swmd_solve_group_f32 takes up to 4): their K blocks
# (4 x ~14 MB at c4) stay L2-resident together while a column is solved for each
GROUP = 4


def _solve_group32(dc, members, LD, max_iter, counter, s):
    import ctypes

    nq = len(members)
    P = ctypes.c_void_p * nq
    kp = P(*[m[0] for m in members])
    kmp = P(*[m[1] for m in members])
    rp = P(*[m[2] for m in members])
    wp = P(*[m[3] for m in members])
    ep = P(*[m[4] for m in members])
    vr = (ctypes.c_int32 * nq)(*[m[5] for m in members])
    _lib.call("swmd_solve_group_f32", dc.col_ptr.data_ptr(), dc.rows.data_ptr(), dc.vals.data_ptr(),
              dc.n_cols, dc.order.data_ptr(), nq, ctypes.addressof(kp), ctypes.addressof(kmp),
              ctypes.addressof(rp), ctypes.addressof(vr), LD, max_iter, ctypes.addressof(wp),
              ctypes.addressof(ep), dc.col_offset, dc.n_key, counter.data_ptr(), s)


def _reset_err(err: torch.Tensor) -> None:
    e = err.view(-1, _lib.ERR_WORDS)
    e[:, 0] = _INT64_MAX
    e[:, 1] = _INT64_MAX
    e[:, 2] = 0
    e[:, 3] = _INT64_MAX


# widest query the fp32 solve kernels take (swmd_solve_f32: CTA per column up
# to 256 words); wider queries of a batch run on the fp64 path
F32_MAX_V_R = 256


def solve_batch_f32(queries, corpus, embeddings, config, ws) -> list:
    """``sinkhorn_wmd_batch`` semantics in fp32 (see module docstring).

    A query wider than F32_MAX_V_R words is solved by the fp64 path instead
    (its result is at least as accurate), so one wide query never aborts the
    batch."""
    from .solver import SolverResult, select_native, sinkhorn_wmd

    t_start = time.perf_counter()
    n_vocab = corpus.n_rows
    emb_shape = tuple(embeddings.shape)
    results: list = [None] * len(queries)
    items, wide = [], []
    t0 = time.perf_counter()
    for k, q in enumerate(queries):
        try:
            if isinstance(q, SparseVector):
                q = q.to_dense()
            q = np.asarray(q, dtype=np.float64)
            if q.shape != (n_vocab,) or emb_shape[0] != n_vocab:
                raise ValueError(f"shape mismatch: query {q.shape}, embeddings {emb_shape}, "
                                 f"corpus rows {n_vocab}")
            if q.ndim == 1 and q.flags.c_contiguous and q.size:
                sel, w = select_native(q, ws)
            else:
                sel, w = select_nonzero(q)
            if sel.size > F32_MAX_V_R:
                wide.append((k, q))
                continue
            items.append((k, sel, w))
        except (ValueError, ArithmeticError) as exc:
            results[k] = exc
    t_select = time.perf_counter() - t0
    if wide:
        import dataclasses

        cfg64 = dataclasses.replace(config, precision="f64")
        emb64 = np.asarray(embeddings, dtype=np.float64) if not hasattr(embeddings, "device") \
            else embeddings
        for k, q in wide:
            try:
                results[k] = sinkhorn_wmd(q, corpus, emb64, cfg64, workspace=ws)
            except (ValueError, ArithmeticError) as exc:
                results[k] = exc
    if not items:
        return results

    dev = device()
    s = stream_ptr(dev)
    dc = DeviceCorpus.of(corpus, dev)
    de = DeviceEmbeddings.of(embeddings, dev, dtype=torch.float32)
    dws = ws.on(dev)
    V, N = dc.n_rows, dc.n_cols
    # column layout of the batch
    offs, woffs, off, woff = [], [], 0, 0
    for _, sel, _ in items:
        offs.append(off)
        woffs.append(woff)
        off += _block_width(sel.size)
        woff += sel.size
    LD = (off + 3) // 4 * 4
    words = np.concatenate([sel for _, sel, _ in items]).astype(np.int64)
    weights = np.concatenate([w for _, _, w in items]).astype(np.float32)
    col_word = np.full(LD, -1, dtype=np.int32)
    for (_, sel, _), o, wo in zip(items, offs, woffs):
        col_word[o: o + sel.size] = np.arange(wo, wo + sel.size, dtype=np.int32)
    words_d = torch.from_numpy(words).to(dev, non_blocking=True)
    col_d = torch.from_numpy(col_word).to(dev, non_blocking=True)
    w_d = torch.from_numpy(weights).to(dev, non_blocking=True)

    K = dws.flat("k32", V * LD, torch.float32)
    KM = dws.flat("km32", V * LD, torch.float32)
    use_list = dc.present_rows is not None and dc.n_present < V
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    _lib.call("swmd_cost_build_batch_f32", de.E.data_ptr(), de.V, de.dim, de.ld,
              words_d.data_ptr(), col_d.data_ptr(), LD, float(config.lam), de.norms.data_ptr(),
              dc.present_rows.data_ptr() if use_list else None,
              dc.n_present if use_list else 0, K.data_ptr(), KM.data_ptr(), s)
    ev[1].record()

    nq = len(items)
    out = dws.flat("wmd32", nq * N, torch.float32)
    err = dws.flat("err32", nq * _lib.ERR_WORDS, torch.int64)
    counter = dws.flat("counter32", 1, torch.int32)
    _reset_err(err)
    iters = [config.max_iter] * nq
    conv = [False] * nq
    ptrs = []
    for n, ((k, sel, _), o, wo) in enumerate(zip(items, offs, woffs)):
        ptrs.append((K.data_ptr() + 4 * o, KM.data_ptr() + 4 * o, w_d.data_ptr() + 4 * wo,
                     out.data_ptr() + 4 * n * N, err.data_ptr() + 8 * n * _lib.ERR_WORDS,
                     int(sel.size)))
    launches = 2   # the Gram build + the error-record reset
    if config.tol is None:
        # queries of one padded width share a launch, GROUP at a time: each
        # claimed column is solved for every query of the group in turn
        by_width: dict[int, list[int]] = {}
        for n, p in enumerate(ptrs):
            if p[5] <= 64:
                by_width.setdefault(_block_width(p[5]), []).append(n)
            else:
                Kp, KMp, rp, wmd_p, err_p, v_r = p
                _solve32(dc, Kp, KMp, rp, v_r, LD, 0, config.max_iter, None, None, wmd_p,
                         err_p, counter, s)
                launches += 1
        for members in by_width.values():
            for g0 in range(0, len(members), GROUP):
                _solve_group32(dc, [ptrs[n] for n in members[g0: g0 + GROUP]], LD,
                               config.max_iter, counter, s)
                launches += 1
        global last_launches
        last_launches = launches
    else:
        for n, (Kp, KMp, rp, wmd_p, err_p, v_r) in enumerate(ptrs):
            iters[n], conv[n] = _tol_loop(dc, Kp, KMp, rp, v_r, LD, wmd_p, err, n,
                                          counter, s, config, dws)
    ev[2].record()
    # the float64 results the reference returns, widened on the device (a host
    # astype of 64 x 100k floats costs more than the transfer), then one pinned
    # device->host copy of every query's distances and error record
    out64 = dws.flat("wmd64", nq * N)
    out64.copy_(out)
    host = ws.pinned("batch32_out", nq * N + nq * _lib.ERR_WORDS, torch.int64)
    h_wmd = host[: nq * N].view(torch.float64)
    h_err = host[nq * N:]
    h_wmd.copy_(out64, non_blocking=True)
    h_err.copy_(err, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    wmd_h = np.empty((nq, N), dtype=np.float64)      # detached from the pinned workspace
    _lib.call("swmd_host_copy", wmd_h.ctypes.data, h_wmd.data_ptr(), wmd_h.nbytes,
              min(16, os.cpu_count() or 1))
    err_h = h_err.numpy().reshape(nq, _lib.ERR_WORDS)
    t_dist = ev[0].elapsed_time(ev[1]) / 1e3
    t_iter = ev[1].elapsed_time(ev[2]) / 1e3
    t_total = time.perf_counter() - t_start
    for n, ((k, sel, _), o, wo) in enumerate(zip(items, offs, woffs)):
        msg = _error_message(err_h[n], dc, K.data_ptr() + 4 * o, KM.data_ptr() + 4 * o,
                             w_d.data_ptr() + 4 * wo, sel.size, LD, counter, s, dws)
        if msg is not None:
            results[k] = DegeneracyError(msg)
            continue
        timings = {"select": t_select / nq, "distances": t_dist / nq, "precompute": 0.0,
                   "init": 0.0, "iterations": t_iter / nq, "final": 0.0, "total": t_total / nq}
        results[k] = SolverResult(wmd=wmd_h[n], iterations_run=iters[n],
                                  converged=conv[n], timings=timings)
    return results


def _tol_loop(dc, Kp, KMp, rp, v_r, LD, wmd_p, err, n, counter, s, config, dws):
    """Per-iteration launches with the max-norm change read back (solver.py:170-183)."""
    N = dc.n_cols
    bufs = (dws.flat("x32a", N * v_r, torch.float32), dws.flat("x32b", N * v_r, torch.float32))
    e = err.view(-1, _lib.ERR_WORDS)[n]
    err_p = e.data_ptr()
    cur, iterations, converged = None, 0, False
    for t in range(config.max_iter):
        nxt = bufs[t % 2]
        e[2] = 0
        _solve32(dc, Kp, KMp, rp, v_r, LD, t, t + 1, cur.data_ptr() if cur is not None else None,
                 nxt.data_ptr(), None, err_p, counter, s)
        he = e.cpu().numpy()
        iterations += 1
        cur = nxt
        if he[0] != _INT64_MAX or nonpositive_fires(he):
            return iterations, False
        if float(he[2:3].view(np.float64)[0]) < config.tol:
            converged = True
            break
    _solve32(dc, Kp, KMp, rp, v_r, LD, iterations, iterations, cur.data_ptr(), None, wmd_p,
             err_p, counter, s)
    return iterations, converged


def _error_message(he, dc, Kp, KMp, rp, v_r, LD, counter, s, dws):
    zd = zero_denominator_event(he, dc.n_key)
    code_zero = zd[0] if zd is not None else None
    code_np = int(he[1]) if nonpositive_fires(he) else None
    if code_np is not None and (code_zero is None or code_np < code_zero):
        # replay to the failing check with x stored (rare error path)
        N = dc.n_cols
        xa = dws.flat("x32ra", N * v_r, torch.float32)
        xb = dws.flat("x32rb", N * v_r, torch.float32)
        e = torch.empty(_lib.ERR_WORDS, dtype=torch.int64, device=dc.device)
        cur = None
        for t in range(code_np // 2):
            nxt = (xa, xb)[t % 2]
            _reset_err(e)
            _solve32(dc, Kp, KMp, rp, v_r, LD, t, t + 1,
                     cur.data_ptr() if cur is not None else None, nxt.data_ptr(), None,
                     e.data_ptr(), counter, s)
            cur = nxt
        flat_local = int(torch.argmin(cur).item())
        val = float(cur[flat_local].item())
        return f"nonpositive iterate entry {val} at flat index {dc.col_offset * v_r + flat_local}"
    if zd is not None:
        return f"zero denominator at nonzero ({zd[1]}, {zd[2]})"
    return None
