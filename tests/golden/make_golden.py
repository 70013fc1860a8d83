"""Generate the golden fixtures from the REFERENCE package itself.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    python tests/golden/make_golden.py [small c1 c2 c3 c5]

Outputs (committed):
  small.npz  - 50 small seeded instances built by the reference's own
               ``synth.random_instance`` (the envelope of its acceptance
               suite, test_acceptance.py:37-49) with their inputs, the
               reference's per-kernel outputs and its solver output for
               lam in {1, 10}.
  c1.npz, c2.npz - full ``wmd`` of the reference solver on the seeded
               Zipf configs (paper_2107_06433_b200.synth), plus sha256
               fingerprints of the generated inputs.
  c3.npz, c5.npz - reference top-100 (stable argsort), the top-101 indices
               and values (the (k+1)-th decides boundary near-ties), sum, and
               a strided sample of ``wmd`` (the full vectors are too big to
               commit).
  c4.npz      - 64 fp64 reference solves of the c4 instance: top-11, sums,
               samples.
  tol.npz     - the reference's ``tol`` early exit (solver.py:170-183):
               iterations_run, converged, wmd and the per-iteration
               max|x - x_prev| of its loop, on c1/c2-shaped and small cases.

The reference runs with SolverConfig(deterministic=True, workers=os.cpu_count()),
which is bitwise equal to its serial mode (test_acceptance.py:126-151).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import sinkwmd  # noqa: E402  (the reference)
from sinkwmd.sparse import CsrMatrix  # noqa: E402
from sinkwmd.synth import random_instance  # noqa: E402

from paper_2107_06433_b200 import synth  # noqa: E402


def fingerprint(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def make_small():
    """Reference kernel + solver outputs on its own small random instances."""
    out = {}
    for k in range(50):
        seed = 1000 + k
        rng = np.random.default_rng(seed)
        n_vocab = int(rng.integers(8, 65))
        n_docs = int(rng.integers(2, 17))
        v_r = int(rng.integers(1, min(8, n_vocab) + 1))
        dim = int(rng.integers(2, 9))
        inst = random_instance(seed, n_vocab=n_vocab, n_docs=n_docs, v_r=v_r,
                               dim=dim, density=0.25)
        c = inst.corpus
        p = f"i{k}_"
        out[p + "emb"] = inst.embeddings
        out[p + "query"] = inst.query
        out[p + "row_ptr"] = c.row_ptr
        out[p + "col_idx"] = c.col_idx
        out[p + "values"] = c.values
        out[p + "shape"] = np.array([c.n_rows, c.n_cols])
        for lam in (1.0, 10.0):
            cfg = sinkwmd.SolverConfig(lam=lam, max_iter=15)
            out[p + f"wmd_lam{int(lam)}"] = sinkwmd.sinkhorn_wmd(
                inst.query, c, inst.embeddings, cfg).wmd
        sel, weights = sinkwmd.select_nonzero(inst.query)
        cost = sinkwmd.euclidean_rows(inst.embeddings, sel)
        mats = sinkwmd.precompute(cost, weights, 10.0)
        out[p + "cost"] = cost
        out[p + "kernel"] = mats.kernel
        out[p + "kor"] = mats.kernel_over_r
        out[p + "kcost"] = mats.kernel_cost
        u = np.random.default_rng(seed + 7).random((c.n_cols, sel.size)) + 0.1
        out[p + "u"] = u
        x = np.zeros_like(u)
        sinkwmd.fused_iteration(c, mats, u, x)
        out[p + "x1"] = x
        out[p + "final"] = sinkwmd.fused_final(c, mats, u)
        out[p + "sddmm"] = sinkwmd.sddmm(c, mats.kernel, u)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print("small.npz: 50 instances")


def make_config(name: str, full: bool):
    cfg = synth.CONFIGS[name]
    t0 = time.time()
    inst = synth.zipf_instance(cfg)
    rp, ci, v = synth.csc_to_csr(inst.n_vocab, inst.n_docs, inst.col_ptr, inst.rows, inst.vals)
    corpus = CsrMatrix(inst.n_vocab, inst.n_docs, rp, ci, v)
    t1 = time.time()
    corpus.csc_index()
    t2 = time.time()
    scfg = sinkwmd.SolverConfig(lam=cfg.lam, max_iter=cfg.max_iter,
                                workers=os.cpu_count() or 1, deterministic=True)
    res = sinkwmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, scfg)
    t3 = time.time()
    wmd = res.wmd
    order = np.argsort(wmd, kind="stable")
    out = dict(
        config=np.array(name),
        seed=np.array(cfg.seed),
        nnz=np.array(inst.nnz),
        fp_corpus=np.array(fingerprint(inst.col_ptr, inst.rows, inst.vals)),
        fp_query=np.array(fingerprint(inst.query)),
        fp_embeddings=np.array(fingerprint(inst.embeddings)),
        top100=order[:100],
        top100_wmd=wmd[order[:100]],
        top101=order[:101],
        top101_wmd=wmd[order[:101]],
        wmd_sum=np.array(float(np.sum(wmd))),
        sample_stride=np.array(max(1, wmd.size // 1000)),
        sample=wmd[:: max(1, wmd.size // 1000)],
        ref_timings=np.array([res.timings[k] for k in
                              ("select", "distances", "precompute", "init",
                               "iterations", "final", "total")]),
        ref_workers=np.array(os.cpu_count() or 1),
    )
    if full:
        out["wmd"] = wmd
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}.npz: nnz={inst.nnz} gen {t1 - t0:.1f}s csc {t2 - t1:.1f}s "
          f"solve {t3 - t2:.2f}s timings {res.timings}")


def make_c4():
    """64 fp64 reference solves on the c4 instance (the fp32 path is checked
    against these within 1e-4)."""
    cfg = synth.CONFIGS["c4"]
    t0 = time.time()
    inst = synth.zipf_instance(cfg)
    rp, ci, v = synth.csc_to_csr(inst.n_vocab, inst.n_docs, inst.col_ptr, inst.rows, inst.vals)
    corpus = CsrMatrix(inst.n_vocab, inst.n_docs, rp, ci, v)
    corpus.csc_index()
    scfg = sinkwmd.SolverConfig(lam=cfg.lam, max_iter=cfg.max_iter,
                                workers=os.cpu_count() or 1, deterministic=True)
    E64 = inst.embeddings.astype(np.float64)
    stride = max(1, inst.n_docs // 500)
    tops, topv, sums, samples, vrs = [], [], [], [], []
    for q in inst.queries:
        res = sinkwmd.sinkhorn_wmd(q, corpus, E64, scfg)
        order = np.argsort(res.wmd, kind="stable")
        tops.append(order[:11])
        topv.append(res.wmd[order[:11]])
        sums.append(float(np.sum(res.wmd)))
        samples.append(res.wmd[::stride])
        vrs.append(int(np.count_nonzero(q)))
    np.savez_compressed(
        os.path.join(HERE, "c4.npz"), config=np.array("c4"), seed=np.array(cfg.seed),
        nnz=np.array(inst.nnz),
        fp_corpus=np.array(fingerprint(inst.col_ptr, inst.rows, inst.vals)),
        fp_embeddings=np.array(fingerprint(inst.embeddings)),
        top10=np.array(tops)[:, :10], top10_wmd=np.array(topv)[:, :10],
        top11=np.array(tops), top11_wmd=np.array(topv), wmd_sum=np.array(sums),
        sample_stride=np.array(stride), sample=np.array(samples), v_r=np.array(vrs))
    print(f"c4.npz: nnz={inst.nnz} queries={len(inst.queries)} v_r={vrs[:8]}... "
          f"{time.time() - t0:.1f}s")


def _ref_tol_run(query, corpus, emb, lam, max_iter, tol):
    """The reference solver's result plus the max|x - x_prev| of every
    iteration, recomputed by the reference's own pieces in its loop order
    (solver.py:160-183: update_u, fused_iteration, max-norm check)."""
    scfg = sinkwmd.SolverConfig(lam=lam, max_iter=max_iter, tol=tol,
                                workers=os.cpu_count() or 1, deterministic=True)
    res = sinkwmd.sinkhorn_wmd(query, corpus, emb, scfg)
    sel, weights = sinkwmd.select_nonzero(query)
    mats = sinkwmd.precompute(sinkwmd.euclidean_rows(emb, sel), weights, lam)
    x = np.full((corpus.n_cols, sel.size), 1.0 / sel.size)
    deltas = []
    for _ in range(res.iterations_run):
        u = sinkwmd.solver.update_u(x)
        xn = np.zeros_like(x)
        sinkwmd.fused_iteration(corpus, mats, u, xn, workers=os.cpu_count() or 1,
                                deterministic=True)
        deltas.append(float(np.max(np.abs(xn - x))))
        x = xn
    return res, np.array(deltas)


def make_tol():
    """Pinned tol semantics: c1 and c2-shaped Zipf instances at lam=1 (the
    reference's own tol test uses lam=1, test_solver.py:112-129), a run
    that exhausts max_iter, and small random instances."""
    out = {}
    cases = []
    for name, n_docs, lam, max_iter, tol in [("c1", None, 1.0, 500, 1e-9),
                                             ("c2", 1000, 1.0, 500, 1e-9),
                                             ("c2", 1000, 1.0, 6, 1e-12),
                                             ("c1", None, 10.0, 200, 1e-7)]:
        inst = synth.zipf_instance(name, n_docs=n_docs)
        rp, ci, v = synth.csc_to_csr(inst.n_vocab, inst.n_docs, inst.col_ptr, inst.rows, inst.vals)
        corpus = CsrMatrix(inst.n_vocab, inst.n_docs, rp, ci, v)
        res, deltas = _ref_tol_run(inst.query, corpus, inst.embeddings, lam, max_iter, tol)
        cases.append((f"{name}:{n_docs or 0}", lam, max_iter, tol, res, deltas))
    for k in range(6):
        seed = 1000 + k
        rng = np.random.default_rng(seed)
        n_vocab = int(rng.integers(8, 65))
        n_docs = int(rng.integers(2, 17))
        v_r = int(rng.integers(1, min(8, n_vocab) + 1))
        dim = int(rng.integers(2, 9))
        inst = random_instance(seed, n_vocab=n_vocab, n_docs=n_docs, v_r=v_r, dim=dim,
                               density=0.25)
        res, deltas = _ref_tol_run(inst.query, inst.corpus, inst.embeddings, 1.0, 500, 1e-9)
        cases.append((f"small:{k}", 1.0, 500, 1e-9, res, deltas))
    for n, (spec, lam, max_iter, tol, res, deltas) in enumerate(cases):
        p = f"t{n}_"
        out[p + "spec"] = np.array(spec)
        out[p + "params"] = np.array([lam, max_iter, tol])
        out[p + "iterations"] = np.array(res.iterations_run)
        out[p + "converged"] = np.array(res.converged)
        out[p + "wmd"] = res.wmd
        out[p + "deltas"] = deltas
        print(f"tol case {spec} lam={lam} max_iter={max_iter} tol={tol}: "
              f"{res.iterations_run} iterations, converged={res.converged}, "
              f"last deltas {deltas[-3:]}")
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "tol.npz"), **out)


def main(argv):
    sinkwmd.kernels.warmup()
    which = argv or ["small", "c1", "c2", "c3", "c4", "c5", "tol"]
    for w in which:
        if w == "small":
            make_small()
        elif w == "tol":
            make_tol()
        elif w == "c4":
            make_c4()
        else:
            make_config(w, full=w in ("c1", "c2"))


if __name__ == "__main__":
    main(sys.argv[1:])
