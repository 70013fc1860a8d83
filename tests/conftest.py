"""Shared fixtures: the `gpu` marker, golden fixtures, the CPU oracle (checker only)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and libswmd.so")


def max_rel_err(got, want) -> float:
    """The reference's relative error (conftest.py:25-27, validation.py:32-34)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if want.size == 0:
        return 0.0
    denom = np.maximum(np.abs(want), np.finfo(np.float64).tiny)
    return float(np.max(np.abs(got - want) / denom))


def golden(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def small_golden():
    return golden("small")


def small_instance(g, k: int):
    """Inputs of golden small instance k as (query, CsrMatrix, embeddings)."""
    from paper_2107_06433_b200.sparse import CsrMatrix

    p = f"i{k}_"
    n_rows, n_cols = (int(v) for v in g[p + "shape"])
    corpus = CsrMatrix(n_rows, n_cols, g[p + "row_ptr"], g[p + "col_idx"], g[p + "values"])
    return g[p + "query"], corpus, g[p + "emb"]


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle

    oracle.lib()
    return oracle


def column_subset(corpus, cols):
    """Corpus restricted to the given columns, renumbered in order (conftest.py:16-22)."""
    from paper_2107_06433_b200.sparse import CsrMatrix

    cp, rows, _, vals = corpus.csc_index()
    cols = np.asarray(cols)
    new_cp = [0]
    r_out, v_out = [], []
    for c in cols:
        a, b = cp[c], cp[c + 1]
        r_out.append(rows[a:b])
        v_out.append(vals[a:b])
        new_cp.append(new_cp[-1] + (b - a))
    return CsrMatrix.from_csc(corpus.n_rows, len(cols), np.array(new_cp),
                              np.concatenate(r_out), np.concatenate(v_out))


def tol_case(g, n: int):
    """Inputs and parameters of tol golden case n (tests/golden/tol.npz):
    (query, CsrMatrix corpus, embeddings, lam, max_iter, tol)."""
    from paper_2107_06433_b200 import synth

    spec = str(g[f"t{n}_spec"])
    lam, max_iter, tol = (float(v) for v in g[f"t{n}_params"])
    kind, arg = spec.split(":")
    if kind == "small":
        q, corpus, emb = small_instance(golden("small"), int(arg))
    else:
        inst = synth.zipf_instance(kind, n_docs=int(arg) or None)
        q, corpus, emb = inst.query, inst.corpus(), inst.embeddings
    return q, corpus, emb, lam, int(max_iter), tol


def check_topk(got, ref_idx, ref_val, k: int, rtol: float = 1e-9, ref_full=None):
    """Top-k parity (north_star: identical top-k document indices).

    ``ref_idx`` / ``ref_val``: the reference's top-(k+1) (np.argsort stable)
    indices and values.  The stable top-k of ``got`` must equal the
    reference's, except at a rank p where the document placed there is a
    near-tie (within ``rtol``) of the reference's value at rank p — the only
    legitimate flip.  A document from outside the reference's
    top-(k+1) may only enter when the reference's rank-p and rank-(k+1)
    values are themselves within ``rtol`` (a boundary tie).  ``ref_full``
    (the whole reference vector) makes the check exact.  Returns the flips
    (rank, got doc, reference doc) for reporting; raises AssertionError
    otherwise."""
    got = np.asarray(got)
    top = np.argsort(got, kind="stable")[:k]
    ref_idx = np.asarray(ref_idx)[: k + 1]
    ref_val = np.asarray(ref_val)[: k + 1]
    if np.array_equal(top, ref_idx[:k]):
        return []
    pos = {int(d): p for p, d in enumerate(ref_idx)}
    flips = []
    for p in range(k):
        d = int(top[p])
        if d == int(ref_idx[p]):
            continue
        rv = ref_val[p]
        if ref_full is not None:
            v = float(ref_full[d])
        elif d in pos:
            v = float(ref_val[pos[d]])
        else:
            v = float(got[d])
            assert abs(ref_val[k] - rv) <= rtol * max(abs(rv), abs(ref_val[k])), (
                f"rank {p}: doc {d} from outside the reference top-{k + 1} without a boundary tie")
        assert abs(v - rv) <= rtol * max(abs(v), abs(rv)), (
            f"rank {p}: doc {d} (reference value {v!r}) where the reference has doc "
            f"{int(ref_idx[p])} ({rv!r})")
        flips.append((p, d, int(ref_idx[p])))
    return flips
