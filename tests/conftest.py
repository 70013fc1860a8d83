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
