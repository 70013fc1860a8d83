"""Public-API edge cases against the reference's own outputs
(tests/golden/edge.npz, made by tests/golden/make_edge.py from the
reference): empty corpus, max_iter = 1, float32 embeddings, list and
strided queries, tol = 0, a one-word document."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, max_rel_err

import paper_2107_06433_b200 as swmd
from paper_2107_06433_b200.sparse import CsrMatrix

pytestmark = pytest.mark.gpu
RTOL = 1e-9


@pytest.fixture(scope="module")
def edge():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g = golden("edge")
    V = g["emb"].shape[0]
    N = g["wmd_iter1"].shape[0]
    corpus = CsrMatrix(V, N, g["row_ptr"], g["col_idx"], g["values"])
    return g, corpus


def test_max_iter_one(edge):
    g, corpus = edge
    r = swmd.sinkhorn_wmd(g["q"], corpus, g["emb"], swmd.SolverConfig(lam=10.0, max_iter=1))
    assert max_rel_err(r.wmd, g["wmd_iter1"]) <= RTOL and r.iterations_run == 1


def test_float32_embeddings_are_coerced(edge):
    g, corpus = edge
    r = swmd.sinkhorn_wmd(g["q"], corpus, g["emb"].astype(np.float32), swmd.SolverConfig(lam=10.0))
    assert max_rel_err(r.wmd, g["wmd_f32emb"]) <= RTOL


def test_list_and_strided_queries(edge):
    g, corpus = edge
    r = swmd.sinkhorn_wmd(list(g["q"]), corpus, g["emb"], swmd.SolverConfig(lam=10.0))
    assert max_rel_err(r.wmd, g["wmd_list"]) <= RTOL
    wide = np.zeros(2 * g["q"].size)
    wide[::2] = g["q"]
    r = swmd.sinkhorn_wmd(wide[::2], corpus, g["emb"], swmd.SolverConfig(lam=10.0))
    assert max_rel_err(r.wmd, g["wmd_strided"]) <= RTOL


def test_tol_zero_never_converges(edge):
    g, corpus = edge
    r = swmd.sinkhorn_wmd(g["q"], corpus, g["emb"], swmd.SolverConfig(lam=10.0, max_iter=9, tol=0.0))
    assert r.iterations_run == int(g["tol0_iters"]) and r.converged == bool(g["tol0_conv"])
    assert max_rel_err(r.wmd, g["wmd_tol0"]) <= RTOL


def test_empty_corpus(edge):
    g, _ = edge
    V = g["emb"].shape[0]
    empty = CsrMatrix(V, 0, np.zeros(V + 1, dtype=np.int64), np.zeros(0, dtype=np.int64),
                      np.zeros(0))
    r = swmd.sinkhorn_wmd(g["q"], empty, g["emb"], swmd.SolverConfig(max_iter=3))
    assert r.wmd.shape == tuple(g["empty_shape"])
    assert r.iterations_run == int(g["empty_iters"]) and r.converged == bool(g["empty_conv"])
    unf = swmd.unfused_sparse_wmd(g["q"], empty, g["emb"], swmd.SolverConfig(max_iter=3))
    assert unf.shape == (0,)


def test_sparse_vector_query_native_path_same_bits():
    """A SparseVector query (the reference's ingest output) goes through the
    native runtime without densifying; the distances are the dense query's."""
    from paper_2107_06433_b200 import synth
    from paper_2107_06433_b200.sparse import SparseVector

    inst = synth.zipf_instance("c2")
    corpus = inst.corpus()
    sel = np.flatnonzero(inst.query > 0)
    sv = SparseVector(inst.query.size, sel, inst.query[sel])
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15)
    dense = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg)
    sparse = swmd.sinkhorn_wmd(sv, corpus, inst.embeddings, cfg)
    assert np.array_equal(dense.wmd, sparse.wmd)
    assert max_rel_err(sparse.wmd, golden("c2")["wmd"]) <= RTOL
    # an empty histogram still raises the reference's error
    with pytest.raises(swmd.EmptyQueryError):
        swmd.sinkhorn_wmd(SparseVector(inst.query.size, [], []), corpus, inst.embeddings, cfg)
