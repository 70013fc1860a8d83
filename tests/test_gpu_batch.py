"""The multi-query fp32 group launch (swmd_solve_group_f32 / reg_solve_mq):
per-query isolation of errors inside one launch, and the same bits as the
per-iteration single-query kernel."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import max_rel_err

import paper_2107_06433_b200 as swmd
from paper_2107_06433_b200 import batch, synth
from paper_2107_06433_b200.sparse import CsrMatrix

pytestmark = pytest.mark.gpu

F32_RTOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _instance(seed=7, V=2000, N=150, dim=32):
    rng = np.random.default_rng(seed)
    emb = synth.normal_embeddings(rng, V, dim, np.float32)
    cp, rows, vals = synth.zipf_corpus_csc(rng, V, N, 1, 90)
    return rng, emb, cp, rows, vals, CsrMatrix.from_csc(V, N, cp, rows, vals)


def test_group_launch_matches_oracle_per_query(oracle_lib):
    """Queries of one padded width share launches (groups of up to 4); every
    query's distances match the fp64 oracle within 1e-4."""
    rng, emb, cp, rows, vals, corpus = _instance()
    widths = [17, 18, 20, 24, 21, 23, 19, 22, 5, 6, 7]   # 8 in the 24-wide bucket, 3 in the 8-wide
    queries = [synth.zipf_query(rng, corpus.n_rows, v) for v in widths]
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15, precision="f32")
    out = swmd.sinkhorn_wmd_batch(queries, corpus, emb, cfg)
    # 24-wide bucket: 8 queries -> 2 group launches; 8-wide: 3 -> 1; plus Gram + reset
    assert batch.last_launches == 2 + 2 + 1
    E64 = emb.astype(np.float64)
    for q, r in zip(queries, out):
        assert isinstance(r, swmd.SolverResult), r
        want = oracle_lib.solve(q, cp, rows, vals, E64, lam=10.0, max_iter=15).wmd
        assert max_rel_err(r.wmd, want) <= F32_RTOL


def test_group_launch_equals_single_query_kernel():
    """tol = 0 never converges, so the tol path runs the same max_iter passes
    one launch at a time with the single-query kernel: same bits."""
    rng, emb, cp, rows, vals, corpus = _instance(seed=9)
    queries = [synth.zipf_query(rng, corpus.n_rows, v) for v in (30, 31, 32, 29)]
    grouped = swmd.sinkhorn_wmd_batch(queries, corpus, emb,
                                      swmd.SolverConfig(lam=10.0, max_iter=12, precision="f32"))
    single = swmd.sinkhorn_wmd_batch(queries, corpus, emb,
                                     swmd.SolverConfig(lam=10.0, max_iter=12, tol=0.0,
                                                       precision="f32"))
    for a, b in zip(grouped, single):
        assert np.array_equal(a.wmd, b.wmd)
        assert b.iterations_run == 12 and not b.converged


def test_group_isolates_a_degenerate_query(oracle_lib):
    """A zero denominator in one query of a group raises for that query only."""
    V, N = 64, 6
    emb = np.zeros((V, 4), dtype=np.float32)
    emb[:, 0] = np.linspace(0.0, 1.0, V, dtype=np.float32)
    emb[40:48, 1] = 1e3                       # words 40-47 far from everything
    trip = [(i, j, 1.0 + ((i + j) % 3)) for j in range(N) for i in range(j, 40, 7)]
    from paper_2107_06433_b200.sparse import csr_from_triplets

    corpus = csr_from_triplets(trip, V, N)
    good = np.zeros(V)
    good[[1, 2, 3]] = [0.2, 0.3, 0.5]
    bad = np.zeros(V)
    bad[[40, 41, 42]] = [0.2, 0.3, 0.5]       # exp(-lam * M) underflows on every row
    cfg = swmd.SolverConfig(lam=50.0, max_iter=5, precision="f32")
    out = swmd.sinkhorn_wmd_batch([good, bad, good], corpus, emb, cfg)
    assert isinstance(out[1], swmd.DegeneracyError), out[1]
    assert "zero denominator" in str(out[1])
    assert isinstance(out[0], swmd.SolverResult) and isinstance(out[2], swmd.SolverResult)
    assert np.array_equal(out[0].wmd, out[2].wmd)
