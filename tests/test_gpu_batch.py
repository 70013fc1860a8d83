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


@pytest.mark.parametrize("V,dim,widths,trim", [(300, 20, [5, 9], 0), (1000, 300, [64, 33, 8, 31], 0),
                                               (129, 5, [3], 0), (2500, 17, [40] * 7, 0),
                                               (257, 16, [12, 13], 0), (400, 24, [9], 4),
                                               (700, 40, [17, 20], 4)])
def test_gram_kernels_agree(V, dim, widths, trim):
    """The tensor-core Gram (tcgen05 kind::tf32 with the 3xTF32 split, TMEM
    accumulator) against the FFMA Gram on the same batch: K and K*M over
    row / column / depth counts that are not multiples of the 128 x 256 x 16
    tile (and row strides that rule out its 32-byte stores), with and without a
    present-row list.  3xTF32 keeps fp32-level dot
    products: |dK| <= 2e-5 K-scale (lam * dM), far inside the batch's 1e-4."""
    import os

    import torch

    from paper_2107_06433_b200 import _lib
    from paper_2107_06433_b200.device import device, stream_ptr

    rng = np.random.default_rng(V + dim)
    dev = device()
    s = stream_ptr(dev)
    emb = synth.normal_embeddings(rng, V, dim, np.float32)
    ld = (dim + 3) // 4 * 4
    E = torch.zeros((V, ld), dtype=torch.float32, device=dev)
    E[:, :dim] = torch.from_numpy(emb).to(dev)
    norms = torch.empty(V, dtype=torch.float32, device=dev)
    _lib.call("swmd_row_norms_f32", E.data_ptr(), V, dim, ld, norms.data_ptr(), s)
    words, col_word, off = [], [], 0
    for w in widths:
        sel = np.sort(rng.choice(V, size=w, replace=False))
        blk = (w + 7) // 8 * 8
        col_word += list(range(off, off + w)) + [-1] * (blk - w)
        words += list(sel)
        off += w
    if trim:                       # a row stride that is a multiple of 4 but not of 8
        assert all(c < 0 for c in col_word[-trim:])
        col_word = col_word[:-trim]
    LD = len(col_word)
    assert LD % 4 == 0 and (trim == 0 or LD % 8 == 4)
    words_d = torch.tensor(words, dtype=torch.int64, device=dev)
    col_d = torch.tensor(col_word, dtype=torch.int32, device=dev)
    for present in (None, np.sort(rng.choice(V, size=max(1, (2 * V) // 3), replace=False))):
        rl = torch.tensor(present, dtype=torch.int32, device=dev) if present is not None else None
        outs = {}
        for mode in ("ffma", "tc5"):
            os.environ["SWMD_GRAM32"] = mode
            K = torch.full((V, LD), -1.0, dtype=torch.float32, device=dev)
            KM = torch.full((V, LD), -1.0, dtype=torch.float32, device=dev)
            try:
                _lib.call("swmd_cost_build_batch_f32", E.data_ptr(), V, dim, ld, words_d.data_ptr(),
                          col_d.data_ptr(), LD, 10.0, norms.data_ptr(),
                          rl.data_ptr() if rl is not None else None,
                          int(rl.numel()) if rl is not None else 0, K.data_ptr(), KM.data_ptr(), s)
                torch.cuda.synchronize()
            finally:
                os.environ.pop("SWMD_GRAM32", None)
            outs[mode] = (K.cpu().numpy(), KM.cpu().numpy())
        rows = np.arange(V) if present is None else present
        for a, b in zip(outs["ffma"], outs["tc5"]):
            assert np.array_equal(a == -1.0, b == -1.0)          # the same entries written
            assert np.max(np.abs(a[rows] - b[rows])) <= 2e-5
        # exact zeros: a word against itself, and padding columns
        Kt = outs["tc5"][0]
        pad = np.array(col_word) < 0
        assert np.all(Kt[rows][:, pad] == 0.0)
