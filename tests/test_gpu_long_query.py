"""The long-query solve (32 < v_r <= 256, `cta2_solve`: a CTA per column, two
K rows reduced per warp step) against the CPU oracle: every row-width
instantiation (1-4 sixteen-byte chunks per lane, rows that fill their last
chunk and rows that do not), columns shorter than one CTA step and longer
than the staged index arrays, the reference's degeneracy messages, the tol
path and the shard split.  Reference: _jit.py:164-183, 291-312 at large v_r.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import max_rel_err

import paper_2107_06433_b200 as swmd
from paper_2107_06433_b200 import synth
from paper_2107_06433_b200.sparse import CsrMatrix

pytestmark = pytest.mark.gpu

RTOL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    swmd.kernels.warmup()


def _case(seed, V, N, kmin, kmax, v_r, dim=48):
    rng = np.random.default_rng(seed)
    emb = synth.normal_embeddings(rng, V, dim)
    cp, rows, vals = synth.zipf_corpus_csc(rng, V, N, kmin, kmax)
    q = synth.zipf_query(rng, V, v_r)
    return q, CsrMatrix.from_csc(V, N, cp, rows, vals), emb, (cp, rows, vals)


# ldk = v_r rounded up to 4; chunks per lane = ceil(ldk / 64); "whole" rows: ldk == 64 * chunks
@pytest.mark.parametrize("v_r", [33, 40, 61, 64, 65, 96, 127, 128, 129, 150, 190, 192, 193,
                                 200, 250, 253, 256])
def test_row_width_instantiations(v_r, oracle_lib):
    q, corpus, emb, (cp, rows, vals) = _case(500 + v_r, 3000, 140, 1, 70, v_r)
    got = swmd.sinkhorn_wmd(q, corpus, emb, swmd.SolverConfig(lam=10.0, max_iter=15)).wmd
    want = oracle_lib.solve(q, cp, rows, vals, emb, lam=10.0, max_iter=15).wmd
    assert max_rel_err(got, want) <= RTOL


@pytest.mark.parametrize("v_r", [70, 256])
def test_columns_longer_than_the_staged_index(v_r, oracle_lib):
    """Columns of 450-700 nonzeros: some fit the 512-entry staged (row id,
    value) arrays, some are read from global memory."""
    q, corpus, emb, (cp, rows, vals) = _case(77 + v_r, 4000, 20, 450, 700, v_r, dim=32)
    assert int(np.diff(cp).max()) > 512 and int(np.diff(cp).min()) < 512
    got = swmd.sinkhorn_wmd(q, corpus, emb, swmd.SolverConfig(lam=5.0, max_iter=6)).wmd
    want = oracle_lib.solve(q, cp, rows, vals, emb, lam=5.0, max_iter=6).wmd
    assert max_rel_err(got, want) <= RTOL


@pytest.mark.parametrize("v_r", [40, 130])
def test_zero_denominator_message_matches_oracle(v_r, oracle_lib):
    """exp(-lam*M) underflows for far words: the first (i, j) the reference's
    CSR walk reports, from whichever half-warp saw it."""
    rng = np.random.default_rng(9 + v_r)
    V, N = 400, 30
    emb = rng.normal(size=(V, 4)) * 30
    cp, rows, vals = synth.zipf_corpus_csc(rng, V, N, 2, 40)
    corpus = CsrMatrix.from_csc(V, N, cp, rows, vals)
    q = np.zeros(V)
    q[rng.choice(V, size=v_r, replace=False)] = 1.0 / v_r
    cfg = swmd.SolverConfig(lam=50.0, max_iter=4)
    with pytest.raises(swmd.DegeneracyError) as exc:
        swmd.sinkhorn_wmd(q, corpus, emb, cfg)
    with pytest.raises(oracle_lib.OracleDegeneracy) as want:
        oracle_lib.solve(q, cp, rows, vals, emb, lam=50.0, max_iter=4)
    assert str(exc.value) == str(want.value)


def test_tol_path_matches_oracle(oracle_lib):
    """One launch per iteration with x carried through HBM (x_in / x_out)."""
    q, corpus, emb, (cp, rows, vals) = _case(4242, 2500, 90, 3, 60, 80)
    cfg = swmd.SolverConfig(lam=1.0, max_iter=60, tol=1e-9)
    res = swmd.sinkhorn_wmd(q, corpus, emb, cfg)
    want = oracle_lib.solve(q, cp, rows, vals, emb, lam=1.0, max_iter=60, tol=1e-9)
    assert res.iterations_run == want.iterations_run and res.converged == want.converged
    assert max_rel_err(res.wmd, want.wmd) <= RTOL


def test_max_iter_one_and_empty_column_free_corpus(oracle_lib):
    q, corpus, emb, (cp, rows, vals) = _case(31337, 2000, 64, 1, 9, 200)
    got = swmd.sinkhorn_wmd(q, corpus, emb, swmd.SolverConfig(lam=10.0, max_iter=1)).wmd
    want = oracle_lib.solve(q, cp, rows, vals, emb, lam=10.0, max_iter=1).wmd
    assert max_rel_err(got, want) <= RTOL


def test_column_blocks_are_bitwise_identical():
    """Each column is solved by one CTA whatever the block it arrives in, so
    the shard split cannot change a bit (distributed.py, sparse.py:261-276)."""
    from paper_2107_06433_b200.distributed import DeviceShardSolver, shard_bounds

    q, corpus, emb, _ = _case(2024, 3000, 200, 5, 90, 256)
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15)
    one = swmd.sinkhorn_wmd(q, corpus, emb, cfg).wmd
    sel, w = swmd.select_nonzero(q)
    solver = DeviceShardSolver(corpus, emb)
    for world in (2, 3):
        b = shard_bounds(corpus, world)
        got = np.concatenate([solver(sel, w, int(b[r]), int(b[r + 1]), cfg, None).wmd
                              for r in range(world)])
        assert np.array_equal(got, one), world


def test_hot_row_entry_point_is_bitwise_the_plain_solve():
    """swmd_solve_hot_f64 with the corpus's hot-row index (the K rows of the
    most frequent vocabulary rows read from a shared-memory slab when
    SWMD_CTA_HOT is set, else ignored) gives the bits of swmd_solve_f64."""
    import torch

    from paper_2107_06433_b200 import _lib
    from paper_2107_06433_b200.device import DeviceCorpus, DeviceEmbeddings, device, stream_ptr
    from paper_2107_06433_b200.solver import QueryPlan, SinkhornWorkspace

    q, corpus, emb, _ = _case(99, 3000, 160, 5, 90, 200)
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15)
    dev = device()
    dc, de = DeviceCorpus.of(corpus, dev), DeviceEmbeddings.of(emb, dev)
    sel, w = swmd.select_nonzero(q)
    plan = QueryPlan(sel, w, dc, de, cfg, SinkhornWorkspace())
    plan.enqueue_distances()
    plan.enqueue_solve()
    torch.cuda.synchronize()
    want = plan.wmd.clone()
    slot, ids = dc.hot_index()
    assert ids is not None and int(slot[ids.long()].min()) == 0
    counts = np.bincount(np.asarray(corpus.csc_index()[1]), minlength=3000)
    assert counts[int(ids[0])] == counts.max()
    plan.wmd.zero_()
    _lib.call("swmd_err_reset", plan.err.data_ptr(), plan.stream)
    _lib.call("swmd_solve_hot_f64", dc.col_ptr.data_ptr(), dc.rows.data_ptr(), dc.vals.data_ptr(),
              dc.n_cols, dc.order.data_ptr(), plan.K.data_ptr(), plan.KM.data_ptr(),
              plan.r_dev.data_ptr(), plan.v_r, plan.ldk, 0, cfg.max_iter, None, None,
              plan.wmd.data_ptr(), dc.col_offset, dc.n_key, plan.group, dc.max_len,
              plan.err.data_ptr(), plan.counter.data_ptr(), stream_ptr(dev), 0,
              slot.data_ptr(), ids.data_ptr(), int(ids.numel()))
    torch.cuda.synchronize()
    assert torch.equal(plan.wmd, want)


def test_suite_with_the_hot_row_slab_enabled():
    """The slab variant is opt-in (SWMD_CTA_HOT=<rows>, read once per
    process): rerun this file's solver cases in a child process with it on."""
    import os
    import subprocess
    import sys

    if os.environ.get("SWMD_CTA_HOT_CHILD"):
        pytest.skip("already the child run")
    env = dict(os.environ, SWMD_CTA_HOT="48", SWMD_CTA_HOT_CHILD="1")
    res = subprocess.run([sys.executable, "-m", "pytest", __file__, "-x", "-q", "-p", "no:cacheprovider",
                          "-k", "row_width or staged_index or zero_denominator or tol_path or hot_row"],
                         env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]


def test_empty_column_raises_the_reference_error(oracle_lib):
    """A document with no words: x collapses to 0 after the first pass and the
    reference's update_u check names the entry (solver.py:95-103)."""
    rng = np.random.default_rng(5)
    V, N, v_r = 600, 9, 70
    emb = synth.normal_embeddings(rng, V, 16)
    cp, rows, vals = synth.zipf_corpus_csc(rng, V, N, 3, 30)
    # drop every entry of column 4
    keep = np.ones(rows.size, dtype=bool)
    keep[cp[4]:cp[5]] = False
    lens = np.diff(cp)
    lens[4] = 0
    cp2 = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    rows2, vals2 = rows[keep], vals[keep]
    corpus = CsrMatrix.from_csc(V, N, cp2, rows2, vals2)
    q = synth.zipf_query(rng, V, v_r)
    cfg = swmd.SolverConfig(lam=2.0, max_iter=5)
    with pytest.raises(swmd.DegeneracyError) as exc:
        swmd.sinkhorn_wmd(q, corpus, emb, cfg)
    with pytest.raises(oracle_lib.OracleDegeneracy) as want:
        oracle_lib.solve(q, cp2, rows2, vals2, emb, lam=2.0, max_iter=5)
    assert str(exc.value) == str(want.value)


def test_randomised_long_queries_match_oracle(oracle_lib):
    """Seeded sweep over what cta2_solve specialises on: v_r from 33 to 256
    (1-4 chunks per lane, whole and clamped rows), column lengths from 1 to
    ~600 (shorter than one CTA step, staged, past the staged arrays), lambda
    from 0.5 to 30, 1 to 20 iterations; every case within 1e-9 of the oracle
    with the same top-10, or the oracle's degeneracy message."""
    from conftest import check_topk

    rng = np.random.default_rng(20261021)
    for case in range(24):
        V = int(rng.integers(300, 3000))
        N = int(rng.integers(1, 120))
        dim = int(rng.choice([2, 8, 30, 64]))
        kmin = int(rng.integers(1, 60))
        kmax = min(V, kmin + int(rng.choice([0, 10, 90, 560])))
        v_r = int(rng.integers(33, 257))
        lam = float(rng.choice([0.5, 3.0, 10.0, 30.0]))
        it = int(rng.integers(1, 21))
        emb = synth.normal_embeddings(rng, V, dim)
        cp, rows, vals = synth.zipf_corpus_csc(rng, V, N, kmin, kmax)
        corpus = CsrMatrix.from_csc(V, N, cp, rows, vals)
        q = synth.zipf_query(rng, V, min(v_r, V))
        cfg = swmd.SolverConfig(lam=lam, max_iter=it)
        try:
            want = oracle_lib.solve(q, cp, rows, vals, emb, lam=lam, max_iter=it).wmd
        except oracle_lib.OracleDegeneracy as exc:
            with pytest.raises(swmd.DegeneracyError) as got_exc:
                swmd.sinkhorn_wmd(q, corpus, emb, cfg)
            assert str(got_exc.value) == str(exc), case
            continue
        got = swmd.sinkhorn_wmd(q, corpus, emb, cfg).wmd
        assert max_rel_err(got, want) <= RTOL, (case, V, N, dim, kmin, kmax, v_r, lam, it)
        k = min(10, N)
        order = np.argsort(want, kind="stable")
        check_topk(got, order[: k + 1], want[order[: k + 1]], k, ref_full=want)
