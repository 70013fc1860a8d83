"""Parity of the sm_100a path with the reference (golden fixtures) and the CPU oracle.

Tolerances: fp64 distances within 1e-9 relative (BASELINE.json north_star),
top-k identical; kernel-level pieces far tighter (stated per test).  Every
call goes through libswmd.so.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import check_topk, column_subset, golden, max_rel_err, small_instance, tol_case

import paper_2107_06433_b200 as swmd
from paper_2107_06433_b200 import synth
from paper_2107_06433_b200.sparse import CsrMatrix, csr_from_triplets

pytestmark = pytest.mark.gpu

RTOL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    swmd.kernels.warmup()


def _topk_full(got, want, k):
    """Strict top-k against a full reference vector (conftest.check_topk)."""
    order = np.argsort(want, kind="stable")
    return check_topk(got, order[: k + 1], want[order[: k + 1]], k, ref_full=want)


# -- kernel level, against the reference's own outputs (small.npz) -------------------------

def test_euclidean_rows_bitwise(small_golden):
    g = small_golden
    for k in range(50):
        q, corpus, emb = small_instance(g, k)
        sel = np.flatnonzero(q > 0)
        got = swmd.euclidean_rows(emb, sel)
        assert np.array_equal(got, g[f"i{k}_cost"]), k


def test_euclidean_rows_gram_mode(small_golden):
    g = small_golden
    for k in range(50):
        q, corpus, emb = small_instance(g, k)
        sel = np.flatnonzero(q > 0)
        got = swmd.euclidean_rows(emb, sel, mode=swmd.kernels.COST_MODE_GRAM)
        want = g[f"i{k}_cost"]
        assert np.all(got[sel, np.arange(sel.size)] == 0.0)
        nz = want > 0
        assert np.all(np.abs(got[nz] - want[nz]) <= 1e-12 * want[nz]), k


def test_precompute_and_invariants(small_golden):
    g = small_golden
    for k in range(50):
        q, corpus, emb = small_instance(g, k)
        sel = np.flatnonzero(q > 0)
        mats = swmd.precompute(g[f"i{k}_cost"], q[sel], 10.0)
        # CUDA exp is within 1 ulp of glibc exp
        assert max_rel_err(mats.kernel, g[f"i{k}_kernel"]) <= 4.5e-16
        assert max_rel_err(mats.kernel_over_r, g[f"i{k}_kor"]) <= 7e-16
        assert max_rel_err(mats.kernel_cost, g[f"i{k}_kcost"]) <= 7e-16
        assert np.array_equal(mats.kernel == 1.0, mats.cost == 0.0)
        assert np.all(mats.kernel > 0) and np.all(mats.kernel <= 1.0)


def test_fused_iteration_final_sddmm_spmm(small_golden, oracle_lib):
    g = small_golden
    for k in range(50):
        p = f"i{k}_"
        q, corpus, emb = small_instance(g, k)
        mats = swmd.SinkhornMatrices(g[p + "cost"], g[p + "kernel"], g[p + "kor"],
                                     g[p + "kcost"], 10.0)
        u = g[p + "u"]
        x = np.zeros_like(u)
        swmd.fused_iteration(corpus, mats, u, x)
        assert max_rel_err(x, g[p + "x1"]) <= 1e-13, k
        assert max_rel_err(swmd.fused_final(corpus, mats, u), g[p + "final"]) <= 1e-13, k
        w = swmd.sddmm(corpus, mats.kernel, u)
        assert max_rel_err(w, g[p + "sddmm"]) <= 1e-14, k
        xs = swmd.spmm(corpus, g[p + "sddmm"], mats.kernel_over_r)
        want = oracle_lib.spmm_serial(corpus.row_ptr, corpus.col_idx, g[p + "sddmm"],
                                      mats.kernel_over_r, corpus.n_cols)
        assert max_rel_err(xs, want) <= 1e-14, k


def test_fused_equals_composition(small_golden):
    g = small_golden
    q, corpus, emb = small_instance(g, 3)
    p = "i3_"
    mats = swmd.SinkhornMatrices(g[p + "cost"], g[p + "kernel"], g[p + "kor"], g[p + "kcost"], 10.0)
    u = g[p + "u"]
    fused = np.zeros_like(u)
    swmd.fused_iteration(corpus, mats, u, fused)
    composed = swmd.spmm(corpus, swmd.sddmm(corpus, mats.kernel, u), mats.kernel_over_r)
    assert max_rel_err(fused, composed) <= 1e-14


def test_work_count(small_golden):
    g = small_golden
    q, corpus, emb = small_instance(g, 5)
    p = "i5_"
    mats = swmd.SinkhornMatrices(g[p + "cost"], g[p + "kernel"], g[p + "kor"], g[p + "kcost"], 10.0)
    u = g[p + "u"]
    c1 = np.zeros(1, dtype=np.int64)
    swmd.fused_iteration(corpus, mats, u, np.zeros_like(u), counts=c1)
    assert c1[0] == 2 * corpus.nnz * mats.v_r
    c3 = np.zeros(3, dtype=np.int64)
    swmd.fused_iteration(corpus, mats, u, np.zeros_like(u), workers=3, counts=c3)
    assert c3.sum() == 2 * corpus.nnz * mats.v_r
    with pytest.raises(ValueError, match="deterministic"):
        swmd.fused_iteration(corpus, mats, u, np.zeros_like(u), workers=2, deterministic=True,
                             counts=c3[:2])


def test_zero_denominator_named():
    corpus = csr_from_triplets([(0, 0, 1.0)], 1, 1)
    mats = swmd.SinkhornMatrices(np.zeros((1, 1)), np.array([[0.0]]), np.array([[0.0]]),
                                 np.array([[0.0]]), 1.0)
    with pytest.raises(swmd.DegeneracyError, match=r"\(0, 0\)"):
        swmd.sddmm(corpus, mats.kernel, np.array([[1.0]]))
    with pytest.raises(swmd.DegeneracyError, match=r"zero denominator at nonzero \(0, 0\)"):
        swmd.fused_iteration(corpus, mats, np.array([[1.0]]), np.zeros((1, 1)))


# -- solver, against the reference's solver outputs -------------------------------------------------

def test_small_solver(small_golden):
    g = small_golden
    worst = 0.0
    for k in range(50):
        q, corpus, emb = small_instance(g, k)
        for lam in (1, 10):
            got = swmd.sinkhorn_wmd(q, corpus, emb, swmd.SolverConfig(lam=float(lam))).wmd
            worst = max(worst, max_rel_err(got, g[f"i{k}_wmd_lam{lam}"]))
    assert worst <= RTOL, worst


@pytest.mark.parametrize("mode", ["gram", "direct"])
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_config_parity(name, mode):
    g = golden(name)
    inst = synth.zipf_instance(name)
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15, cost_mode=mode)
    res = swmd.sinkhorn_wmd(inst.query, inst.corpus(), inst.embeddings, cfg)
    err = max_rel_err(res.wmd, g["wmd"])
    assert err <= RTOL, err
    for k in (10, 100):
        _topk_full(res.wmd, g["wmd"], k)
    assert res.iterations_run == 15 and not res.converged
    assert set(res.timings) == {"select", "distances", "precompute", "init", "iterations",
                                "final", "total"}


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_large_config_parity(name):
    g = golden(name)
    inst = synth.zipf_instance(name)
    res = swmd.sinkhorn_wmd(inst.query, inst.corpus(), inst.embeddings,
                            swmd.SolverConfig(lam=10.0, max_iter=15))
    stride = int(g["sample_stride"])
    assert max_rel_err(res.wmd[::stride], g["sample"]) <= RTOL
    top = g["top100"]
    assert max_rel_err(res.wmd[top], g["top100_wmd"]) <= RTOL
    for k in (10, 100):
        check_topk(res.wmd, g["top101"], g["top101_wmd"], k)
    assert abs(float(np.sum(res.wmd)) - float(g["wmd_sum"])) <= RTOL * abs(float(g["wmd_sum"]))


@pytest.mark.parametrize("v_r", [1, 2, 3, 4, 5, 7, 8, 12, 13, 16, 19, 20, 24, 27, 31, 32,
                                 33, 48, 64, 100, 300])
def test_query_length_buckets(v_r, oracle_lib):
    rng = np.random.default_rng(100 + v_r)
    V, N = 3000, 150
    emb = synth.normal_embeddings(rng, V, 64)
    cp, rows, vals = synth.zipf_corpus_csc(rng, V, N, 5, 40)
    q = synth.zipf_query(rng, V, v_r)
    corpus = CsrMatrix.from_csc(V, N, cp, rows, vals)
    got = swmd.sinkhorn_wmd(q, corpus, emb, swmd.SolverConfig(lam=10.0, max_iter=15)).wmd
    want = oracle_lib.solve(q, cp, rows, vals, emb, lam=10.0, max_iter=15).wmd
    assert max_rel_err(got, want) <= RTOL


@pytest.mark.parametrize("kmin,kmax", [(1, 3), (90, 200), (300, 420)])
def test_column_length_regimes(kmin, kmax, oracle_lib):
    """Short columns, columns past the register cache (>96 nonzeros) and the
    32-lanes-per-column regime."""
    rng = np.random.default_rng(kmin)
    V, N = 4000, 120
    emb = synth.normal_embeddings(rng, V, 32)
    cp, rows, vals = synth.zipf_corpus_csc(rng, V, N, kmin, kmax)
    corpus = CsrMatrix.from_csc(V, N, cp, rows, vals)
    for v_r in (6, 19):
        q = synth.zipf_query(rng, V, v_r)
        got = swmd.sinkhorn_wmd(q, corpus, emb, swmd.SolverConfig()).wmd
        want = oracle_lib.solve(q, cp, rows, vals, emb).wmd
        assert max_rel_err(got, want) <= RTOL


# -- acceptance criteria & solver contracts (test_acceptance.py, test_solver.py) -------------

def test_analytic_singletons():
    vecs = np.array([[0.0, 0.0], [1.0, 0.0]])
    query = np.array([1.0, 0.0])
    cfg = swmd.SolverConfig(lam=1.0, max_iter=15)
    same = csr_from_triplets([(0, 0, 1.0)], 2, 1)
    apart = csr_from_triplets([(1, 0, 1.0)], 2, 1)
    assert abs(swmd.sinkhorn_wmd(query, same, vecs, cfg).wmd[0]) <= 1e-12
    assert abs(swmd.sinkhorn_wmd(query, apart, vecs, cfg).wmd[0] - 1.0) <= 1e-12
    res = swmd.sinkhorn_wmd(query, same, vecs, swmd.SolverConfig(lam=1.0, max_iter=15, tol=1e-12))
    assert abs(res.wmd[0]) <= 1e-12 and res.converged and res.iterations_run == 1
    one = swmd.sinkhorn_wmd(query, apart, vecs, swmd.SolverConfig(lam=1.0, max_iter=1))
    assert abs(one.wmd[0] - 1.0) <= 1e-12


def test_zero_column_degenerates_cleanly(oracle_lib):
    corpus = csr_from_triplets([(0, 0, 1.0)], 2, 2)  # column 1 empty
    vecs = np.array([[0.0, 0.0], [1.0, 0.0]])
    with pytest.raises(swmd.DegeneracyError) as exc:
        swmd.sinkhorn_wmd(np.array([1.0, 0.0]), corpus, vecs, swmd.SolverConfig(lam=1.0, max_iter=3))
    cp, rows, _, vals = corpus.csc_index()
    with pytest.raises(oracle_lib.OracleDegeneracy) as want:
        oracle_lib.solve(np.array([1.0, 0.0]), cp, rows, vals, vecs, lam=1.0, max_iter=3)
    assert str(exc.value) == str(want.value)


def test_zero_denominator_in_solver_matches_oracle(oracle_lib):
    # lam large enough that exp(-lam*M) underflows to 0 for far words
    rng = np.random.default_rng(9)
    V, N = 50, 12
    emb = rng.normal(size=(V, 4)) * 30
    cp, rows, vals = synth.zipf_corpus_csc(rng, V, N, 2, 5)
    corpus = CsrMatrix.from_csc(V, N, cp, rows, vals)
    q = np.zeros(V)
    q[[3, 7]] = [0.5, 0.5]
    cfg = swmd.SolverConfig(lam=50.0, max_iter=4)
    with pytest.raises(swmd.DegeneracyError) as exc:
        swmd.sinkhorn_wmd(q, corpus, emb, cfg)
    with pytest.raises(oracle_lib.OracleDegeneracy) as want:
        oracle_lib.solve(q, cp, rows, vals, emb, lam=50.0, max_iter=4)
    assert str(exc.value) == str(want.value)


def test_first_zero_denominator_reported_when_one_lane_sees_several(oracle_lib):
    # two underflowing rows of one column sit in the same lane slot of
    # consecutive rounds (positions 1 and 17, and 1 and 33 with an 8-lane
    # round); the reference's CSR walk reports the smaller row
    V, N = 64, 3
    emb = np.zeros((V, 2))
    emb[:, 0] = np.linspace(0.0, 1.0, V)
    far = [1, 17, 33]
    emb[far, 1] = 1e3                       # exp(-lam * M) underflows to 0
    trip = [(i, 0, 1.0 + (i % 3)) for i in range(48)]
    trip += [(i, 1, 1.0) for i in (0, 2, 5)] + [(i, 2, 2.0) for i in (3, 4)]
    corpus = csr_from_triplets(trip, V, N)
    cp, rows, _, vals = corpus.csc_index()
    q = np.zeros(V)
    q[[0, 2]] = [0.5, 0.5]
    with pytest.raises(swmd.DegeneracyError) as exc:
        swmd.sinkhorn_wmd(q, corpus, emb, swmd.SolverConfig(lam=50.0, max_iter=3))
    with pytest.raises(oracle_lib.OracleDegeneracy) as want:
        oracle_lib.solve(q, cp, rows, vals, emb, lam=50.0, max_iter=3)
    assert str(exc.value) == str(want.value)
    assert "(1, 0)" in str(exc.value)


def test_tol_pinned_to_reference():
    """tol early exit against the reference's own runs (tests/golden/tol.npz,
    solver.py:170-183): same iterations_run and converged, wmd within 1e-9.
    The only tolerated difference is a stop one iteration apart where the
    reference's max|dx| at that iteration is itself within 1e-6 of tol (a
    convergence-boundary tie, reported)."""
    g = golden("tol")
    for n in range(int(g["n_cases"])):
        q, corpus, emb, lam, max_iter, tol = tol_case(g, n)
        res = swmd.sinkhorn_wmd(q, corpus, emb, swmd.SolverConfig(lam=lam, max_iter=max_iter,
                                                                  tol=tol))
        want_it = int(g[f"t{n}_iterations"])
        deltas = g[f"t{n}_deltas"]
        if res.iterations_run != want_it:
            i = min(res.iterations_run, want_it) - 1
            assert abs(res.iterations_run - want_it) == 1 and abs(deltas[i] - tol) <= 1e-6 * tol, (
                n, res.iterations_run, want_it, deltas[i])
            continue
        assert res.converged == bool(g[f"t{n}_converged"]), n
        assert max_rel_err(res.wmd, g[f"t{n}_wmd"]) <= RTOL, n


def test_tol_exit_is_self_consistent():
    inst = synth.zipf_instance("c1", n_docs=40)
    corpus = inst.corpus()
    tol = 1e-9
    res = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings,
                            swmd.SolverConfig(lam=1.0, max_iter=500, tol=tol))
    assert res.converged and res.iterations_run < 500
    more = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings,
                             swmd.SolverConfig(lam=1.0, max_iter=res.iterations_run + 1, tol=tol))
    assert more.iterations_run == res.iterations_run
    assert np.array_equal(more.wmd, res.wmd)
    # the per-iteration (tol) path and the persistent path compute the same bits
    fixed = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings,
                              swmd.SolverConfig(lam=1.0, max_iter=res.iterations_run))
    assert np.array_equal(fixed.wmd, res.wmd)


def test_column_independence_bitwise():
    inst = synth.zipf_instance("c1", n_docs=120)
    corpus = inst.corpus()
    cfg = swmd.SolverConfig()
    full = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg).wmd
    cols = np.random.default_rng(777).choice(120, size=17, replace=False)
    part = swmd.sinkhorn_wmd(inst.query, column_subset(corpus, cols), inst.embeddings, cfg).wmd
    assert np.array_equal(part, full[cols])


def test_shard_counts_bitwise():
    """Column blocks solved separately (the multi-GPU shards) reassemble to the
    single-launch result bit for bit, for 1/2/4/8 shards."""
    from paper_2107_06433_b200.distributed import DeviceShardSolver, shard_bounds

    inst = synth.zipf_instance("c2", n_docs=3000)
    corpus = inst.corpus()
    cfg = swmd.SolverConfig()
    full = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg).wmd
    sel, w = swmd.select_nonzero(inst.query)
    solver = DeviceShardSolver(corpus, inst.embeddings)
    for world in (1, 2, 4, 8):
        b = shard_bounds(corpus, world)
        out = np.concatenate([solver(sel, w, int(b[r]), int(b[r + 1]), cfg, None).wmd
                              for r in range(world)])
        assert np.array_equal(out, full), world


def test_batch_and_workspace():
    inst = synth.zipf_instance("c1", n_docs=50)
    corpus = inst.corpus()
    rng = np.random.default_rng(71)
    queries = [synth.zipf_query(rng, inst.n_vocab, v) for v in (3, 7, 19, 40)]
    cfg = swmd.SolverConfig()
    batch = swmd.sinkhorn_wmd_batch(queries + [np.zeros(inst.n_vocab)], corpus,
                                    inst.embeddings, cfg)
    for qv, r in zip(queries, batch):
        alone = swmd.sinkhorn_wmd(qv, corpus, inst.embeddings, cfg)
        assert np.array_equal(r.wmd, alone.wmd)
    assert isinstance(batch[-1], swmd.EmptyQueryError)
    ws = swmd.SinkhornWorkspace()
    first = swmd.sinkhorn_wmd(queries[2], corpus, inst.embeddings, cfg, workspace=ws)
    snap = first.wmd.copy()
    swmd.sinkhorn_wmd(queries[0], corpus, inst.embeddings, cfg, workspace=ws)
    again = swmd.sinkhorn_wmd(queries[2], corpus, inst.embeddings, cfg, workspace=ws)
    assert np.array_equal(first.wmd, snap) and np.array_equal(again.wmd, first.wmd)


def test_sparse_vector_query_and_embedding_cache():
    inst = synth.zipf_instance("c1", n_docs=30)
    corpus = inst.corpus()
    cfg = swmd.SolverConfig()
    idx = np.flatnonzero(inst.query)
    dense = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg).wmd
    sparse = swmd.sinkhorn_wmd(swmd.SparseVector(inst.n_vocab, idx, inst.query[idx]), corpus,
                               inst.embeddings, cfg).wmd
    assert np.array_equal(dense, sparse)
    # an in-place edit of a cached embedding table is picked up
    emb = inst.embeddings.copy()
    a = swmd.sinkhorn_wmd(inst.query, corpus, emb, cfg).wmd
    emb[:] = emb[::-1]
    b = swmd.sinkhorn_wmd(inst.query, corpus, emb, cfg).wmd
    c = swmd.sinkhorn_wmd(inst.query, corpus, emb.copy(), cfg).wmd
    assert not np.array_equal(a, b) and np.array_equal(b, c)
    # ... including a single-row edit of a row the corpus uses
    row = int(inst.rows[inst.col_ptr[3]])
    emb[row] *= 0.5
    d = swmd.sinkhorn_wmd(inst.query, corpus, emb, cfg).wmd
    e = swmd.sinkhorn_wmd(inst.query, corpus, emb.copy(), cfg).wmd
    assert not np.array_equal(b, d) and np.array_equal(d, e)
    # a read-only table is cached by identity (its buffer cannot change)
    ro = emb.copy()
    ro.flags.writeable = False
    assert np.array_equal(swmd.sinkhorn_wmd(inst.query, corpus, ro, cfg).wmd, e)


def test_torch_cuda_embeddings():
    import torch

    inst = synth.zipf_instance("c1", n_docs=30)
    corpus = inst.corpus()
    cfg = swmd.SolverConfig()
    a = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg).wmd
    b = swmd.sinkhorn_wmd(inst.query, corpus, torch.from_numpy(inst.embeddings).cuda(), cfg).wmd
    assert np.array_equal(a, b)


# -- fp32 multi-query variant (BASELINE config c4) ----------------------------------------------

F32_RTOL = 1e-4


def test_c4_fp32_batch_matches_fp64_reference():
    g = golden("c4")
    inst = synth.zipf_instance("c4")
    cfg = swmd.SolverConfig(lam=10.0, max_iter=20, precision="f32")
    res = swmd.sinkhorn_wmd_batch(inst.queries, inst.corpus(), inst.embeddings, cfg)
    stride = int(g["sample_stride"])
    worst = 0.0
    for k, r in enumerate(res):
        assert isinstance(r, swmd.SolverResult), r
        worst = max(worst, max_rel_err(r.wmd[::stride], g["sample"][k]))
        assert abs(float(np.sum(r.wmd)) - float(g["wmd_sum"][k])) <= F32_RTOL * float(g["wmd_sum"][k])
        top = g["top10"][k]
        assert max_rel_err(r.wmd[top], g["top10_wmd"][k]) <= F32_RTOL
        # fp32 may reorder only reference near-ties within its 1e-4 band
        check_topk(r.wmd, g["top11"][k], g["top11_wmd"][k], 10, rtol=2 * F32_RTOL)
    assert worst <= F32_RTOL, worst


def test_fp32_batch_contract(oracle_lib):
    rng = np.random.default_rng(44)
    V, N = 3000, 120
    emb = synth.normal_embeddings(rng, V, 64, np.float32)
    cp, rows, vals = synth.zipf_corpus_csc(rng, V, N, 5, 40)
    corpus = CsrMatrix.from_csc(V, N, cp, rows, vals)
    queries = [synth.zipf_query(rng, V, v) for v in (3, 8, 19, 64, 100)]
    queries.insert(2, np.zeros(V))                  # fails alone, batch continues
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15, precision="f32")
    out = swmd.sinkhorn_wmd_batch(queries, corpus, emb, cfg)
    assert isinstance(out[2], swmd.EmptyQueryError)
    for q, r in zip(queries, out):
        if isinstance(r, Exception):
            continue
        want = oracle_lib.solve(q, cp, rows, vals, emb.astype(np.float64), lam=10.0,
                                max_iter=15).wmd
        assert max_rel_err(r.wmd, want) <= F32_RTOL
    # single-query entry point and the tol path in fp32
    one = swmd.sinkhorn_wmd(queries[3], corpus, emb, cfg)
    assert np.array_equal(one.wmd, out[3].wmd)
    tol = swmd.sinkhorn_wmd(queries[3], corpus, emb,
                            swmd.SolverConfig(lam=1.0, max_iter=300, tol=1e-6, precision="f32"))
    assert tol.converged and tol.iterations_run < 300


# -- device top-k ---------------------------------------------------------------------------------

@pytest.mark.parametrize("name,k", [("c1", 10), ("c2", 100), ("c2", 1024)])
def test_topk_matches_stable_argsort(name, k):
    inst = synth.zipf_instance(name)
    corpus = inst.corpus()
    cfg = swmd.SolverConfig()
    full = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg).wmd
    top = swmd.sinkhorn_wmd_topk(inst.query, corpus, inst.embeddings, cfg, k)
    want = np.argsort(full, kind="stable")[:k]
    assert np.array_equal(top.indices, want)
    assert np.array_equal(top.wmd, full[want])
    g = golden(name)
    _topk_full(full, g["wmd"], min(k, 100))


def test_topk_ties_go_to_lower_index():
    # identical documents give exactly equal distances (test_ingest.py:119-122)
    inst = synth.zipf_instance("c1", n_docs=50)
    cp, rows, vals = inst.col_ptr, inst.rows, inst.vals
    a, b = cp[7], cp[8]
    reps = 30
    cp2 = np.concatenate([cp, cp[-1] + (b - a) * np.arange(1, reps + 1)])
    rows2 = np.concatenate([rows] + [rows[a:b]] * reps)
    vals2 = np.concatenate([vals] + [vals[a:b]] * reps)
    corpus = CsrMatrix.from_csc(inst.n_vocab, 50 + reps, cp2, rows2, vals2)
    cfg = swmd.SolverConfig()
    full = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg).wmd
    assert np.all(full[50:] == full[7])
    top = swmd.sinkhorn_wmd_topk(inst.query, corpus, inst.embeddings, cfg, 40)
    assert np.array_equal(top.indices, np.argsort(full, kind="stable")[:40])


# -- device CSR -> CSC transpose (replaces the host argsort of sparse.py:98-120) --------------

def _device_csc(corpus):
    import torch
    from paper_2107_06433_b200.device import DeviceCorpus

    dc = DeviceCorpus.from_csr(corpus.n_rows, corpus.n_cols, corpus.row_ptr, corpus.col_idx,
                               corpus.values, torch.device("cuda", 0))
    return (dc.col_ptr.cpu().numpy(), dc.rows.cpu().numpy(), dc.pos.cpu().numpy(),
            dc.vals.cpu().numpy(), dc)


def _host_csc(corpus):
    rp, ci, v = corpus.row_ptr, corpus.col_idx, corpus.values
    return CsrMatrix(corpus.n_rows, corpus.n_cols, rp, ci, v).csc_index()


def _assert_same_csc(corpus):
    cp, rows, pos, vals, dc = _device_csc(corpus)
    hcp, hrows, hpos, hvals = _host_csc(corpus)
    assert np.array_equal(cp, hcp)
    assert np.array_equal(rows, hrows.astype(np.int32))
    assert np.array_equal(pos, hpos)
    assert np.array_equal(vals, hvals)
    present = np.flatnonzero(np.diff(corpus.row_ptr) > 0)
    assert dc.n_present == present.size
    return dc


def test_device_csc_matches_host_small(small_golden):
    for k in range(50):
        _, corpus, _ = small_instance(small_golden, k)
        _assert_same_csc(corpus)


def test_device_csc_matches_host_c2():
    inst = synth.zipf_instance("c2")
    rp, ci, v = synth.csc_to_csr(inst.n_vocab, inst.n_docs, inst.col_ptr, inst.rows, inst.vals)
    corpus = CsrMatrix(inst.n_vocab, inst.n_docs, rp, ci, v)
    _assert_same_csc(corpus)


def test_device_csc_long_and_empty_columns():
    rng = np.random.default_rng(11)
    V, N = 6000, 40
    trip = []
    lens = [0, 1, 33, 257, 1024, 1025, 3000, 0, 5] + list(rng.integers(0, 70, N - 9))
    for j, L in enumerate(lens):
        for i in np.sort(rng.choice(V, size=int(L), replace=False)):
            trip.append((int(i), j, float(rng.integers(1, 5))))
    corpus = csr_from_triplets(trip, V, N)
    _assert_same_csc(corpus)
    empty = csr_from_triplets([], 7, 3)
    cp, rows, pos, vals, dc = _device_csc(empty)
    assert np.array_equal(cp, np.zeros(4, dtype=np.int64)) and rows.size == 0
    assert dc.n_present == 0


def test_csr_corpus_solves_through_device_transpose():
    g = golden("c2")
    inst = synth.zipf_instance("c2")
    rp, ci, v = synth.csc_to_csr(inst.n_vocab, inst.n_docs, inst.col_ptr, inst.rows, inst.vals)
    corpus = CsrMatrix(inst.n_vocab, inst.n_docs, rp, ci, v)
    res = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings,
                            swmd.SolverConfig(lam=10.0, max_iter=15))
    assert corpus._csc_cache is None          # no host transpose happened
    assert max_rel_err(res.wmd, g["wmd"]) <= RTOL


def test_native_plan_graphs_per_query_shape(oracle_lib):
    """The native plan caches one CUDA graph per (v_r, lam, max_iter, mode):
    interleaving query lengths and lambdas must reuse the right one."""
    rng = np.random.default_rng(77)
    V, N = 4000, 300
    emb = synth.normal_embeddings(rng, V, 48)
    cp, rows, vals = synth.zipf_corpus_csc(rng, V, N, 5, 60)
    corpus = CsrMatrix.from_csc(V, N, cp, rows, vals)
    ws = swmd.SinkhornWorkspace()
    queries = [synth.zipf_query(rng, V, v) for v in (5, 19, 32, 19, 5)]
    for rep in range(2):
        for k, q in enumerate(queries):
            lam = (10.0, 3.0)[(k + rep) % 2]
            it = (15, 7)[rep]
            got = swmd.sinkhorn_wmd(q, corpus, emb, swmd.SolverConfig(lam=lam, max_iter=it),
                                    workspace=ws)
            want = oracle_lib.solve(q, cp, rows, vals, emb, lam=lam, max_iter=it).wmd
            assert max_rel_err(got.wmd, want) <= RTOL, (rep, k)
            assert set(got.timings) >= {"select", "distances", "iterations", "total"}
            assert got.timings["distances"] > 0 and got.timings["iterations"] > 0


def test_query_plan_reset_rides_on_the_cost_build(oracle_lib):
    """The device-timed path (QueryPlan: cost build whose first thread resets
    the solve's error record and work counter, then the solve launched with no
    reset of its own) gives the public API's bits, whatever the counter and
    the error record held before."""
    import torch

    from paper_2107_06433_b200 import _lib
    from paper_2107_06433_b200.device import DeviceCorpus, DeviceEmbeddings, device
    from paper_2107_06433_b200.solver import QueryPlan

    inst = synth.zipf_instance("c1", n_docs=300)
    corpus = inst.corpus()
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15)
    sel, w = swmd.select_nonzero(inst.query)
    dev = device()
    dc = DeviceCorpus.of(corpus, dev)
    de = DeviceEmbeddings.of(inst.embeddings, dev)
    plan = QueryPlan(sel, w, dc, de, cfg, swmd.SinkhornWorkspace())
    for _ in range(2):
        plan.counter.fill_(123456)            # a stale counter would skip columns
        plan.err.fill_(7)                     # a stale record would read as an event
        plan.enqueue_distances()
        plan.enqueue_solve()
        torch.cuda.synchronize()
        got = plan.wmd.cpu().numpy()
        assert int(plan.err[0]) == _lib.NO_EVENT and int(plan.err[1]) == _lib.NO_EVENT
        want = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg).wmd
        assert np.array_equal(got, want)
    ref = oracle_lib.solve(inst.query, inst.col_ptr, inst.rows, inst.vals, inst.embeddings,
                           lam=10.0, max_iter=15).wmd
    assert max_rel_err(got, ref) <= RTOL


def test_randomised_instances_match_oracle(oracle_lib):
    """Seeded sweep over the shapes the persistent kernels specialise on:
    v_r from 1 to 40 (register-round solve and CTA solve), column lengths
    from 1 to ~130 (register rounds, slab, past the slab), lambda from 0.5 to
    30, 1 to 20 iterations; every case within 1e-9 of the oracle and the same
    top-10."""
    rng = np.random.default_rng(20261020)
    for case in range(24):
        V = int(rng.integers(200, 3000))
        N = int(rng.integers(1, 150))
        dim = int(rng.choice([2, 8, 30, 64]))
        kmin = int(rng.integers(1, 40))
        kmax = min(V, kmin + int(rng.integers(0, 90)))
        v_r = int(rng.integers(1, 41))
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
        _topk_full(got, want, min(10, N))
