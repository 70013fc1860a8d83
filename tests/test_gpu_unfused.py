"""The device unfused comparator (baseline.unfused_sparse_wmd, reference
baseline.py:67-131) against the reference's goldens and the CPU oracle.

The reference documents its unfused path as bitwise equal to the fused
solver in serial deterministic mode, so the fused solver's goldens pin it;
tolerance 1e-9 relative (fp64, BASELINE.json north_star).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, max_rel_err, small_instance, tol_case

import paper_2107_06433_b200 as swmd
from paper_2107_06433_b200 import synth
from paper_2107_06433_b200.baseline import unfused_sparse_wmd
from paper_2107_06433_b200.sparse import CsrMatrix, csr_from_triplets

pytestmark = pytest.mark.gpu

RTOL = 1e-9
PHASES = {"select", "distances", "precompute", "init", "iterations", "final", "total"}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    swmd.kernels.warmup()


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_unfused_config_parity(name):
    g = golden(name)
    inst = synth.zipf_instance(name)
    timings: dict[str, float] = {}
    got = unfused_sparse_wmd(inst.query, inst.corpus(), inst.embeddings,
                             swmd.SolverConfig(lam=10.0, max_iter=15), timings=timings)
    assert max_rel_err(got, g["wmd"]) <= RTOL
    assert set(timings) == PHASES
    assert np.array_equal(np.argsort(got, kind="stable")[:10], np.argsort(g["wmd"], kind="stable")[:10])


def test_unfused_small_instances(small_golden):
    g = small_golden
    worst = 0.0
    for k in range(50):
        q, corpus, emb = small_instance(g, k)
        for lam in (1, 10):
            got = unfused_sparse_wmd(q, corpus, emb, swmd.SolverConfig(lam=float(lam)))
            worst = max(worst, max_rel_err(got, g[f"i{k}_wmd_lam{lam}"]))
    assert worst <= RTOL, worst


def test_unfused_matches_fused():
    inst = synth.zipf_instance("c1")
    corpus = inst.corpus()
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15)
    fused = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg).wmd
    unf = unfused_sparse_wmd(inst.query, corpus, inst.embeddings, cfg)
    assert max_rel_err(unf, fused) <= 1e-13


def test_unfused_tol_against_reference():
    """The reference's unfused loop stops on the same max|dx| < tol test as the
    solver (baseline.py:119-121 vs solver.py:179-183): its distances are the
    tol goldens' (cases at a convergence-boundary tie are skipped)."""
    g = golden("tol")
    checked = 0
    for n in range(int(g["n_cases"])):
        q, corpus, emb, lam, max_iter, tol = tol_case(g, n)
        deltas = g[f"t{n}_deltas"]
        if np.any(np.abs(deltas - tol) <= 1e-6 * tol):
            continue
        got = unfused_sparse_wmd(q, corpus, emb, swmd.SolverConfig(lam=lam, max_iter=max_iter,
                                                                    tol=tol))
        assert max_rel_err(got, g[f"t{n}_wmd"]) <= RTOL, n
        checked += 1
    assert checked >= 1


@pytest.mark.parametrize("v_r", [1, 3, 4, 7, 13, 19, 20, 31, 32, 33, 40, 47, 57, 64])
def test_unfused_query_lengths(v_r, oracle_lib):
    rng = np.random.default_rng(300 + v_r)
    V, N = 3000, 150
    emb = synth.normal_embeddings(rng, V, 64)
    cp, rows, vals = synth.zipf_corpus_csc(rng, V, N, 1, 60)
    q = synth.zipf_query(rng, V, v_r)
    corpus = CsrMatrix.from_csc(V, N, cp, rows, vals)
    got = unfused_sparse_wmd(q, corpus, emb, swmd.SolverConfig(lam=10.0, max_iter=15))
    want = oracle_lib.solve(q, cp, rows, vals, emb, lam=10.0, max_iter=15).wmd
    assert max_rel_err(got, want) <= RTOL


def test_unfused_rejects_long_queries():
    rng = np.random.default_rng(5)
    V = 500
    emb = synth.normal_embeddings(rng, V, 8)
    cp, rows, vals = synth.zipf_corpus_csc(rng, V, 10, 2, 9)
    corpus = CsrMatrix.from_csc(V, 10, cp, rows, vals)
    with pytest.raises(ValueError, match="v_r <= 64"):
        unfused_sparse_wmd(synth.zipf_query(rng, V, 65), corpus, emb, swmd.SolverConfig())


def test_unfused_zero_column_is_nonpositive_iterate():
    corpus = csr_from_triplets([(0, 0, 1.0)], 2, 2)  # column 1 empty: x stays 0
    vecs = np.array([[0.0, 0.0], [1.0, 0.0]])
    with pytest.raises(swmd.DegeneracyError, match=r"^nonpositive iterate entry$"):
        unfused_sparse_wmd(np.array([1.0, 0.0]), corpus, vecs,
                           swmd.SolverConfig(lam=1.0, max_iter=3))


def test_unfused_zero_denominator_matches_oracle(oracle_lib):
    V, N = 64, 3
    emb = np.zeros((V, 2))
    emb[:, 0] = np.linspace(0.0, 1.0, V)
    emb[[1, 17, 33], 1] = 1e3                 # exp(-lam * M) underflows to 0
    trip = [(i, 0, 1.0 + (i % 3)) for i in range(48)]
    trip += [(i, 1, 1.0) for i in (0, 2, 5)] + [(i, 2, 2.0) for i in (3, 4)]
    corpus = csr_from_triplets(trip, V, N)
    cp, rows, _, vals = corpus.csc_index()
    q = np.zeros(V)
    q[[0, 2]] = [0.5, 0.5]
    with pytest.raises(swmd.DegeneracyError) as exc:
        unfused_sparse_wmd(q, corpus, emb, swmd.SolverConfig(lam=50.0, max_iter=3))
    with pytest.raises(oracle_lib.OracleDegeneracy) as want:
        oracle_lib.solve(q, cp, rows, vals, emb, lam=50.0, max_iter=3)
    assert str(exc.value) == str(want.value) == "zero denominator at nonzero (1, 0)"


def test_unfused_plan_repeats_and_graph_replay():
    """Every solve restarts from x = 1/v_r: a second enqueue and a CUDA-graph
    replay of the plan (how bench.py times it) give the same bits."""
    import torch

    from paper_2107_06433_b200.baseline import UnfusedPlan
    from paper_2107_06433_b200.device import DeviceCorpus, DeviceEmbeddings
    from paper_2107_06433_b200.solver import SinkhornWorkspace

    inst = synth.zipf_instance("c1")
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15)
    sel, w = swmd.select_nonzero(inst.query)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        dc = DeviceCorpus.of(inst.corpus())
        de = DeviceEmbeddings.of(inst.embeddings)
        plan = UnfusedPlan(sel, w, dc, de, cfg, SinkhornWorkspace())
        plan.enqueue_distances()
        plan.enqueue_solve()
        first = plan.wmd.clone()
        plan.enqueue_solve()
        second = plan.wmd.clone()
        side.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            plan.enqueue_solve()
        plan.wmd.zero_()
        g.replay()
        side.synchronize()
        third = plan.wmd.clone()
    assert torch.equal(first, second) and torch.equal(first, third)
    assert max_rel_err(first.cpu().numpy(), golden("c1")["wmd"]) <= RTOL
