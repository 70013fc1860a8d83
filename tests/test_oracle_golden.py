"""Pin the CPU oracle (oracle/swmd_oracle.c) to outputs of the reference itself.

The fixtures in tests/golden/ were produced by the reference package
(tests/golden/make_golden.py imports /root/reference/pkg/src/sinkwmd).  The
oracle restates the reference's numba kernels in C with the same operation
order and no FMA contraction, so every comparison here is BITWISE.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden, small_instance

from paper_2107_06433_b200 import synth


def _fp(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def test_small_kernels_bitwise(small_golden, oracle_lib):
    g = small_golden
    o = oracle_lib
    for k in range(50):
        p = f"i{k}_"
        q, corpus, emb = small_instance(g, k)
        sel = np.flatnonzero(q > 0)
        cost = o.euclid_rows(emb, sel)
        assert np.array_equal(cost, g[p + "cost"]), k
        kern, kor, kcost = o.precompute(cost, q[sel], 10.0)
        assert np.array_equal(kern, g[p + "kernel"]), k
        assert np.array_equal(kor, g[p + "kor"]), k
        assert np.array_equal(kcost, g[p + "kcost"]), k
        u = g[p + "u"]
        x = o.fused_iter_serial(corpus.row_ptr, corpus.col_idx, corpus.values, kern, kor, u)
        assert np.array_equal(x, g[p + "x1"]), k
        wf = o.fused_final_serial(corpus.row_ptr, corpus.col_idx, corpus.values, kern, kcost, u)
        assert np.array_equal(wf, g[p + "final"]), k
        w = o.sddmm_serial(corpus.row_ptr, corpus.col_idx, corpus.values, kern, u)
        assert np.array_equal(w, g[p + "sddmm"]), k
        # the column-block traversal equals the CSR traversal bitwise
        cp, rows, _, vals = corpus.csc_index()
        xc = o.fused_iter_columns(cp, rows, vals, kern, kor, u, blocks=3)
        assert np.array_equal(xc, x), k


def test_small_solver_bitwise(small_golden, oracle_lib):
    g = small_golden
    for k in range(50):
        q, corpus, emb = small_instance(g, k)
        cp, rows, _, vals = corpus.csc_index()
        for lam in (1, 10):
            res = oracle_lib.solve(q, cp, rows, vals, emb, lam=float(lam), max_iter=15, blocks=2)
            assert np.array_equal(res.wmd, g[f"i{k}_wmd_lam{lam}"]), (k, lam)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_config_full_bitwise(name, oracle_lib):
    g = golden(name)
    inst = synth.zipf_instance(name)
    assert _fp(inst.col_ptr, inst.rows, inst.vals) == str(g["fp_corpus"])
    assert _fp(inst.query) == str(g["fp_query"])
    assert _fp(inst.embeddings) == str(g["fp_embeddings"])
    res = oracle_lib.solve(inst.query, inst.col_ptr, inst.rows, inst.vals, inst.embeddings,
                           lam=inst.config.lam, max_iter=inst.config.max_iter)
    assert np.array_equal(res.wmd, g["wmd"])


def test_c3_sampled_bitwise(oracle_lib):
    g = golden("c3")
    inst = synth.zipf_instance("c3")
    assert _fp(inst.col_ptr, inst.rows, inst.vals) == str(g["fp_corpus"])
    res = oracle_lib.solve(inst.query, inst.col_ptr, inst.rows, inst.vals, inst.embeddings,
                           lam=10.0, max_iter=15)
    stride = int(g["sample_stride"])
    assert np.array_equal(res.wmd[::stride], g["sample"])
    order = np.argsort(res.wmd, kind="stable")
    assert np.array_equal(order[:100], g["top100"])
    assert float(np.sum(res.wmd)) == float(g["wmd_sum"])


def test_column_blocks_match_reference_semantics(oracle_lib):
    from paper_2107_06433_b200.sparse import column_blocks

    rng = np.random.default_rng(5)
    for _ in range(200):
        lens = rng.integers(0, 9, size=int(rng.integers(1, 40)))
        cp = np.concatenate(([0], np.cumsum(lens))).astype(np.int64)
        for p in (1, 2, 3, 5, 8, 64):
            assert np.array_equal(oracle_lib.column_blocks(cp, p), column_blocks(cp, p))


def test_c4_oracle_pinned_on_four_queries(oracle_lib):
    g = golden("c4")
    inst = synth.zipf_instance("c4")
    assert _fp(inst.col_ptr, inst.rows, inst.vals) == str(g["fp_corpus"])
    E64 = inst.embeddings.astype(np.float64)
    stride = int(g["sample_stride"])
    for k in (0, 21, 42, 63):
        res = oracle_lib.solve(inst.queries[k], inst.col_ptr, inst.rows, inst.vals, E64,
                               lam=10.0, max_iter=20)
        assert np.array_equal(res.wmd[::stride], g["sample"][k]), k


def test_oracle_tol_path_pinned(oracle_lib):
    """The oracle's tol early exit equals the reference's (tests/golden/tol.npz,
    solver.py:170-183): iterations_run, converged, every max|dx| and wmd bitwise."""
    from conftest import tol_case

    g = golden("tol")
    for n in range(int(g["n_cases"])):
        q, corpus, emb, lam, max_iter, tol = tol_case(g, n)
        cp, rows, _, vals = corpus.csc_index()
        res = oracle_lib.solve(q, cp, rows, vals, emb, lam=lam, max_iter=max_iter, tol=tol,
                               blocks=3)
        assert res.iterations_run == int(g[f"t{n}_iterations"]), n
        assert res.converged == bool(g[f"t{n}_converged"]), n
        assert np.array_equal(res.deltas, g[f"t{n}_deltas"]), n
        assert np.array_equal(res.wmd, g[f"t{n}_wmd"]), n


def test_check_topk_rules():
    """The strict top-k checker the GPU parity tests use."""
    from conftest import check_topk

    ref = np.array([0.5, 0.1, 0.3, 0.2, 0.9, 0.30000000000000004])
    idx = np.argsort(ref, kind="stable")
    assert check_topk(ref, idx, ref[idx], 3) == []
    # swapping the near-tie at ranks 2/3 (docs 2 and 5) is legitimate at k=3 and k=4
    got = ref.copy()
    got[5] = 0.3 - 1e-16
    assert check_topk(got, idx, ref[idx], 3, ref_full=ref) == [(2, 5, 2)]
    # a real reordering is not
    bad = ref.copy()
    bad[0] = 0.15
    with pytest.raises(AssertionError):
        check_topk(bad, idx, ref[idx], 3, ref_full=ref)
    with pytest.raises(AssertionError):                 # outside doc, no boundary tie
        check_topk(bad, idx[:4], ref[idx][:4], 3)


def test_oracle_pinned_on_edge_cases(oracle_lib):
    """The oracle against the reference's edge-case runs (tests/golden/edge.npz):
    max_iter = 1, float32 embeddings coerced to float64, tol = 0."""
    from paper_2107_06433_b200.sparse import CsrMatrix

    g = golden("edge")
    V, N = g["emb"].shape[0], g["wmd_iter1"].shape[0]
    cp, rows, _, vals = CsrMatrix(V, N, g["row_ptr"], g["col_idx"], g["values"]).csc_index()
    r = oracle_lib.solve(g["q"], cp, rows, vals, g["emb"], lam=10.0, max_iter=1)
    assert np.array_equal(r.wmd, g["wmd_iter1"])
    r = oracle_lib.solve(g["q"], cp, rows, vals, g["emb"].astype(np.float32).astype(np.float64),
                         lam=10.0, max_iter=15)
    assert np.array_equal(r.wmd, g["wmd_f32emb"])
    r = oracle_lib.solve(g["q"], cp, rows, vals, g["emb"], lam=10.0, max_iter=9, tol=0.0)
    assert np.array_equal(r.wmd, g["wmd_tol0"])
    assert r.iterations_run == int(g["tol0_iters"]) and r.converged == bool(g["tol0_conv"])
