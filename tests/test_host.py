"""Host-side logic (no GPU): containers, config, argument checks, the C ABI exports."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO

import paper_2107_06433_b200 as swmd
from paper_2107_06433_b200 import _lib, synth
from paper_2107_06433_b200.sparse import (
    CsrMatrix,
    SparseVector,
    StructuralError,
    column_blocks,
    csr_from_triplets,
    csr_validate,
    nnz_partition,
    partitions_to_arrays,
)


# -- the C ABI --------------------------------------------------------------------------

def _header_symbols() -> list[str]:
    text = open(os.path.join(REPO, "include", "swmd.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return re.findall(r"^\s*(?:int|int64_t)\s+(swmd_\w+)\s*\(", text, flags=re.M)


def test_library_exports_every_header_symbol():
    syms = _header_symbols()
    assert len(syms) >= 12
    lib = _lib.load()           # loads without a GPU
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.swmd_abi_version() == 2


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cuda_means_loud_failure(monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    inst = swmd.synth.zipf_instance("c1", n_docs=5) if hasattr(swmd, "synth") else \
        synth.zipf_instance("c1", n_docs=5)
    with pytest.raises(_lib.NativeUnavailable):
        swmd.sinkhorn_wmd(inst.query, inst.corpus(), inst.embeddings, swmd.SolverConfig())


# -- SolverConfig / init_x / update_u (solver.py:22-103) ---------------------------------

@pytest.mark.parametrize("kwargs", [dict(lam=0.0), dict(lam=-1.0), dict(max_iter=0),
                                    dict(workers=0), dict(tol=-1e-9),
                                    dict(cost_mode="fast")])
def test_config_invalid(kwargs):
    with pytest.raises(ValueError):
        swmd.SolverConfig(**kwargs)


def test_init_x_and_update_u():
    assert swmd.init_x(1, 1).tolist() == [[1.0]]
    x = swmd.init_x(19, 5000)
    assert x.shape == (5000, 19) and np.all(x == 1.0 / 19)
    with pytest.raises(ValueError):
        swmd.init_x(0, 1)
    assert swmd.update_u(np.array([[0.25]])).tolist() == [[4.0]]
    with pytest.raises(swmd.DegeneracyError, match="nonpositive iterate entry 0.0 at flat index 1"):
        swmd.update_u(np.array([[1.0, 0.0]]))


def test_shape_mismatch_and_empty_query_before_device():
    inst = synth.zipf_instance("c1", n_docs=4)
    corpus = inst.corpus()
    with pytest.raises(ValueError, match="shape mismatch"):
        swmd.sinkhorn_wmd(inst.query[:-1], corpus, inst.embeddings, swmd.SolverConfig())
    with pytest.raises(swmd.EmptyQueryError):
        swmd.sinkhorn_wmd(np.zeros(inst.n_vocab), corpus, inst.embeddings, swmd.SolverConfig())


def test_select_nonzero():
    sel, r = swmd.select_nonzero(np.array([0.0, 0.5, 0.0, 0.5]))
    assert sel.tolist() == [1, 3] and r.tolist() == [0.5, 0.5]
    with pytest.raises(swmd.EmptyQueryError):
        swmd.select_nonzero(np.zeros(2))
    with pytest.raises(ValueError):
        swmd.select_nonzero(np.array([-0.1, 1.1]))


# -- containers (sparse.py) -----------------------------------------------------------------

def test_from_csc_round_trip_matches_csr_construction():
    inst = synth.zipf_instance("c1", n_docs=60)
    a = CsrMatrix.from_csc(inst.n_vocab, inst.n_docs, inst.col_ptr, inst.rows, inst.vals)
    rp, ci, v = synth.csc_to_csr(inst.n_vocab, inst.n_docs, inst.col_ptr, inst.rows, inst.vals)
    b = CsrMatrix(inst.n_vocab, inst.n_docs, rp, ci, v)
    assert np.array_equal(a.row_ptr, b.row_ptr)
    assert np.array_equal(a.col_idx, b.col_idx)
    assert np.array_equal(a.values, b.values)
    for x, y in zip(a.csc_index(), b.csc_index()):
        assert np.array_equal(x, y)
    # pos maps CSC slots to CSR positions
    cp, rows, pos, vals = b.csc_index()
    assert np.array_equal(b.values[pos], vals)
    assert np.array_equal(b.row_of_nnz()[pos], rows)


def test_csc_rows_ascend_within_columns():
    inst = synth.zipf_instance("c2", n_docs=300)
    cp, rows, _, _ = inst.corpus().csc_index()
    for j in range(inst.n_docs):
        seg = rows[cp[j]:cp[j + 1]]
        assert np.all(seg[1:] > seg[:-1])


def test_csr_from_triplets_sums_and_drops():
    m = csr_from_triplets([(0, 1, 1.0), (0, 1, 2.0), (1, 0, 1.0), (1, 0, -1.0)], 2, 2)
    assert m.nnz == 1 and m.col_idx.tolist() == [1] and m.values.tolist() == [3.0]
    assert csr_validate(m) == []
    with pytest.raises(StructuralError):
        csr_from_triplets([(2, 0, 1.0)], 2, 2)


def test_sparse_vector():
    v = SparseVector(5, [1, 3], [0.25, 0.75])
    assert v.nnz == 2 and v.to_dense().tolist() == [0, 0.25, 0, 0.75, 0]
    for bad in (([3, 1], [1.0, 1.0]), ([1, 5], [1.0, 1.0]), ([1], [0.0])):
        with pytest.raises(StructuralError):
            SparseVector(5, *bad)


def test_immutability():
    m = csr_from_triplets([(0, 0, 1.0)], 1, 1)
    with pytest.raises(AttributeError):
        m.n_rows = 3
    with pytest.raises(ValueError):
        m.values[0] = 2.0


def test_partitions_and_blocks():
    rng = np.random.default_rng(7)
    for _ in range(300):
        counts = rng.integers(0, 6, size=int(rng.integers(1, 40)))
        rp = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
        nnz = int(rp[-1])
        p = int(rng.integers(1, nnz + 3))
        parts = nnz_partition(rp, nnz, p)
        sizes = [q.size for q in parts]
        assert sum(sizes) == nnz and max(sizes) - min(sizes) <= 1
        assert sizes == sorted(sizes, reverse=True)
        for q in parts:
            if q.nnz_begin < nnz:
                assert rp[q.start_row] <= q.nnz_begin < rp[q.start_row + 1]
        bounds, starts = partitions_to_arrays(parts)
        assert bounds[-1] == nnz
        b = column_blocks(rp, min(p, 8))
        assert b[0] == 0 and b[-1] == rp.size - 1 and np.all(np.diff(b) >= 0)


# -- the synthetic generator ---------------------------------------------------------------------

def test_generator_shapes_and_normalisation():
    inst = synth.zipf_instance("c2", n_docs=2000)
    lens = np.diff(inst.col_ptr)
    assert lens.min() >= 10 and lens.max() <= 80
    sums = np.add.reduceat(inst.vals, inst.col_ptr[:-1])
    assert np.allclose(sums, 1.0, rtol=0, atol=1e-12)
    assert np.count_nonzero(inst.query) == 19
    assert abs(inst.query.sum() - 1.0) < 1e-12
    assert np.allclose(np.linalg.norm(inst.embeddings, axis=1), 1.0)
    # Zipf head: the top word occurs in nearly every document
    assert np.mean(inst.rows[inst.col_ptr[:-1]] == 0) > 0.9


def test_generator_is_deterministic_and_thread_independent():
    a = synth.zipf_instance("c1")
    b = synth.zipf_instance("c1")
    assert np.array_equal(a.rows, b.rows) and np.array_equal(a.vals, b.vals)
    rng1, rng2 = np.random.default_rng(11), np.random.default_rng(11)
    x = synth.zipf_corpus_csc(rng1, 1000, 300, 5, 20, chunk=40)
    y = synth.zipf_corpus_csc(rng2, 1000, 300, 5, 20, chunk=40)
    for p, q in zip(x, y):
        assert np.array_equal(p, q)


def test_embedding_fingerprint_sees_one_element_edits():
    """a writeable table is hashed in full, so editing one element
    (anywhere) changes its cache key; a read-only table is sampled."""
    from paper_2107_06433_b200.device import _fingerprint, _read_only

    E = np.random.default_rng(0).standard_normal((20_000, 30))
    f0 = _fingerprint(E)
    old = E[5, 7]
    E[5, 7] = old + 1.0
    f1 = _fingerprint(E)
    E[5, 7] = old
    assert f1 != f0 and _fingerprint(E) == f0
    v = E.view()
    v.flags.writeable = False
    assert not _read_only(v)                    # its base is still writeable
    R = E.copy()
    R.flags.writeable = False
    assert _read_only(R)


def test_every_package_module_imports():
    """Modules imported lazily on the GPU paths (batch, baseline, distributed)
    must at least import on a CPU-only box."""
    import importlib
    import pkgutil

    import paper_2107_06433_b200 as pkg

    for m in pkgutil.iter_modules(pkg.__path__):
        if m.name.startswith("lib"):          # libswmd.so: the ctypes library, not a module
            continue
        importlib.import_module(f"paper_2107_06433_b200.{m.name}")


def test_native_select_matches_select_nonzero():
    """swmd_select_query (the native scan behind the public API and the batch
    path) returns select_nonzero's (sel, weights) and raises its errors
    (kernels.py:74-88), NaN entries skipped like numpy's r > 0."""
    import numpy as np

    from paper_2107_06433_b200.kernels import EmptyQueryError, select_nonzero
    from paper_2107_06433_b200.solver import SinkhornWorkspace, select_native

    rng = np.random.default_rng(3)
    ws = SinkhornWorkspace()
    for n in (1, 31, 32, 33, 100, 5000):
        for _ in range(10):
            q = np.zeros(n)
            k = int(rng.integers(1, min(n, 300) + 1))
            idx = rng.choice(n, size=k, replace=False)
            q[idx] = rng.random(k) + 1e-3
            if n > 40:
                q[rng.choice(n, 3, replace=False)] = np.nan
            a, b = select_native(q, ws), select_nonzero(q)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    with pytest.raises(ValueError, match="nonnegative"):
        select_native(np.array([0.0, -1.0, 2.0]), ws)
    with pytest.raises(EmptyQueryError):
        select_native(np.zeros(64), ws)
