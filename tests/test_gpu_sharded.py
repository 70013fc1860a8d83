"""sinkhorn_wmd_sharded's device path (NCCL, one rank on cuda:0): the solve
writes into the gather slot, one all_gather_into_tensor, one readback.
Multi-rank host logic is covered by tests/test_distributed_cpu.py (gloo); a
box with one GPU cannot host two NCCL ranks."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import golden, max_rel_err

import paper_2107_06433_b200 as swmd
from paper_2107_06433_b200 import synth
from paper_2107_06433_b200.sparse import csr_from_triplets

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


def test_sharded_device_gather_matches_golden(nccl_group):
    from paper_2107_06433_b200.distributed import DeviceShardSolver, sinkhorn_wmd_sharded

    g = golden("c2")
    inst = synth.zipf_instance("c2")
    corpus = inst.corpus()
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15)
    solver = DeviceShardSolver(corpus, inst.embeddings)
    res = sinkhorn_wmd_sharded(inst.query, corpus, inst.embeddings, cfg, solver=solver)
    assert max_rel_err(res.wmd, g["wmd"]) <= 1e-9
    assert res.iterations_run == 15 and not res.converged
    assert res.timings["iterations"] > 0.0
    single = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg).wmd
    assert np.array_equal(res.wmd, single)


def test_sharded_device_tol(nccl_group):
    from paper_2107_06433_b200.distributed import sinkhorn_wmd_sharded

    inst = synth.zipf_instance("c1", n_docs=60)
    corpus = inst.corpus()
    cfg = swmd.SolverConfig(lam=1.0, max_iter=300, tol=1e-10)
    res = sinkhorn_wmd_sharded(inst.query, corpus, inst.embeddings, cfg)
    one = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg)
    assert res.converged == one.converged and res.iterations_run == one.iterations_run
    assert np.array_equal(res.wmd, one.wmd)


def test_sharded_device_degeneracy_message(nccl_group):
    from paper_2107_06433_b200.distributed import sinkhorn_wmd_sharded

    corpus = csr_from_triplets([(0, 0, 1.0)], 2, 2)  # column 1 empty
    vecs = np.array([[0.0, 0.0], [1.0, 0.0]])
    cfg = swmd.SolverConfig(lam=1.0, max_iter=3)
    with pytest.raises(swmd.DegeneracyError) as want:
        swmd.sinkhorn_wmd(np.array([1.0, 0.0]), corpus, vecs, cfg)
    with pytest.raises(swmd.DegeneracyError) as got:
        sinkhorn_wmd_sharded(np.array([1.0, 0.0]), corpus, vecs, cfg)
    assert str(got.value) == str(want.value)


# -- workers -> GPUs in one process (sinkhorn_wmd_devices) --------------------------------------

def _devs(n):
    import torch

    return [torch.device("cuda", 0)] * n   # one GPU here: n blocks on it, one plan each


@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_devices_split_is_bitwise(n):
    from paper_2107_06433_b200.solver import sinkhorn_wmd_devices

    inst = synth.zipf_instance("c2")
    corpus = inst.corpus()
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15)
    one = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg)
    got = sinkhorn_wmd_devices(inst.query, corpus, inst.embeddings, cfg, _devs(n))
    assert np.array_equal(got.wmd, one.wmd)
    assert got.iterations_run == 15 and set(got.timings) == set(one.timings)
    assert isinstance(got.timings, dict)


def test_devices_tol_lockstep_matches_single():
    from paper_2107_06433_b200.solver import sinkhorn_wmd_devices

    inst = synth.zipf_instance("c1", n_docs=80)
    corpus = inst.corpus()
    cfg = swmd.SolverConfig(lam=1.0, max_iter=300, tol=1e-10)
    one = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg)
    got = sinkhorn_wmd_devices(inst.query, corpus, inst.embeddings, cfg, _devs(3))
    assert (got.iterations_run, got.converged) == (one.iterations_run, one.converged)
    assert np.array_equal(got.wmd, one.wmd)


def test_devices_degeneracy_is_the_single_solve_error(oracle_lib):
    from paper_2107_06433_b200.solver import sinkhorn_wmd_devices

    inst = synth.zipf_instance("c1", n_docs=40)
    cp, rows, vals = inst.col_ptr.copy(), inst.rows, inst.vals
    a, b = cp[33], cp[34]                       # empty column 33 (last block)
    rows = np.delete(rows, np.s_[a:b])
    vals = np.delete(vals, np.s_[a:b])
    cp[34:] -= (b - a)
    from paper_2107_06433_b200.sparse import CsrMatrix

    corpus = CsrMatrix.from_csc(inst.n_vocab, 40, cp, rows, vals)
    cfg = swmd.SolverConfig(max_iter=4)
    with pytest.raises(swmd.DegeneracyError) as want:
        swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg)
    with pytest.raises(swmd.DegeneracyError) as got:
        sinkhorn_wmd_devices(inst.query, corpus, inst.embeddings, cfg, _devs(3))
    assert str(got.value) == str(want.value)


def test_workers_on_one_gpu_is_the_plain_solve():
    """workers maps to min(workers, #GPUs) devices: one GPU -> the one-launch path."""
    inst = synth.zipf_instance("c1")
    corpus = inst.corpus()
    a = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, swmd.SolverConfig(workers=8))
    b = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, swmd.SolverConfig())
    assert np.array_equal(a.wmd, b.wmd)
