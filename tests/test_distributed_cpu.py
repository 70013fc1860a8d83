"""The multi-GPU sharding logic, run as 2 gloo ranks on CPU.

The per-shard compute is injected: here a CPU shard solver built on the
oracle (the checker), on the GPU box the DeviceShardSolver.  What is under
test is the product's host logic in distributed.py — the column_blocks
split, the padded all-gather, the per-iteration all-reduce(MAX) of the tol
path and the cross-rank degeneracy merge.
"""

from __future__ import annotations

import os
import pickle
import re
import socket
import sys
import tempfile

import numpy as np
import pytest

from conftest import REPO


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleShardSolver:
    """Reference semantics on one column block, via the oracle kernels."""

    def __init__(self, corpus, emb):
        self.cp, self.rows, _, self.vals = corpus.csc_index()
        self.emb = emb

    def __call__(self, sel, weights, c0, c1, config, allreduce_max):
        import oracle
        from paper_2107_06433_b200.solver import DegEvent, ShardResult

        cost = oracle.euclid_rows(self.emb, sel)
        K, KoR, KM = oracle.precompute(cost, weights, config.lam)
        a, b = self.cp[c0], self.cp[c1]
        cp = self.cp[c0: c1 + 1] - a
        rows, vals = self.rows[a:b], self.vals[a:b]
        v_r = sel.size
        x = np.full((c1 - c0, v_r), 1.0 / v_r)
        iters, converged, event = 0, False, None

        def check(xx, code):
            if xx.size and np.min(xx) <= 0.0:
                f = int(np.argmin(xx))
                val, flat = float(xx.flat[f]), c0 * v_r + f
                return DegEvent(code, (val, flat), f"nonpositive iterate entry {val} at flat index {flat}")
            return None

        def zero(exc, code):
            i, j = (int(v) for v in re.findall(r"-?\d+", str(exc))[:2])
            return DegEvent(code, (i, j + c0), f"zero denominator at nonzero ({i}, {j + c0})")

        for t in range(config.max_iter):
            event = check(x, 2 * t)
            if event is None:
                try:
                    xn = oracle.fused_iter_columns(cp, rows, vals, K, KoR, 1.0 / x, blocks=1)
                except oracle.OracleDegeneracy as exc:
                    event = zero(exc, 2 * t + 1)
                    xn = x
            iters += 1
            fail = event is not None
            delta = float(np.max(np.abs(xn - x))) if xn.size else 0.0
            if allreduce_max is not None:
                g = allreduce_max(np.array([delta, 1.0 if fail else 0.0]))
                delta, fail = float(g[0]), bool(g[1] > 0)
            x = xn
            if fail:
                break
            if config.tol is not None and delta < config.tol:
                converged = True
                break
        wmd = np.zeros(c1 - c0)
        if event is None and not (allreduce_max is not None and fail):
            event = check(x, 2 * iters)
            if event is None:
                try:
                    wmd = oracle.fused_final_columns(cp, rows, vals, K, KM, 1.0 / x, blocks=1)
                except oracle.OracleDegeneracy as exc:
                    event = zero(exc, 2 * iters + 1)
        return ShardResult(wmd, iters, converged, {}, event)


def _worker(rank, world, port, case, out_dir):
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import torch.distributed as dist

    from paper_2107_06433_b200 import SolverConfig
    from paper_2107_06433_b200.distributed import sinkhorn_wmd_sharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    query, corpus, emb, cfg = _case(case)
    solver = OracleShardSolver(corpus, emb)
    try:
        res = sinkhorn_wmd_sharded(query, corpus, emb, cfg, solver=solver)
        out = ("ok", res.wmd, res.iterations_run, res.converged)
    except ArithmeticError as exc:
        out = ("err", str(exc))
    with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as f:
        pickle.dump(out, f)
    dist.destroy_process_group()


def _case(case):
    from paper_2107_06433_b200 import SolverConfig, synth
    from paper_2107_06433_b200.sparse import CsrMatrix

    if case == "plain":
        inst = synth.zipf_instance("c1", n_docs=90)
        return inst.query, inst.corpus(), inst.embeddings, SolverConfig()
    if case == "tol":
        inst = synth.zipf_instance("c1", n_docs=60)
        return inst.query, inst.corpus(), inst.embeddings, SolverConfig(lam=1.0, max_iter=300,
                                                                        tol=1e-10)
    if case == "degenerate":
        inst = synth.zipf_instance("c1", n_docs=40)
        cp, rows, vals = inst.col_ptr.copy(), inst.rows, inst.vals
        # empty column 33 (it lands in the second shard)
        a, b = cp[33], cp[34]
        rows = np.delete(rows, np.s_[a:b])
        vals = np.delete(vals, np.s_[a:b])
        cp[34:] -= (b - a)
        corpus = CsrMatrix.from_csc(inst.n_vocab, 40, cp, rows, vals)
        return inst.query, corpus, inst.embeddings, SolverConfig(max_iter=4)
    raise KeyError(case)


def _run(case, world):
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), case, d), nprocs=world,
                           join=True, start_method="spawn")
        outs = []
        for r in range(world):
            with open(os.path.join(d, f"r{r}.pkl"), "rb") as f:
                outs.append(pickle.load(f))
    return outs


@pytest.mark.parametrize("case", ["plain", "tol", "degenerate"])
def test_two_ranks_match_one(case):
    one = _run(case, 1)[0]
    two = _run(case, 2)
    for out in two:
        assert out[0] == one[0]
        if one[0] == "ok":
            assert np.array_equal(out[1], one[1])
            assert out[2] == one[2] and out[3] == one[3]
        else:
            assert out[1] == one[1]


def test_one_rank_matches_oracle_solve():
    import oracle

    query, corpus, emb, cfg = _case("plain")
    got = _run("plain", 1)[0]
    cp, rows, _, vals = corpus.csc_index()
    want = oracle.solve(query, cp, rows, vals, emb).wmd
    assert np.array_equal(got[1], want)


def test_degenerate_message_matches_oracle():
    import oracle

    query, corpus, emb, cfg = _case("degenerate")
    cp, rows, _, vals = corpus.csc_index()
    with pytest.raises(oracle.OracleDegeneracy) as want:
        oracle.solve(query, cp, rows, vals, emb, max_iter=4)
    outs = _run("degenerate", 2)
    assert all(o == ("err", str(want.value)) for o in outs)


def test_tol_converges_globally():
    outs = _run("tol", 2)
    assert all(o[3] for o in outs) and outs[0][2] == outs[1][2] < 300
