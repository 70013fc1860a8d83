"""Latency-bound floor of the persistent solve: a corpus of a handful of
columns (one warp each, nothing else on the GPU), timed per column with the
SOLVE_TRACE build.  python scripts/latency_probe.py  (SWMD_LIB=<traced .so>)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_06433_b200 as swmd  # noqa: E402
from paper_2107_06433_b200 import _lib, synth  # noqa: E402
from paper_2107_06433_b200.device import DeviceCorpus, DeviceEmbeddings  # noqa: E402
from paper_2107_06433_b200.solver import QueryPlan, SinkhornWorkspace  # noqa: E402
from paper_2107_06433_b200.sparse import CsrMatrix  # noqa: E402

dev = torch.device("cuda", 0)
lib = _lib.lib()
base = synth.zipf_instance("c2")
rng = np.random.default_rng(0)
for length in (10, 16, 32, 48, 80):
    n = 4
    rows = np.concatenate([np.sort(rng.choice(base.n_vocab, length, replace=False)) for _ in range(n)])
    cp = np.arange(n + 1, dtype=np.int64) * length
    vals = np.full(rows.size, 1.0 / length)
    corpus = CsrMatrix.from_csc(base.n_vocab, n, cp, rows.astype(np.int64), vals)
    cfg = swmd.SolverConfig(lam=10.0, max_iter=15)
    sel, w = swmd.select_nonzero(base.query)
    dc = DeviceCorpus.of(corpus, dev)
    de = DeviceEmbeddings.of(base.embeddings, dev)
    plan = QueryPlan(sel, w, dc, de, cfg, SinkhornWorkspace())
    for _ in range(5):
        plan.enqueue_distances()
        plan.enqueue_solve()
    torch.cuda.synchronize()
    buf = np.zeros((n, 4), dtype=np.int64)
    lib.swmd_debug_strace(ctypes.c_void_p(buf.ctypes.data), ctypes.c_int64(buf.nbytes))
    dur = (buf[:, 1] - buf[:, 0]) / 1e3
    pt = np.zeros((64, 20), dtype=np.int64)
    lib.swmd_debug_ptrace(ctypes.c_void_p(pt.ctypes.data), ctypes.c_int64(pt.nbytes))
    per = np.diff(pt[:n, :15], axis=1)          # cycles between pass starts (passes 0..13)
    print(f"len {length:3d}: pass cycles (clock64, median over passes 1-13): {np.median(per[:, 1:], axis=1)}")
    print(f"len {length:3d}: column alone {dur.mean():6.2f} us -> {dur.mean() / 16 * 1e3:6.0f} ns "
          f"({dur.mean() / 16 * 1965:5.0f} cycles) per pass")
