"""Per-column timeline of the persistent solve (SOLVE_TRACE build):
python scripts/solve_trace.py c2   (SWMD_LIB=<traced libswmd.so>)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_06433_b200 as swmd  # noqa: E402
from paper_2107_06433_b200 import _lib, synth  # noqa: E402
from paper_2107_06433_b200.device import DeviceCorpus, DeviceEmbeddings, stream_ptr  # noqa: E402
from paper_2107_06433_b200.solver import QueryPlan, SinkhornWorkspace  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
lib = _lib.lib()
for name in sys.argv[1:] or ["c2"]:
    inst = synth.zipf_instance(name)
    corpus = inst.corpus()
    cfg = swmd.SolverConfig(lam=inst.config.lam, max_iter=inst.config.max_iter)
    sel, w = swmd.select_nonzero(inst.query)
    dc = DeviceCorpus.of(corpus, dev)
    de = DeviceEmbeddings.of(inst.embeddings, dev)
    plan = QueryPlan(sel, w, dc, de, cfg, SinkhornWorkspace())
    for _ in range(3):
        plan.enqueue_distances()
        plan.enqueue_solve()
    torch.cuda.synchronize()
    _lib.call("swmd_l2_flush", flush.data_ptr(), flush.numel(), stream_ptr(dev))
    plan.enqueue_distances()
    plan.enqueue_solve()
    torch.cuda.synchronize()
    n = min(dc.n_cols, 1 << 20)
    buf = np.zeros((n, 4), dtype=np.int64)
    lib.swmd_debug_strace(ctypes.c_void_p(buf.ctypes.data), ctypes.c_int64(buf.nbytes))
    t0, t1 = buf[:, 0], buf[:, 1]
    ln = buf[:, 2] & 0xffffffff
    sm = buf[:, 2] >> 32
    base = t0.min()
    dur = (t1 - t0) / 1e3
    print(f"{name}: {n} columns, kernel span {(t1.max() - base) / 1e3:.1f} us "
          f"(first start -> last end), last start at {(t0.max() - base) / 1e3:.1f} us")
    for lo, hi in [(0, 16), (16, 32), (32, 48), (48, 64), (64, 81), (81, 1 << 30)]:
        m = (ln >= lo) & (ln < hi)
        if m.any():
            print(f"  len {lo:3d}-{min(hi, 999) - 1:3d}: {m.sum():6d} cols, duration mean {dur[m].mean():6.2f} us "
                  f"(min {dur[m].min():.2f}, max {dur[m].max():.2f}), per pass {dur[m].mean() / (cfg.max_iter + 1):.3f} us")
    # busy warps over time
    edges = np.linspace(0, (t1.max() - base) / 1e3, 11)
    st, en = (t0 - base) / 1e3, (t1 - base) / 1e3
    busy = [int(((st < b) & (en > b)).sum()) for b in edges[1:-1]]
    print("  columns in flight at 10..90 % of the span:", busy)
    per_sm = np.bincount(sm, minlength=148)
    print(f"  columns per SM: min {per_sm.min()} max {per_sm.max()}")
    edges = np.linspace(0, (t1.max() - base) / 1e3, 41)
    print("  in flight (40 buckets):", [int(((st < b) & (en > b)).sum()) for b in edges[1:-1]])
    out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
    os.makedirs(out, exist_ok=True)
    np.save(os.path.join(out, f"strace_{name}.npy"), np.stack([ln, sm, t0 - base, t1 - base], 1))
