"""Per-CTA timeline of the TMA cost build (COST_TRACE build): python scripts/cost_trace.py c2"""
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
    torch.cuda.synchronize()
    _lib.call("swmd_l2_flush", flush.data_ptr(), flush.numel(), stream_ptr(dev))
    plan.enqueue_distances()
    torch.cuda.synchronize()
    buf = np.zeros((1024, 8), dtype=np.uint64)
    lib.swmd_debug_trace(ctypes.c_void_p(buf.ctypes.data), ctypes.c_int64(buf.nbytes))
    n = int(np.count_nonzero(buf[:, 0]))
    t = buf[:n, :8].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    names = ["start", "q_loaded", "box0", "box_mid", "gram_end", "epi_end", "gram_end*", "epi_end*"]
    print("  (* = last warp of the CTA; others = warp 0)")
    print(f"{name}: {n} CTAs; per-stage µs after the first CTA start (min / median / max):")
    for k, nm in enumerate(names):
        print(f"  {nm:9s} {rel[:, k].min():7.2f} {np.median(rel[:, k]):7.2f} {rel[:, k].max():7.2f}")
