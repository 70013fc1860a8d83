"""Time the cost build alone (L2 flushed before each launch): python scripts/cost_probe.py c2 c3"""
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
    ts = []
    for _ in range(50):
        _lib.call("swmd_l2_flush", flush.data_ptr(), flush.numel(), stream_ptr(dev))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.enqueue_distances()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ts]
    print(f"{os.environ.get('TAG', '')} {name}: cost build {1e3 * np.mean(ms):.1f} us "
          f"(min {1e3 * np.min(ms):.1f})", flush=True)
