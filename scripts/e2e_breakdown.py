"""Where the public-API time goes at c2 (GPU box): python scripts/e2e_breakdown.py"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_06433_b200 as swmd  # noqa: E402
from paper_2107_06433_b200 import synth  # noqa: E402
from paper_2107_06433_b200.device import DeviceCorpus, DeviceEmbeddings, device  # noqa: E402
from paper_2107_06433_b200.solver import _native_plan  # noqa: E402

inst = synth.zipf_instance(sys.argv[1] if len(sys.argv) > 1 else "c2")
corpus = inst.corpus()
cfg = swmd.SolverConfig()
ws = swmd.SinkhornWorkspace()
q, E = inst.query, inst.embeddings
for _ in range(20):
    swmd.sinkhorn_wmd(q, corpus, E, cfg, workspace=ws)
torch.cuda.synchronize()
n = 300


def timeit(label, fn):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{label:40s} {1e6 * (time.perf_counter() - t0) / n:8.1f} us", flush=True)


dev = device()
dc = DeviceCorpus.of(corpus, dev)
de = DeviceEmbeddings.of(E, dev)
plan = _native_plan(ws, dc, de, dev)
timeit("sinkhorn_wmd (public API)", lambda: swmd.sinkhorn_wmd(q, corpus, E, cfg, workspace=ws))
timeit("device()", device)
timeit("DeviceCorpus.of", lambda: DeviceCorpus.of(corpus, dev))
timeit("DeviceEmbeddings.of", lambda: DeviceEmbeddings.of(E, dev))
timeit("_native_plan", lambda: _native_plan(ws, dc, de, dev))
timeit("plan.run (one C call)", lambda: plan.run(q, cfg))
t = plan.times
print("plan times_ms: cost %.4f solve %.4f | host: select %.4f enqueued %.4f synced %.4f copied %.4f"
      % tuple(float(v) for v in t[:6]))
from paper_2107_06433_b200 import _lib  # noqa: E402
st = np.zeros(200, dtype=np.int64)
timeit("swmd_select_query", lambda: _lib.lib().swmd_select_query(q.ctypes.data, q.size,
                                                                 st.ctypes.data, 64))
