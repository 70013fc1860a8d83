"""c4 breakdown on one GPU: the batched fp32 cost build and each query's solve
(CUDA events on the solver stream), by query width.

    python scripts/c4_probe.py [reps]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_06433_b200 as swmd  # noqa: E402
from paper_2107_06433_b200 import batch, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inst = synth.zipf_instance("c4")
corpus = inst.corpus()
cfg = swmd.SolverConfig(lam=10.0, max_iter=20, precision="f32")
ws = swmd.SinkhornWorkspace()
rec = []
orig = batch._solve32


def timed(*a, **k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    orig(*a, **k)
    e1.record()
    rec.append((a[4], e0, e1))


batch._solve32 = timed
for r in range(reps + 1):
    rec.clear()
    t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t[0].record()
    res = swmd.sinkhorn_wmd_batch(inst.queries, corpus, inst.embeddings, cfg, workspace=ws)
    t[1].record()
    torch.cuda.synchronize()
    if r == 0:
        continue
    solves = [(v, a.elapsed_time(b)) for v, a, b in rec]
    tot = t[0].elapsed_time(t[1])
    s_sum = sum(ms for _, ms in solves)
    print(f"rep {r}: batch {tot:.2f} ms (events), solves sum {s_sum:.2f} ms, "
          f"cost build {res[0].timings['distances'] * len(res) * 1e3:.2f} ms")
vr = np.array([v for v, _ in solves])
ms = np.array([m for _, m in solves])
for lo, hi in ((1, 16), (17, 32), (33, 48), (49, 64)):
    m = (vr >= lo) & (vr <= hi)
    if m.any():
        print(f"v_r {lo:2d}-{hi:2d}: {m.sum():2d} queries, mean solve {ms[m].mean():.3f} ms, "
              f"{ms[m].mean() / vr[m].mean() * 1e3:.1f} us per word")
print("nnz", inst.nnz, "sum v_r", int(vr.sum()))
