"""c4 by padded query width: each group launch of the fp32 batch timed with
CUDA events (solver stream), summed per width.

    python scripts/c4_width_probe.py [reps]
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2107_06433_b200 as swmd  # noqa: E402
from paper_2107_06433_b200 import batch, synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inst = synth.zipf_instance("c4")
inst.embeddings.flags.writeable = False
corpus = inst.corpus()
cfg = swmd.SolverConfig(lam=10.0, max_iter=20, precision="f32")
ws = swmd.SinkhornWorkspace()
rec = []
orig = batch._solve_group32


def timed(dc, members, LD, max_iter, counter, s):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    orig(dc, members, LD, max_iter, counter, s)
    e1.record()
    rec.append((batch._block_width(members[0][5]), len(members), e0, e1))


batch._solve_group32 = timed
acc = defaultdict(lambda: [0, 0.0])
for r in range(reps + 1):
    rec.clear()
    swmd.sinkhorn_wmd_batch(inst.queries, corpus, inst.embeddings, cfg, workspace=ws)
    torch.cuda.synchronize()
    if r == 0:
        continue
    for w, nq, a, b in rec:
        acc[w][0] += nq
        acc[w][1] += a.elapsed_time(b)
tot = 0.0
for w in sorted(acc):
    nq, ms = acc[w]
    print(f"width {w:3d}: {nq // reps:2d} queries, {ms / reps:7.3f} ms per batch, {ms / nq:6.3f} ms per query")
    tot += ms / reps
print(f"solves total {tot:.2f} ms per batch")
