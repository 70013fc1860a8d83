"""Host-side overhead of sinkhorn_wmd_batch(precision='f32') at c4 (GPU box)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2107_06433_b200 as swmd
from paper_2107_06433_b200 import synth

inst = synth.zipf_instance("c4")
inst.embeddings.flags.writeable = False
corpus = inst.corpus()
cfg = swmd.SolverConfig(lam=10.0, max_iter=20, precision="f32")
ws = swmd.SinkhornWorkspace()
for _ in range(2):
    swmd.sinkhorn_wmd_batch(inst.queries, corpus, inst.embeddings, cfg, workspace=ws)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    res = swmd.sinkhorn_wmd_batch(inst.queries, corpus, inst.embeddings, cfg, workspace=ws)
print("batch ms", 1e3 * (time.perf_counter() - t0) / 3,
      "device ms", 1e3 * sum(r.timings["distances"] + r.timings["iterations"] for r in res))
pr = cProfile.Profile()
pr.enable()
swmd.sinkhorn_wmd_batch(inst.queries, corpus, inst.embeddings, cfg, workspace=ws)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
