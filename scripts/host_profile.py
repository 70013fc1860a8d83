"""Host-side overhead of the public API at c2 (run on a GPU box)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2107_06433_b200 as swmd
from paper_2107_06433_b200 import synth

inst = synth.zipf_instance("c2")
inst.embeddings.flags.writeable = False   # a serving table: resident copy keyed by identity
corpus = inst.corpus()
cfg = swmd.SolverConfig()
ws = swmd.SinkhornWorkspace()
for _ in range(5):
    swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg, workspace=ws)
torch.cuda.synchronize()
t0 = time.perf_counter()
n = 200
for _ in range(n):
    swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg, workspace=ws)
print("e2e ms/call", 1e3 * (time.perf_counter() - t0) / n)
pr = cProfile.Profile()
pr.enable()
for _ in range(n):
    swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, cfg, workspace=ws)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
