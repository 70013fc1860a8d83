"""Where the first public-API call's time goes at c2 (fresh corpus object and
embedding array): python scripts/cold_breakdown.py"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2107_06433_b200 as swmd  # noqa: E402
from paper_2107_06433_b200 import synth  # noqa: E402
from paper_2107_06433_b200.device import DeviceCorpus, DeviceEmbeddings, device  # noqa: E402
from paper_2107_06433_b200.solver import _native_plan  # noqa: E402

inst = synth.zipf_instance("c2")
c0, E0 = inst.corpus(), inst.embeddings.copy()
E0.flags.writeable = False
t_end = time.perf_counter() + 1.5          # GPU clocks up before anything is timed
while time.perf_counter() < t_end:
    swmd.sinkhorn_wmd(inst.query, c0, E0, swmd.SolverConfig())
torch.cuda.synchronize()
corpus = inst.corpus()
E = inst.embeddings.copy()
E.flags.writeable = False
ws = swmd.SinkhornWorkspace()
dev = device()


def t(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{label:32s} {1e3 * (time.perf_counter() - t0):8.2f} ms", flush=True)
    return r


dc = t("DeviceCorpus.of (CSC upload)", lambda: DeviceCorpus.of(corpus, dev))
de = t("DeviceEmbeddings.of (E upload)", lambda: DeviceEmbeddings.of(E, dev))
t("row norms", lambda: de.norms)
t("compact rows (E_c)", lambda: dc.compact_rows(de))
plan = t("native plan create", lambda: _native_plan(ws, dc, de, dev))
t("first run (graph capture)", lambda: plan.run(inst.query, swmd.SolverConfig()))
t("second run", lambda: plan.run(inst.query, swmd.SolverConfig()))
