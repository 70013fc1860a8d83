"""Max relative error of the B200 path against the committed reference
fixtures (tests/golden) for c1, c2 (full vectors) and c3/c5 (samples)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2107_06433_b200 as swmd  # noqa: E402
from paper_2107_06433_b200 import synth  # noqa: E402

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


for name in (sys.argv[1:] or ["c1", "c2", "c3", "c5"]):
    g = np.load(os.path.join(G, f"{name}.npz"))
    inst = synth.zipf_instance(name)
    res = swmd.sinkhorn_wmd(inst.query, inst.corpus(), inst.embeddings,
                            swmd.SolverConfig(lam=inst.config.lam, max_iter=inst.config.max_iter))
    if "wmd" in g:
        err = rel(res.wmd, g["wmd"])
    else:
        err = rel(res.wmd[:: int(g["sample_stride"])], g["sample"])
    top = np.argsort(res.wmd, kind="stable")[:100]
    print(f"{name}: max rel err {err:.3e}  top100 identical {bool(np.array_equal(top, g['top100']))}",
          flush=True)
