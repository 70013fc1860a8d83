"""Per-rank work of the column-sharded solve, measured one shard at a time on
one GPU (no rank waits on another): for world = 1, 2, 4, 8, the slowest
shard's device step (cost build + solve, L2 flushed before each step).  The
driver's multi-GPU run measures the real scaling; this is the compute part
of it, without the final all-gather.   python scripts/shard_projection.py c3"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_06433_b200 as swmd  # noqa: E402
from paper_2107_06433_b200 import _lib, synth  # noqa: E402
from paper_2107_06433_b200.device import DeviceEmbeddings, stream_ptr  # noqa: E402
from paper_2107_06433_b200.distributed import DeviceShardSolver, shard_bounds  # noqa: E402
from paper_2107_06433_b200.solver import QueryPlan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dev = torch.device("cuda", 0)
inst = synth.zipf_instance(name)
corpus = inst.corpus()
cfg = swmd.SolverConfig(lam=inst.config.lam, max_iter=inst.config.max_iter)
sel, w = swmd.select_nonzero(inst.query)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
solver = DeviceShardSolver(corpus, inst.embeddings, dev=dev)
de = DeviceEmbeddings.of(inst.embeddings, dev)
base = None
for world in (1, 2, 4, 8):
    bounds = shard_bounds(corpus, world)
    worst = 0.0
    for rank in range(world):
        c0, c1 = int(bounds[rank]), int(bounds[rank + 1])
        solver(sel, w, c0, c1, cfg, None)
        dc = solver._blocks[(c0, c1)]
        plan = QueryPlan(sel, w, dc, de, cfg, solver.ws)
        for _ in range(2):
            plan.enqueue_distances()
            plan.enqueue_solve()
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            _lib.call("swmd_l2_flush", flush.data_ptr(), flush.numel(), stream_ptr(dev))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            plan.enqueue_distances()
            plan.enqueue_solve()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        t = float(np.mean([x.elapsed_time(y) for x, y in ts]))
        worst = max(worst, t)
        del solver._blocks[(c0, c1)]
    base = base or worst
    print(f"{name} world={world}: slowest shard {worst:.3f} ms  "
          f"(x{base / worst:.2f} vs 1 GPU, compute-only efficiency {base / worst / world:.1%})", flush=True)
