"""A/B of the persistent solve's claim order on one GPU (c2 by default).

    python scripts/order_probe.py [c2] [reps]

Times the solve (CUDA events on the solver stream, L2 flushed before every
step) with the longest-first order and the planned orders of
paper_2107_06433_b200.schedule, and checks the distances are bitwise equal.
If gpurun_out/strace_<cfg>.npy (scripts/solve_trace.py) exists, a per-length
cost table fitted from that timeline is tried as well.
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2107_06433_b200 as swmd  # noqa: E402
from paper_2107_06433_b200 import _lib, schedule, synth  # noqa: E402
from paper_2107_06433_b200.device import DeviceCorpus, DeviceEmbeddings, stream_ptr  # noqa: E402
from paper_2107_06433_b200.solver import QueryPlan, SinkhornWorkspace  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
inst = synth.zipf_instance(name)
corpus = inst.corpus()
cfg = swmd.SolverConfig(lam=inst.config.lam, max_iter=inst.config.max_iter)
sel, w = swmd.select_nonzero(inst.query)
dc = DeviceCorpus.of(corpus, dev)
de = DeviceEmbeddings.of(inst.embeddings, dev)
plan = QueryPlan(sel, w, dc, de, cfg, SinkhornWorkspace())
lens = np.diff(dc.host_col_ptr)
sms = torch.cuda.get_device_properties(0).multi_processor_count
s = stream_ptr(dev)


def run(order_np, label):
    dc.order = torch.from_numpy(np.ascontiguousarray(order_np, dtype=np.int32)).to(dev)
    for _ in range(5):
        plan.enqueue_distances()
        plan.enqueue_solve()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        _lib.call("swmd_l2_flush", flush.data_ptr(), flush.numel(), s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        plan.enqueue_distances()
        a.record()
        plan.enqueue_solve()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    us = np.array([x.elapsed_time(y) * 1e3 for x, y in ts])
    print(f"{label:40s} solve mean {us.mean():6.2f} us  median {np.median(us):6.2f}  min {us.min():6.2f}",
          flush=True)
    return plan.wmd.clone()


slots = 16 * sms
ref = run(schedule.longest_first(lens), "longest-first")
variants = [("balanced (model)", schedule.balanced_order(lens, slots))]
rounds = (lens + 15) // 16
slab = (np.clip(lens - 32, 0, 48) + 15) // 16
for label, (f, r, sl) in {"r1 model 0.55/0.14/0.33": (0.55, 0.14, 0.33),
                          "flat 0.3/0.3/0.3": (0.3, 0.3, 0.3),
                          "r2 trace fit 0.5/0.02/0.2": (0.5, 0.02, 0.2),
                          "r2 trace fit x 0.5/0.1/0.25": (0.5, 0.1, 0.25),
                          "fixed-heavy 0.8/0.1/0.3": (0.8, 0.1, 0.3),
                          "slab-heavy 0.4/0.2/0.5": (0.4, 0.2, 0.5)}.items():
    cost = f + r * np.minimum(rounds, 2) + sl * slab
    variants.append((f"balanced ({label})", schedule.balanced_order(lens, slots, cost=cost)))
tr = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", f"strace_{name}.npy")
if os.path.exists(tr) and os.environ.get("ORDERS_ALL"):
    d = np.load(tr)
    dur = (d[:, 3] - d[:, 2]) / 1e3
    ln = d[:, 0].astype(np.int64)
    table = np.zeros(lens.max() + 1)
    for L in range(lens.max() + 1):
        m = ln == L
        table[L] = np.median(dur[m]) if m.any() else np.nan
    good = ~np.isnan(table)
    table = np.interp(np.arange(table.size), np.flatnonzero(good), table[good])
    cost = table[lens]
    print("trace cost table (len: us):", {L: round(float(table[L]), 2) for L in range(10, lens.max() + 1, 5)})
    variants.append(("balanced (trace table)", schedule.balanced_order(lens, slots, cost=cost)))
    for sl in (15 * sms, 17 * sms):
        variants.append((f"balanced (trace, slots {sl // sms}/SM)",
                         schedule.balanced_order(lens, sl, cost=cost)))
if os.environ.get("ORDERS_ALL"):
    rng = np.random.default_rng(0)
    variants.append(("random", rng.permutation(lens.size).astype(np.int32)))
    variants.append(("shortest-first", schedule.longest_first(lens)[::-1].copy()))
for label, order in variants:
    got = run(order, label)
    assert torch.equal(got, ref), f"{label}: distances differ"
print("all orders bitwise equal")
