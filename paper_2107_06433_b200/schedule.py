"""Work order of the persistent solve: which document column each warp claims next.

The persistent solve kernels run a fixed number of resident warps ("slots";
one column per warp at a time) that claim columns through one atomic counter
in the order of ``DeviceCorpus.order``.  A column's time is nearly fixed by
its length (a dependency chain of 16 passes), so the launch's span is a
makespan-scheduling problem: ``N`` jobs with known lengths on ``S`` identical
machines, each machine pulling the next job when it frees up.

Longest-first (LPT) is near optimal when every slot runs many columns (c3:
1M columns on 2,368 slots), but at c2 (5,000 columns, 2.1 per slot) it is
the textbook bad case: after two columns per slot the remaining 264 shortest
columns start when every slot frees up at about the same time and each adds a
whole short-column latency (~12 us) to the span.

``balanced_order`` plans the schedule instead: MULTIFIT (first-fit-decreasing
under a binary-searched capacity) packs the predicted column times into ``S``
bins — the shortest columns end up three to a bin, the others in long+short
pairs — and the plan is serialised into the claim order by each column's
planned start time, so the dynamic claim reproduces the plan when the
predictions hold and degrades gracefully when they do not.

The C runtime has the same planner (``swmd_schedule_order``, called by
``device.claim_order``); this module is its numpy restatement, used by the
tests to check it and by scripts/order_probe.py.
"""

from __future__ import annotations

import numpy as np

__all__ = ["column_cost", "balanced_order", "longest_first", "plan_makespan"]

# per-pass time model of reg_solve (relative units): a fixed part (owner
# reduction, reciprocal, u publish), the register rounds (processed
# together), then one serial step per 16-nonzero slab / L2 round.  The
# constants are the A/B winner on the B200 (profiles/r02_summary.md): the
# realised span is not monotone in model accuracy — a fit to the c2
# SOLVE_TRACE timeline (0.41/0.22/0.36) planned a 2 us longer span.  With the
# shuffle reduction (REG_SHRED) the fixed per-pass part shrank and the flat
# model (0.3/0.3/0.3) won: 55.6 us vs 56.9 us for the round-1 constants
COST_FIXED = 0.3
COST_REG = 0.3
COST_SLAB = 0.3
COST_L2 = 0.4


def column_cost(lens: np.ndarray, reg_rounds: int = 2, slab_rows: int = 48) -> np.ndarray:
    """Predicted relative time of one column of each length."""
    lens = np.asarray(lens, dtype=np.int64)
    rounds = (lens + 15) // 16
    reg = np.minimum(rounds, reg_rounds)
    rq = 16 * reg_rounds
    slab = (np.clip(lens - rq, 0, slab_rows) + 15) // 16
    l2 = (np.maximum(lens - rq - slab_rows, 0) + 15) // 16
    return COST_FIXED + COST_REG * reg + COST_SLAB * slab + COST_L2 * l2


def longest_first(lens: np.ndarray) -> np.ndarray:
    return np.argsort(-np.asarray(lens), kind="stable").astype(np.int32)


def _ffd(w_sorted: np.ndarray, slots: int, cap: float) -> np.ndarray | None:
    """First-fit-decreasing into ``slots`` bins of capacity ``cap``; bin of
    every item or None when the items do not fit."""
    room = np.full(slots, cap)
    out = np.empty(w_sorted.size, dtype=np.int64)
    eps = cap * 1e-12
    for k, w in enumerate(w_sorted):
        b = int(np.argmax(room >= w - eps))
        if room[b] < w - eps:
            return None
        room[b] -= w
        out[k] = b
    return out


def _lpt_makespan(w_sorted: np.ndarray, slots: int) -> float:
    import heapq

    heap = [0.0] * slots
    for w in w_sorted:
        heapq.heapreplace(heap, heap[0] + w)
    return max(heap)


def balanced_order(lens: np.ndarray, slots: int, cost: np.ndarray | None = None,
                   max_ratio: int = 8, iters: int = 24, reg_rounds: int = 2,
                   slab_rows: int = 48) -> np.ndarray:
    """Claim order (int32 column ids) for ``slots`` resident warps.

    Falls back to longest-first when every slot runs many columns
    (N > max_ratio * slots: the tail is a negligible share) or when every
    column starts in the first wave (N <= slots).
    """
    lens = np.asarray(lens, dtype=np.int64)
    n = lens.size
    if n <= slots or n > max_ratio * slots or slots < 1:
        return longest_first(lens)
    w = (column_cost(lens, reg_rounds, slab_rows) if cost is None
         else np.asarray(cost, dtype=np.float64))
    idx = np.argsort(-w, kind="stable")
    ws = w[idx]
    lo = max(ws.sum() / slots, ws[0])
    hi = _lpt_makespan(ws, slots)
    best = _ffd(ws, slots, hi * (1 + 1e-9))
    if best is None:          # cannot happen (LPT packs into its own makespan)
        return longest_first(lens)
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        got = _ffd(ws, slots, mid)
        if got is None:
            lo = mid
        else:
            hi, best = mid, got
        if hi - lo <= 1e-4 * hi:
            break
    # planned start of every item: prefix sums inside its bin (items of a bin
    # arrive in decreasing cost order, the FFD order)
    start = np.empty(n)
    fill = np.zeros(slots)
    for k in range(n):
        b = best[k]
        start[k] = fill[b]
        fill[b] += ws[k]
    # claim order = planned start time; the first wave (start 0) first
    perm = np.lexsort((np.arange(n), start))
    return idx[perm].astype(np.int32)


def plan_makespan(lens: np.ndarray, order: np.ndarray, slots: int,
                  cost: np.ndarray | None = None) -> float:
    """Simulated span of the dynamic claim (each free slot takes the next
    column of ``order``) under the cost model."""
    import heapq

    lens = np.asarray(lens, dtype=np.int64)
    w = column_cost(lens) if cost is None else np.asarray(cost, dtype=np.float64)
    heap = [0.0] * min(slots, len(order))
    heapq.heapify(heap)
    for j in order:
        heapq.heapreplace(heap, heap[0] + w[j])
    return max(heap) if heap else 0.0
