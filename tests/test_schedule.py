"""The persistent solve's claim order (swmd_schedule_order, host C) against its
numpy restatement (paper_2107_06433_b200/schedule.py).  CPU only: the planner
is host code in libswmd.so."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2107_06433_b200 import _lib, schedule, synth


def _c_order(col_ptr, slots, reg_rounds=2, slab_rows=48, max_ratio=8):
    cp = np.ascontiguousarray(col_ptr, dtype=np.int64)
    out = np.empty(cp.size - 1, dtype=np.int32)
    rc = _lib.lib().swmd_schedule_order(cp.ctypes.data, cp.size - 1, slots, reg_rounds,
                                        slab_rows, max_ratio, out.ctypes.data)
    assert rc == 0
    return out


@pytest.mark.parametrize("name,n_docs,slots", [
    ("c2", None, 2368), ("c2", 3000, 2368), ("c2", 9000, 1776), ("c1", None, 100),
    ("c5", 4000, 1184), ("c1", 1500, 296)])
def test_c_planner_matches_restatement(name, n_docs, slots):
    cp = synth.zipf_instance(name, n_docs=n_docs).col_ptr
    got = _c_order(cp, slots)
    want = schedule.balanced_order(np.diff(cp), slots)
    assert np.array_equal(got, want)
    assert np.array_equal(np.sort(got), np.arange(cp.size - 1))   # a permutation


def test_planned_span_not_worse_than_longest_first():
    cp = synth.zipf_instance("c2").col_ptr
    lens = np.diff(cp)
    for slots in (1776, 2368, 2960):
        plan = schedule.plan_makespan(lens, _c_order(cp, slots), slots)
        lpt = schedule.plan_makespan(lens, schedule.longest_first(lens), slots)
        lb = schedule.column_cost(lens).sum() / slots
        assert lb <= plan <= lpt + 1e-12


@pytest.mark.parametrize("lens,slots", [
    ([], 4), ([5], 4), ([3, 1, 2], 4),          # every column in the first wave
    (list(range(1, 200)), 3),                   # > max_ratio columns per slot
    ([7] * 50 + [0] * 10, 20)])                 # ties and empty columns
def test_fallbacks_and_edges(lens, slots):
    cp = np.concatenate([[0], np.cumsum(np.asarray(lens, dtype=np.int64))]).astype(np.int64)
    got = _c_order(cp, slots)
    want = schedule.balanced_order(np.asarray(lens, dtype=np.int64), slots)
    assert np.array_equal(got, want)
    if len(lens) <= slots or len(lens) > 8 * slots:
        assert np.array_equal(got, schedule.longest_first(np.asarray(lens)))


def test_bad_arguments():
    cp = np.array([0, 1], dtype=np.int64)
    out = np.empty(1, dtype=np.int32)
    assert _lib.lib().swmd_schedule_order(cp.ctypes.data, 1, 4, 0, 48, 8, out.ctypes.data) == _lib.EINVAL
    assert _lib.lib().swmd_schedule_order(None, 1, 4, 2, 48, 8, out.ctypes.data) == _lib.EINVAL
