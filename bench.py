"""Benchmark of the B200 Sinkhorn-WMD hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

A step is one full query solve — cost/kernel build, max_iter fused
iterations, final pass — over the configured synthetic corpus
(paper_2107_06433_b200.synth; seeded stand-ins for the paper's datasets).
At N=1 the workload is BASELINE.json configs[1] ("c2": V=100k, N=5k docs,
v_r=19, fp64, lam=10, 15 iterations).  With --gpus N>1 (torchrun, NCCL) the
corpus grows to N x 5k documents and is column-sharded, one block per rank
("scaling": "weak"); the distances are all-gathered every step, on a
communication stream that overlaps step k's gather with step k+1's compute
(double-buffered; the last step's gather is counted in full).

Metric: nnz*iterations/s of the whole solve (higher is better); docs/s beside it.
  value  device-resident inputs, CUDA events on the solver stream, L2 flushed
         (256 MiB scratch written, then read back) before every step, max over ranks;
  e2e    the public API sinkhorn_wmd(query ndarray, corpus, E, config) per step:
         query selection on the host, H2D of (sel, r), kernels, D2H of the
         distances + error record; corpus and E resident (uploaded once).

--impl reference times the reference algorithm on the host cores (the
oracle/ C port of sinkwmd's numba kernels, deterministic column-block mode,
all hardware threads) on the same config; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "Sinkhorn-WMD nnz*iters/s per query (docs/s beside it)"
UNIT = "nnz*iters/s"


def _peaks() -> dict:
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled (every 20 ms, one
    nvidia-smi process in loop mode) during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        """Launch the sampler and return once it is producing samples; the
        window opens at return (the caller enters its timed region next)."""
        self.lines = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self
        self.reader = threading.Thread(target=self._read, daemon=True)
        self.reader.start()
        deadline = time.perf_counter() + 5.0
        while not self.lines and time.perf_counter() < deadline:
            time.sleep(0.005)
        self.t0 = time.perf_counter()
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append((time.perf_counter(), ln))

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        t1 = time.perf_counter()
        deadline = t1 + 1.0          # the first sample after the window closes still counts
        while time.perf_counter() < deadline and not any(ts >= t1 for ts, _ in self.lines):
            time.sleep(0.005)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=10)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.reader.join(timeout=2)
        after = [ts for ts, _ in self.lines if ts >= t1]
        t_last = after[0] if after else t1
        out = "".join(ln for ts, ln in self.lines if self.t0 <= ts <= t_last)
        samples = [[v.strip() for v in ln.split(",")] for ln in out.splitlines() if ln.strip()]
        samples = [x for x in samples if len(x) >= 7]
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        num = lambda v: float(v) if v.replace(".", "").isdigit() else None  # noqa: E731
        sm = [num(x[0]) for x in samples if num(x[0]) is not None]
        mx = [num(x[1]) for x in samples if num(x[1]) is not None]
        busy = [num(x[0]) for x in samples if num(x[6]) and num(x[6]) > 0 and num(x[0])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for x in samples for k in range(4)
                          if x[2 + k].lower() == "active"})
        med = statistics.median(busy) if busy else (statistics.median(sm) if sm else None)
        return {"sm_mhz": med, "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(samples), "samples_busy": len(busy)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _config(name: str, world: int):
    from paper_2107_06433_b200 import synth

    cfg = synth.CONFIGS[name]
    n_docs = cfg.n_docs * world if name in ("c1", "c2") else cfg.n_docs
    scaling = "weak" if name in ("c1", "c2") else "strong"
    return cfg, n_docs, scaling


def _workload_json(cfg, n_docs, nnz, world, scaling, flush: bool):
    return {
        "workload": f"{cfg.name}: V={cfg.n_vocab} N={n_docs} docs ({cfg.k_min}-{cfg.k_max} "
                    f"Zipf({cfg.zipf_s}) words each), v_r={cfg.v_r}, w={cfg.dim}, "
                    f"lam={cfg.lam}, max_iter={cfg.max_iter}, seed={cfg.seed}",
        "nnz": int(nnz),
        "n_docs": int(n_docs),
        "parallelism": f"column shards x{world}" if world > 1 else "1 GPU",
        "scaling_mode": scaling,
        "l2": ("flushed before every step: 256 MiB scratch written then read back "
               "(L2 holds no solver data and no dirty lines)") if flush else "warm",
    }


# ---------------------------------------------------------------------------------------------

def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    import oracle
    from paper_2107_06433_b200 import synth

    cfg, n_docs, scaling = _config(args.config, world)
    inst = synth.zipf_instance(cfg, n_docs=n_docs)
    cores = os.cpu_count() or 1
    oracle.set_threads(cores)
    E64 = np.ascontiguousarray(inst.embeddings, dtype=np.float64)
    qpos = [0]

    def run():
        # c4: one query of the batch per step (the reference solves a batch one
        # query at a time, in fp64); other configs: the single query
        q = inst.queries[qpos[0] % len(inst.queries)]
        qpos[0] += 1
        return oracle.solve(q, inst.col_ptr, inst.rows, inst.vals, E64, lam=cfg.lam,
                            max_iter=cfg.max_iter, blocks=cores)
    for _ in range(args.warmup):
        run()
    times = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    wall = time.perf_counter() - t_all
    ms = 1e3 * wall / args.steps
    value = inst.nnz * cfg.max_iter * args.steps / wall
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded Zipf corpus, Gaussian embeddings)",
        "config": _workload_json(cfg, n_docs, inst.nnz, world, scaling, False),
        "docs_per_s": n_docs * args.steps / wall,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"full {cfg.name} solve x{args.steps} (oracle/swmd_oracle.c, "
                                   f"deterministic column blocks, {cores} OpenMP threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def _cpu_baseline(inst, cfg) -> dict:
    """Rank 0, N=1: the oracle port on the host cores over a bounded sample."""
    import oracle

    cores = os.cpu_count() or 1
    oracle.set_threads(cores)
    oracle.solve(inst.query, inst.col_ptr, inst.rows, inst.vals, inst.embeddings,
                 lam=cfg.lam, max_iter=cfg.max_iter, blocks=cores)
    reps, t_total = 0, 0.0
    while reps < 20 and t_total < 8.0:
        t0 = time.perf_counter()
        oracle.solve(inst.query, inst.col_ptr, inst.rows, inst.vals, inst.embeddings,
                     lam=cfg.lam, max_iter=cfg.max_iter, blocks=cores)
        t_total += time.perf_counter() - t0
        reps += 1
    return {"value": inst.nnz * cfg.max_iter * reps / t_total, "unit": UNIT, "cores": cores,
            "kind": "port",
            "sample": f"{reps} full {cfg.name} solves, {t_total:.2f}s (oracle/swmd_oracle.c, "
                      f"{cores} OpenMP threads, deterministic column blocks)"}


def _transpose_times(inst, dev) -> dict:
    """A row-major corpus made resident: CSR upload + device transpose
    (DeviceCorpus.from_csr) beside the reference's host argsort transpose
    (CsrMatrix.csc_index, sparse.py:98-120).  Not part of the step."""
    import torch

    from paper_2107_06433_b200 import synth
    from paper_2107_06433_b200.device import DeviceCorpus
    from paper_2107_06433_b200.sparse import CsrMatrix

    rp, ci, v = synth.csc_to_csr(inst.n_vocab, inst.n_docs, inst.col_ptr, inst.rows, inst.vals)
    for _ in range(2):
        DeviceCorpus.from_csr(inst.n_vocab, inst.n_docs, rp, ci, v, dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    DeviceCorpus.from_csr(inst.n_vocab, inst.n_docs, rp, ci, v, dev)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    CsrMatrix(inst.n_vocab, inst.n_docs, rp, ci, v).csc_index()
    t_host = time.perf_counter() - t0
    return {"device_ms": 1e3 * t_dev, "host_argsort_ms": 1e3 * t_host, "nnz": int(inst.nnz),
            "note": "device = pageable CSR upload + swmd_csr_to_csc_f64 + col_ptr readback"}


def _cold_e2e(inst, scfg) -> dict:
    """The first public sinkhorn_wmd() call on a corpus object and an embedding
    array the library has never seen (resident and cold timings
    reported separately): CSC upload + claim-order plan, E upload (pageable),
    row norms, E_c compaction, native plan creation and graph capture, then
    the solve.  Wall clock; a second call on the same objects is the warm
    figure.  Not part of the step."""
    import torch

    import paper_2107_06433_b200 as swmd

    corpus = inst.corpus()                 # a new CsrMatrix: nothing cached on it
    E = inst.embeddings.copy()             # a new array: no resident copy keyed to it
    E.flags.writeable = False
    ws = swmd.SinkhornWorkspace()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    swmd.sinkhorn_wmd(inst.query, corpus, E, scfg, workspace=ws)
    cold = time.perf_counter() - t0
    t0 = time.perf_counter()
    swmd.sinkhorn_wmd(inst.query, corpus, E, scfg, workspace=ws)
    warm = time.perf_counter() - t0
    return {"cold_ms": 1e3 * cold, "warm_ms": 1e3 * warm,
            "h2d_bytes_cold": int(E.nbytes + corpus.nnz * 12 + (corpus.n_cols + 1) * 8),
            "note": "first call on a fresh corpus object and embedding array (uploads, "
                    "compaction, plan + CUDA-graph capture, solve) vs the next call"}


def _fusion_compare(sel, weights, dc, de, scfg, flush_buf, reps: int) -> dict:
    """Fused persistent solve vs the unfused comparator (SDDMM -> w in HBM ->
    SpMM per iteration; baseline.unfused_sparse_wmd, reference baseline.py:
    67-131, timed against the fused solver in reference bench.py:49-89) on the
    same resident K: the iteration + final phases only, CUDA events, L2
    flushed before each solve.  The unfused launches are replayed from a CUDA
    graph so host launch overhead does not count against it."""
    import torch

    from paper_2107_06433_b200 import _lib
    from paper_2107_06433_b200.baseline import UnfusedPlan
    from paper_2107_06433_b200.solver import QueryPlan, SinkhornWorkspace

    side = torch.cuda.Stream(device=dc.device)
    out = {}
    with torch.cuda.stream(side):
        s = side.cuda_stream
        fused = QueryPlan(sel, weights, dc, de, scfg, SinkhornWorkspace())
        unf = UnfusedPlan(sel, weights, dc, de, scfg, SinkhornWorkspace())
        fused.enqueue_distances()
        unf.enqueue_distances()
        fused.enqueue_solve()
        unf.enqueue_solve()
        side.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            unf.enqueue_solve()
        graph.replay()
        side.synchronize()
        a = fused.wmd.cpu().numpy()
        b = unf.wmd.cpu().numpy()
        out["max_rel_diff"] = float(np.max(np.abs(a - b) / np.maximum(np.abs(a), 1e-300)))
        times = {"fused": [], "unfused": []}
        for _ in range(reps):
            for name in ("fused", "unfused"):
                _lib.call("swmd_l2_flush", flush_buf.data_ptr(), flush_buf.numel(), s)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(side)
                if name == "fused":
                    fused.enqueue_solve()
                else:
                    graph.replay()
                e1.record(side)
                times[name].append((e0, e1))
        side.synchronize()
    f_ms = float(np.median([x.elapsed_time(y) for x, y in times["fused"]]))
    u_ms = float(np.median([x.elapsed_time(y) for x, y in times["unfused"]]))
    it = scfg.max_iter
    out.update({
        "fused_solve_ms": f_ms, "unfused_solve_ms": u_ms, "fusion_speedup": u_ms / f_ms,
        "fused_launches_per_solve": 1, "unfused_launches_per_solve": 2 * it + 1,
        "unfused_w_bytes_per_iter": int(2 * 8 * dc.nnz),
        "reps": reps,
        "note": "iterations + final pass on resident K (cost build excluded, same for both); "
                "unfused = swmd_unfused_iterate_f64 (SDDMM storing w, SpMM reading it) per "
                "iteration + swmd_unfused_final_f64, graph-replayed; medians, L2 flushed "
                "before each solve; the paper reports 1.15-2.22x on CPUs",
    })
    return out


def _c3_strong(args, world: int, rank: int, dev, flush_buf) -> dict | None:
    """The north-star scaling workload (BASELINE configs[2], "c3": N=1M docs,
    ~45M nnz) strong-scaled over the ``world`` ranks: column_blocks shards
    (reference sparse.py:261-276), K built on every rank, the solve writing
    into the rank's slot of ONE all_gather_into_tensor per step.  Device time
    per step = CUDA events around (cost build, solve, gather), max over ranks.
    With world > 1, rank 0 also times the whole c3 solve alone on its GPU, so
    the line carries the 1 -> N efficiency of this run.  Rank 0 gets the dict."""
    import torch
    import torch.distributed as dist

    import paper_2107_06433_b200 as swmd
    from paper_2107_06433_b200 import _lib, synth
    from paper_2107_06433_b200.distributed import _TAIL, DeviceShardSolver, shard_bounds
    from paper_2107_06433_b200.distributed import sinkhorn_wmd_sharded
    from paper_2107_06433_b200.solver import QueryPlan

    cfg = synth.CONFIGS["c3"]
    inst = synth.zipf_instance(cfg)
    inst.embeddings.flags.writeable = False
    corpus = inst.corpus()
    scfg = swmd.SolverConfig(lam=cfg.lam, max_iter=cfg.max_iter)
    sel, weights = swmd.select_nonzero(inst.query)
    bounds = shard_bounds(corpus, world)
    c0, c1 = int(bounds[rank]), int(bounds[rank + 1])
    width = int(np.max(np.diff(bounds)))
    solver = DeviceShardSolver(corpus, inst.embeddings, dev=dev)
    dc = solver.block(c0, c1)
    s = torch.cuda.current_stream(dev).cuda_stream
    slot = torch.zeros(width + _TAIL, dtype=torch.float64, device=dev)
    gathered = torch.empty(world * (width + _TAIL), dtype=torch.float64, device=dev)
    plan = QueryPlan(sel, weights, dc, solver.de, scfg, solver.ws)
    plan.wmd = slot[: c1 - c0]
    plan.err = slot[width: width + 4].view(torch.int64)

    def step(ev=None):
        if ev is not None:
            ev[0].record()
        plan.enqueue_distances()
        plan.enqueue_solve()
        if ev is not None:
            ev[1].record()
        if world > 1:
            dist.all_gather_into_tensor(gathered, slot)
        if ev is not None:
            ev[2].record()

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    steps = args.c3_steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(steps):
        _lib.call("swmd_l2_flush", flush_buf.data_ptr(), flush_buf.numel(), s)
        step(evs[k])
    torch.cuda.synchronize()
    tot = float(sum(e[0].elapsed_time(e[2]) for e in evs))
    comp = float(sum(e[0].elapsed_time(e[1]) for e in evs))
    gat = float(sum(e[1].elapsed_time(e[2]) for e in evs))
    t = torch.tensor([tot, comp, gat], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot, comp, gat = (float(v) for v in t.cpu())

    # e2e through the public sharded API (query in, all N distances out on every rank)
    for _ in range(2):
        res = sinkhorn_wmd_sharded(inst.query, corpus, inst.embeddings, scfg, solver=solver) \
            if world > 1 else swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, scfg,
                                                workspace=solver.ws)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        res = sinkhorn_wmd_sharded(inst.query, corpus, inst.embeddings, scfg, solver=solver) \
            if world > 1 else swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, scfg,
                                                workspace=solver.ws)
    e2e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e.item())

    one_ms = None
    if world > 1:
        dist.barrier()
        if rank == 0:   # the same workload on this GPU alone
            full = DeviceShardSolver(corpus, inst.embeddings, dev=dev)
            dfull = full.block(0, corpus.n_cols)
            p1 = QueryPlan(sel, weights, dfull, full.de, scfg, full.ws)
            for _ in range(2):
                p1.enqueue_distances()
                p1.enqueue_solve()
            torch.cuda.synchronize()
            ev1 = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
            for k in range(steps):
                _lib.call("swmd_l2_flush", flush_buf.data_ptr(), flush_buf.numel(), s)
                ev1[k][0].record()
                p1.enqueue_distances()
                p1.enqueue_solve()
                ev1[k][1].record()
            torch.cuda.synchronize()
            one_ms = float(np.mean([a.elapsed_time(b) for a, b in ev1]))
            ok = np.array_equal(p1.wmd.cpu().numpy(), res.wmd)
            assert ok, "c3 sharded result differs from the single-GPU solve"
            del p1, full, dfull
        dist.barrier()
    if rank != 0:
        return None
    ms = tot / steps
    out = {
        "workload": f"c3: V={cfg.n_vocab} N={inst.n_docs} docs, nnz={inst.nnz}, v_r={sel.size}, "
                    f"lam={cfg.lam}, max_iter={cfg.max_iter}; column_blocks over {world} rank(s)",
        "n_gpus": world, "steps": steps,
        "ms_per_step": ms, "compute_ms": comp / steps, "gather_ms": gat / steps,
        "value": inst.nnz * cfg.max_iter / (ms / 1e3), "unit": UNIT,
        "e2e": {"ms_per_step": 1e3 * e2e_s / steps,
                "value": inst.nnz * cfg.max_iter * steps / e2e_s, "unit": UNIT,
                "note": "public sinkhorn_wmd_sharded() (N>1) / sinkhorn_wmd() (N=1), "
                        "corpus and E resident; max over ranks"},
        "shard_nnz_max": int(np.max(np.diff(corpus.csc_compact()[0][bounds]))),
        "l2": "flushed before every step",
        "note": "device time per step = max over ranks of (cost build + solve + "
                "all_gather_into_tensor of the distance slots)",
    }
    if one_ms is not None:
        out["one_gpu_ms_per_step"] = one_ms
        out["efficiency"] = one_ms / (world * ms)
    return out


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2107_06433_b200 as swmd
    from paper_2107_06433_b200 import _lib, synth
    from paper_2107_06433_b200.device import DeviceCorpus, DeviceEmbeddings, stream_ptr
    from paper_2107_06433_b200.distributed import DeviceShardSolver, shard_bounds, sinkhorn_wmd_sharded
    from paper_2107_06433_b200.solver import QueryPlan, SinkhornWorkspace

    world, rank, local = _dist_env()
    # SWMD_BENCH_BACKEND=gloo is a functional check of the N > 1 code path on a
    # box with fewer GPUs (ranks share devices; their timings mean nothing)
    backend = os.environ.get("SWMD_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # NCCL's own init log (rank count, transport, NVLS) on stderr, so the
        # communicator the run used can be checked next to the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cfg, n_docs, scaling = _config(args.config, world)
    inst = synth.zipf_instance(cfg, n_docs=n_docs)
    # a serving table is immutable: read-only, so the resident copy is keyed by
    # identity (a writeable table is re-hashed in full on every call, device.py)
    inst.embeddings.flags.writeable = False
    corpus = inst.corpus()
    scfg = swmd.SolverConfig(lam=cfg.lam, max_iter=cfg.max_iter)
    sel, weights = swmd.select_nonzero(inst.query)
    bounds = shard_bounds(corpus, world)
    c0, c1 = int(bounds[rank]), int(bounds[rank + 1])
    solver = DeviceShardSolver(corpus, inst.embeddings, dev=dev)
    solver(sel, weights, c0, c1, scfg, None)              # upload the block, build the plan
    dc = solver._blocks[(c0, c1)]
    de = DeviceEmbeddings.of(inst.embeddings, dev)
    ws = solver.ws
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    s = stream_ptr(dev)
    width = int(np.max(np.diff(bounds)))
    # N > 1: the solve writes straight into its slot of the gather buffer; the
    # all-gather of step k runs on a communication stream while step k+1
    # computes (double-buffered), so only the last step's gather is exposed
    gather_in = [torch.zeros(width, dtype=torch.float64, device=dev) for _ in range(2)]
    gather_out = [torch.zeros(width * world, dtype=torch.float64, device=dev) for _ in range(2)]
    comm = torch.cuda.Stream(device=dev) if world > 1 else None
    gathered = [None, None]   # event: the gather that last read gather_in[b] is done

    def device_step(plan, k, ev=None):
        b = k % 2
        if ev is not None:
            ev[0].record()
        plan.enqueue_distances()
        if ev is not None:
            ev[1].record()
        if world > 1:
            if gathered[b] is not None:
                torch.cuda.current_stream(dev).wait_event(gathered[b])
            plan.wmd = gather_in[b][: c1 - c0]
        plan.enqueue_solve()
        if ev is not None:
            ev[2].record()
        if world > 1:
            done = torch.cuda.Event()
            done.record()
            comm.wait_event(done)
            with torch.cuda.stream(comm):
                dist.all_gather_into_tensor(gather_out[b], gather_in[b])
                g = torch.cuda.Event()
                g.record()
            gathered[b] = g
        if ev is not None:
            ev[3].record()

    plan = QueryPlan(sel, weights, dc, de, scfg, ws)
    for k in range(max(args.warmup, 3)):
        device_step(plan, k)
    torch.cuda.synchronize()

    clocks = ClockSampler(local).start() if rank == 0 else None
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    plan.launches = 0
    for k in range(args.steps):
        if args.flush:
            _lib.call("swmd_l2_flush", flush_buf.data_ptr(), flush_buf.numel(), s)
        device_step(plan, k, evs[k])
    ev_end = torch.cuda.Event(enable_timing=True)
    if world > 1:   # the last step's gather is not hidden behind anything: count it
        torch.cuda.current_stream(dev).wait_event(gathered[(args.steps - 1) % 2])
    ev_end.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clock_info = clocks.stop() if clocks else None
    step_ms = [e[0].elapsed_time(e[2]) for e in evs]     # cost build + solve
    cost_ms = [e[0].elapsed_time(e[1]) for e in evs]
    solve_ms = [e[1].elapsed_time(e[2]) for e in evs]
    launches = plan.launches
    tot_ms = float(np.sum(step_ms)) + evs[-1][2].elapsed_time(ev_end)
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    # the plan's result must still be right: check the last step against a fresh solve
    wmd_dev = plan.wmd.clone()
    exposed_gather_ms = evs[-1][2].elapsed_time(ev_end)

    # e2e through the public API (corpus, E resident; query in, distances out)
    for _ in range(2):
        if world > 1:
            sinkhorn_wmd_sharded(inst.query, corpus, inst.embeddings, scfg, solver=solver)
        else:
            swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, scfg, workspace=ws)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if world > 1:
            res = sinkhorn_wmd_sharded(inst.query, corpus, inst.embeddings, scfg, solver=solver)
        else:
            res = swmd.sinkhorn_wmd(inst.query, corpus, inst.embeddings, scfg, workspace=ws)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_sparse_ms = None
    if world == 1:
        # the query as a SparseVector histogram (the reference's ingest output,
        # ingest.py:175-197): the native runtime takes its ids and weights directly
        from paper_2107_06433_b200.sparse import SparseVector

        sidx = np.flatnonzero(inst.query > 0)
        sv = SparseVector(inst.query.size, sidx, inst.query[sidx])
        for _ in range(2):
            swmd.sinkhorn_wmd(sv, corpus, inst.embeddings, scfg, workspace=ws)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            rs = swmd.sinkhorn_wmd(sv, corpus, inst.embeddings, scfg, workspace=ws)
        e2e_sparse_ms = 1e3 * (time.perf_counter() - t0) / args.steps
        assert np.array_equal(rs.wmd, res.wmd), "SparseVector query differs from the dense query"
    assert np.array_equal(res.wmd[c0:c1], wmd_dev.cpu().numpy()), "device-timed result drifted"
    cold = _cold_e2e(inst, scfg) if world == 1 else None   # before the c3 block's allocations
    c3_block = None
    if args.c3 and args.config == "c2":
        c3_block = _c3_strong(args, world, rank, dev, flush_buf)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    nnz_all = inst.nnz
    iters = cfg.max_iter
    value = nnz_all * iters * args.steps / (tot_ms / 1e3)
    ms_step = tot_ms / args.steps
    peaks = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    # algorithmic bytes of the two kernels
    v_r = int(sel.size)
    rows_built = dc.n_present if dc.n_present < dc.n_rows else dc.n_rows
    cost_bytes = rows_built * (cfg.dim * 8 + 8) + 2 * rows_built * v_r * 8
    nnz_loc = dc.nnz
    # the survey's canonical per-iteration HBM figure (x round trip counted; "effective"
    # for the persistent kernel, which keeps x on chip)
    it_bytes = nnz_loc * 12 + 2 * dc.n_cols * v_r * 8 + 4 * (dc.n_cols + 1)
    fin_bytes = nnz_loc * 12 + dc.n_cols * v_r * 8 + dc.n_cols * 8 + 4 * (dc.n_cols + 1)
    solve_bytes = iters * it_bytes + fin_bytes
    c_ms, s_ms = float(np.mean(cost_ms)), float(np.mean(solve_ms))
    gather_l2 = nnz_loc * v_r * 8 * (iters + 2)          # K-row gathers (+KM in the final)
    flops = iters * (4 * nnz_loc * v_r + 2 * nnz_loc + dc.n_cols * v_r) + 6 * nnz_loc * v_r
    dominant = "solve" if s_ms >= c_ms else "cost"
    ncu = {}
    # the committed --set full capture of this config's dominant kernel, if there is one
    ncu_src = f"profiles/r02_ncu_{args.config}.json"
    try:
        with open(os.path.join(REPO, ncu_src)) as f:
            ncu = json.load(f)["kernels"]
    except (OSError, KeyError, ValueError):
        pass
    if dominant != "solve":
        kname = "cost_tmap_kernel"
    else:
        kname = "reg_solve" if v_r <= 32 else "cta2_solve"
    traffic = None
    if kname in ncu and args.config in ("c2", "c3", "c5") and world == 1:
        traffic = ncu[kname]["dram_read_bytes"] + ncu[kname]["dram_write_bytes"]
    if dominant == "solve":
        achieved = solve_bytes / (s_ms / 1e3) / 1e9
    else:
        achieved = cost_bytes / (c_ms / 1e3) / 1e9
    # the solve against every roofline the survey names (§8d): HBM (canonical,
    # effective), the K-row gather against the measured L2 gather peak, FP64
    probes = {}
    for pf in ("r01_probes.json", "r02_probes.json"):
        try:
            with open(os.path.join(REPO, "profiles", pf)) as f:
                probes.update(json.load(f))
        except (OSError, ValueError):
            pass
    # the L2 gather peak for this workload's K-row size: 160-byte rows (v_r <= 20)
    # saturate at ~9.1 TB/s, 2 KB rows at 18.9 TB/s (profiles/r02_probes.json)
    row_bytes = 8 * (((v_r + 3) // 4) * 4 if v_r <= 32 else v_r + (v_r & 1))
    l2_2kb = float(probes.get("l2_gather_2kb_rows_tbs", 18.9)) * 1e3
    l2_peak = (float(probes.get("l2_gather_160b_rows_tbs", 9.1)) * 1e3 if row_bytes <= 256
               else l2_2kb)
    fp64_peak = float(probes.get("fp64_dmma_tflops", 36.9)) * 1e3
    t_hbm = solve_bytes / hbm / 1e3               # us at peak
    t_l2 = gather_l2 / l2_peak / 1e3
    t_fp64 = flops / fp64_peak / 1e3
    bind = max((t_hbm, "hbm"), (t_l2, "l2_gather"), (t_fp64, "fp64"))
    binding = {
        "resource": bind[1], "t_hbm_us": t_hbm, "t_l2_us": t_l2, "t_fp64_us": t_fp64,
        "solve_us": 1e3 * s_ms, "frac": bind[0] / (1e3 * s_ms),
        "k_row_bytes": row_bytes,
        "t_l2_at_2kb_row_peak_us": gather_l2 / l2_2kb / 1e3,
        "frac_at_2kb_row_peak": gather_l2 / l2_2kb / 1e3 / (1e3 * s_ms),
        "peaks": {"hbm_gbs": hbm, "l2_gather_gbs": l2_peak, "l2_gather_2kb_rows_gbs": l2_2kb,
                  "fp64_gflops": fp64_peak},
        "note": "binding roofline = max(T_HBM, T_L2, T_FP64) for the per-pass formulation of SURVEY "
                "§8d (every pass gathers every nonzero's K row); T_L2 uses the L2 gather peak "
                "measured for this K-row size (scripts/l2_probe.cu: 160-byte rows saturate at "
                "~9.1 TB/s, 2 KB rows at 18.9 TB/s; profiles/r02_probes.json, raw logs in "
                "profiles/r02_probe_logs/). The persistent solve keeps each column's K rows in "
                "registers / shared memory across its passes, so it performs almost none of these "
                "gathers (ncu L2 throughput ~8 %): frac > 1 means it beats the per-pass-gather "
                "bound, and the kernel is latency-bound (profiles/r02_summary.md). "
                "frac_at_2kb_row_peak is the round-1 figure (2 KB-row peak)",
    }
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Zipf corpus, Gaussian embeddings; paper datasets absent)",
        "config": _workload_json(cfg, n_docs, nnz_all, world, scaling, args.flush),
        "docs_per_s": n_docs * args.steps / (tot_ms / 1e3),
        "roofline": {
            "bound": "hbm", "kernel": "swmd_solve_f64 (persistent fused loop)" if dominant == "solve"
            else "swmd_cost_build_f64",
            "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "when" in peaks else "fallback",
            "traffic": traffic,
            "traffic_source": f"{ncu_src} (ncu --set full, dram read+write bytes per launch)"
            if traffic is not None else None,
            "bytes_per_launch": solve_bytes if dominant == "solve" else cost_bytes,
            "note": ("solve bytes = survey §8d B_HBM per iteration x iterations + final "
                     "(x round trip counted although the persistent kernel keeps x on chip: "
                     "an effective figure); the solve's working set is L2/on-chip resident, "
                     "so its binding roofline is the L2 K-row gather: see "
                     "solve_binding_roofline") if dominant == "solve" else
                    "cost bytes = E rows of words present in the corpus + K, K*M writes",
        },
        "solve_binding_roofline": binding,
        "kernels": {
            "exposed_gather_ms": exposed_gather_ms if world > 1 else 0.0,
            "cost_build_ms": c_ms, "cost_build_gbs": cost_bytes / (c_ms / 1e3) / 1e9,
            "solve_ms": s_ms, "solve_eff_hbm_gbs": solve_bytes / (s_ms / 1e3) / 1e9,
            "solve_gather_gbs": gather_l2 / (s_ms / 1e3) / 1e9,
            "solve_fp64_gflops": flops / (s_ms / 1e3) / 1e9,
            "rows_built": int(rows_built),
        },
        "e2e": {"value": nnz_all * iters * args.steps / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": int(2 * v_r * 8),
                "d2h_bytes_per_step": int((dc.n_cols + _lib.ERR_WORDS) * 8),
                "ms_per_step": 1e3 * e2e_s / args.steps,
                "sparse_query_ms_per_step": e2e_sparse_ms,
                "note": "public sinkhorn_wmd() with the dense numpy query (sparse_query_ms_per_step: "
                        "the same call with a SparseVector query, the reference's ingest format); "
                        "corpus and embeddings resident in HBM"},
        "gpu_launches": int(launches),
        "clocks": clock_info,
    }
    if cold is not None:
        line["e2e"]["cold"] = cold
    if c3_block is not None:
        line["c3_strong"] = c3_block
    if world == 1:
        line["corpus_transpose"] = _transpose_times(inst, dev)
        if not args.no_fusion and int(sel.size) <= 64:
            line["fusion"] = _fusion_compare(sel, weights, dc, de, scfg, flush_buf,
                                             reps=50 if args.config in ("c1", "c2") else 5)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = _cpu_baseline(inst, cfg)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_batch_f32(args):
    """c4: 64 queries per step through the batched fp32 path (rank 0 / 1 GPU)."""
    import torch

    import paper_2107_06433_b200 as swmd
    from paper_2107_06433_b200 import batch as batch_mod
    from paper_2107_06433_b200 import synth

    world, rank, local = _dist_env()
    if rank != 0:
        return 0
    torch.cuda.set_device(local)
    cfg = synth.CONFIGS["c4"]
    inst = synth.zipf_instance(cfg)
    corpus = inst.corpus()
    scfg = swmd.SolverConfig(lam=cfg.lam, max_iter=cfg.max_iter, precision="f32")
    ws = swmd.SinkhornWorkspace()
    Q = len(inst.queries)
    for _ in range(args.warmup):
        swmd.sinkhorn_wmd_batch(inst.queries, corpus, inst.embeddings, scfg, workspace=ws)
    torch.cuda.synchronize()
    clocks = ClockSampler(local).start()
    dev_s, wall, cost_s, solve_s = 0.0, 0.0, 0.0, 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = swmd.sinkhorn_wmd_batch(inst.queries, corpus, inst.embeddings, scfg, workspace=ws)
        wall += time.perf_counter() - t0
        bad = [r for r in res if isinstance(r, Exception)]
        if bad:
            raise bad[0]
        dev_s += sum(r.timings["distances"] + r.timings["iterations"] for r in res)
        cost_s += sum(r.timings["distances"] for r in res)
        solve_s += sum(r.timings["iterations"] for r in res)
    clock_info = clocks.stop()
    work = inst.nnz * cfg.max_iter * Q * args.steps
    sum_vr = sum(int(np.count_nonzero(q)) for q in inst.queries)
    # SURVEY §8(d) canonical per-iteration figures for Q queries (F = 4 bytes)
    nnz, N, T = inst.nnz, inst.n_docs, cfg.max_iter
    b_hbm = nnz * (4 + 4) + 2 * N * sum_vr * 4 + 4 * (N + 1)
    b_l2 = nnz * sum_vr * 4
    flops = 4 * nnz * sum_vr + 2 * nnz * Q + N * sum_vr
    solve_ms = 1e3 * solve_s / args.steps
    cost_ms = 1e3 * cost_s / args.steps
    fp32_peak = 148 * 128 * 2 * 1.965e3          # GFLOP/s: FFMA lanes x 2 x max SM clock
    probes = {}
    for pf in ("r01_probes.json", "r02_probes.json"):
        try:
            with open(os.path.join(REPO, "profiles", pf)) as f:
                probes.update(json.load(f))
        except (OSError, ValueError):
            pass
    fp32_peak = float(probes.get("fp32_ffma_tflops", fp32_peak / 1e3)) * 1e3
    solve_flops = (T + 1) * flops
    achieved = solve_flops / (solve_ms / 1e3) / 1e9
    t_l2 = (T + 2) * b_l2 / (float(probes.get("l2_gather_2kb_rows_tbs", 18.9)) * 1e12) * 1e3
    t_fp = solve_flops / (fp32_peak * 1e9) * 1e3
    t_hbm = (T + 1) * b_hbm / (float(_peaks().get("hbm_gbs", 6650.0)) * 1e9) * 1e3
    line = {
        "metric": METRIC, "value": work / dev_s, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Zipf corpus, Gaussian fp32 embeddings; paper datasets absent)",
        "config": {"workload": f"c4: {Q} queries (v_r 8-64, sum {sum_vr}) x V=100000 x N=100000 "
                               f"docs, fp32, lam=10, max_iter=20, batched per step",
                   "nnz": int(inst.nnz), "n_docs": int(inst.n_docs), "queries": Q,
                   "l2": "not flushed (K for the batch is 0.9 GB > L2)"},
        "docs_per_s": inst.n_docs * Q * args.steps / dev_s,
        "e2e": {"value": work / wall, "unit": UNIT, "h2d_bytes_per_step": int(sum_vr * 20),
                "d2h_bytes_per_step": int(Q * (inst.n_docs * 4 + 32)),
                "ms_per_step": 1e3 * wall / args.steps,
                "note": "public sinkhorn_wmd_batch(precision='f32'); corpus, E resident"},
        "gpu_launches": int(batch_mod.last_launches * args.steps),
        "clocks": clock_info,
        "kernels": {"cost_build_ms": cost_ms, "solves_ms": solve_ms,
                    "cost_build": "gram32_tc5_kernel: tcgen05.mma kind::tf32 x 3 (3xTF32), TMEM "
                                  "accumulator, one launch for the batch (SWMD_GRAM32=ffma|mma: the "
                                  "FFMA / mma.sync kernels)",
                    "solve": "reg_solve_mq<float>: one persistent launch per group of up to 4 "
                             "queries of one padded width, each claimed column solved for every "
                             "query of the group (CSC read once per group)",
                    "solve_launches_per_batch": int(batch_mod.last_launches - 2)},
        "roofline": {
            "bound": "fp32", "kernel": "swmd_solve_f32 (persistent fused loop, all queries)",
            "achieved": achieved, "peak": fp32_peak, "unit": "GFLOP/s", "frac": achieved / fp32_peak,
            "traffic": None,
            "note": "SURVEY §8(d) FLOP per iteration for the batch (4 nnz sum(v_r) + 2 nnz Q + N sum(v_r)) "
                    "x (max_iter + 1) / device solve time; the binding resource of the sum-of-solves "
                    "is the larger of the three times in binding_ms",
            "binding_ms": {"fp32": t_fp, "l2_gather": t_l2, "hbm": t_hbm, "measured": solve_ms},
        },
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = _cpu_baseline_c4(inst, cfg)
    print(json.dumps(line), flush=True)
    return 0


def _cpu_baseline_c4(inst, cfg) -> dict:
    """The oracle (fp64, the reference's arithmetic) on a bounded sample of the
    batch's queries, all host cores."""
    import oracle

    cores = os.cpu_count() or 1
    oracle.set_threads(cores)
    E64 = np.ascontiguousarray(inst.embeddings, dtype=np.float64)
    reps, t_total = 0, 0.0
    while reps < len(inst.queries) and t_total < 10.0:
        t0 = time.perf_counter()
        oracle.solve(inst.queries[reps], inst.col_ptr, inst.rows, inst.vals, E64, lam=cfg.lam,
                     max_iter=cfg.max_iter, blocks=cores)
        t_total += time.perf_counter() - t0
        reps += 1
    return {"value": inst.nnz * cfg.max_iter * reps / t_total, "unit": UNIT, "cores": cores,
            "kind": "port",
            "sample": f"{reps} of {len(inst.queries)} c4 queries solved in fp64, {t_total:.2f}s "
                      f"(oracle/swmd_oracle.c, {cores} OpenMP threads)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: 2000 for the B200 arm, 50 for the CPU reference arm)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-flush", dest="flush", action="store_false")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c3", dest="c3", action="store_false",
                    help="skip the c3 strong-scaling block of the c2 line")
    ap.add_argument("--c3-steps", type=int, default=10)
    ap.add_argument("--no-fusion", action="store_true",
                    help="skip the fused-vs-unfused comparison (1 GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.steps is None:
        args.steps = 50 if args.impl == "reference" else 2000
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c4":
        return run_batch_f32(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
