#!/usr/bin/env python3
"""Throughput benchmark: train seeds/s of the GraphSAGE products-shaped config.

Workload (BASELINE.json configs[1], "C2"): synthetic ogbn-products-shaped graph
(2.4M vertices, ~64.6M CSR entries incl. self-loops, 100-dim fp32 features,
47 classes), 3-layer mean-GraphSAGE, fanouts [15, 10, 5] (bottom first),
hidden 64, batch 1024, SGD.  A step is one training batch: k-hop sampling ->
fused gather/aggregate -> dense transforms -> softmax-CE -> backward -> SGD.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Our arm (default): ``value`` is measured with every step's inputs already in
HBM (device-to-device staging + one CUDA-graph replay per step); ``e2e`` is the
same metric through the public per-step API (Trainer.train_step) from HOST
seed ids: pinned H2D of the step's inputs and a D2H read of the step's loss
inside the timed region.  Multi-GPU (torchrun): weak scaling, 1024 seeds per
rank per step, one NCCL gradient all-reduce per step inside the graph.

``--impl reference`` times the reference's CPU implementation of the same
path: the oracle port (oracle/, a restatement of the reference's numba/numpy
code pinned to its golden vectors) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

UNIT = "seeds/s"
#: --workload: the driver's line is c2 (BASELINE configs[1], the metric's own config);
#: c3 (configs[2], GCN on the Reddit shape, 602-dim rows) is the wide-row line
WORKLOADS = {
    "c2": dict(metric="train seeds/sec (GraphSAGE products-shape)",
               config=dict(workload="c2-products-shape",
                           graph="synthetic Chung-Lu zipf2.5 (datagen.make_dataset('c2'))", vertices=2_400_000,
                           feat_dim=100, classes=47, model="sage", layers=3, fanouts=[15, 10, 5], hidden=64,
                           batch_size=1024, optimizer="sgd", lr=0.01, hot_ratio=0.0)),
    "c3": dict(metric="train seeds/sec (GCN Reddit-shape)",
               config=dict(workload="c3-reddit-shape",
                           graph="synthetic Chung-Lu zipf2.5 (datagen.make_dataset('c3'))", vertices=233_000,
                           feat_dim=602, classes=41, model="gcn", layers=2, fanouts=[10, 25], hidden=256,
                           batch_size=1024, optimizer="sgd", lr=0.01, hot_ratio=0.0)),
}
METRIC = WORKLOADS["c2"]["metric"]
WORKLOAD = WORKLOADS["c2"]["config"]
CACHE = os.environ.get("HG_BENCH_CACHE", "/tmp/hg_bench_cache")


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# the CPU reference path (oracle port of the reference's per-batch pipeline)
# ---------------------------------------------------------------------------
def cpu_reference_steps(ds, batches, seeds_rng, budget_s, max_steps, warmup=1, wl=None):
    """Time the reference's per-batch path on the host (orchestrator.py:236-256 +
    sampler.sample_khop): oracle sample_khop (C restatement of the numba draw
    + numpy dedup/lexsort) -> float64 gather -> forward/backward (numpy/OpenBLAS)
    -> SGD.  Returns (seeds_per_s, steps_timed, seconds)."""
    from oracle import oracle as O
    g = O.Graph(offsets=ds.offsets, targets=ds.targets.astype(np.int64))
    feats64 = ds.features.astype(np.float64)
    data = O.VertexData(features=feats64, labels=ds.labels, train_mask=ds.train_mask, val_mask=ds.val_mask,
                        test_mask=ds.test_mask)
    wl = wl or WORKLOAD
    cfg = dict(O.DEFAULT_CFG, model=wl["model"], layers=wl["layers"], fanouts=tuple(wl["fanouts"]),
               hidden_dim=wl["hidden"], batch_size=wl["batch_size"], lr=wl["lr"], strategy="case1", hot_ratio=0.0)
    dims = [ds.feat_dim] + [wl["hidden"]] * (wl["layers"] - 1) + [int(ds.labels.max()) + 1]
    W = O.init_params(wl["model"], dims, 0)
    adam = O.Adam()
    n_seeds = 0
    t_total = 0.0
    steps = 0
    for i, seeds in enumerate(batches):
        t0 = time.perf_counter()
        st = O.sample_khop(g, seeds, cfg["fanouts"], seeds_rng[i])
        O.train_batch(cfg, data, W, st, ds.labels[seeds], None, adam)
        dt = time.perf_counter() - t0
        if i < warmup:
            continue
        t_total += dt
        n_seeds += seeds.shape[0]
        steps += 1
        if t_total >= budget_s or steps >= max_steps:
            break
    return n_seeds / t_total, steps, t_total


def host_cores():
    return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def epoch_batches(ds, n_needed, bs=1024, seed=0, rank=0, world=1, strong=False):
    """Full batches from successive epoch shuffles (runplan semantics) with their
    batch rng seeds (batch b of epoch e: batch_sample_seed(seed, e, b)).  Weak
    scaling: rank r takes the epoch's batches b with b % world == r.  Strong
    scaling: every rank walks the same global batches and takes its contiguous
    shard (parallel.shard) of each."""
    from paper_2311_13225_b200 import runplan
    train = ds.train_ids()
    out, seeds = [], []
    epoch = 0
    while len(out) < n_needed:
        order = runplan.shuffle_epoch(train, seed, epoch)
        batches = runplan.split_batches(order, bs)
        for b, x in enumerate(batches):
            if x.shape[0] != bs:
                continue
            if strong:
                from paper_2311_13225_b200.parallel import shard
                x = shard(x, world, rank)
            elif (b % world) != rank:
                continue
            out.append(x)
            seeds.append(runplan.batch_sample_seed(seed, epoch, b))
            if len(out) >= n_needed:
                break
        epoch += 1
    return out, seeds


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_2311_13225_b200.datagen import make_dataset
    wl = WORKLOADS[args.workload]
    ds = make_dataset(args.workload, cache_dir=CACHE)
    batches, rs = epoch_batches(ds, args.warmup + args.steps)
    budget = float(os.environ.get("HG_REF_BUDGET_S", "120"))
    # every host core for the reference's BLAS (torchrun exports OMP_NUM_THREADS=1 to each rank)
    try:
        from threadpoolctl import threadpool_limits
        limits = threadpool_limits(limits=host_cores())
    except Exception:
        limits = None
    v, steps, secs = cpu_reference_steps(ds, batches, rs, budget, args.steps, warmup=args.warmup, wl=wl["config"])
    if limits is not None:
        limits.restore_original_limits()
    line = {"metric": wl["metric"], "value": v, "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * secs / max(steps, 1), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": dict(wl["config"], parallelism="host-cpu", l2_flush="inputs > L2 (feature table)"),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": host_cores(), "kind": "port",
                             "sample": f"{steps} batches of 1024 seeds (requested {args.steps}, capped at "
                                       f"{budget:.0f}s of CPU work) after {args.warmup} warm-up; {cpu_model()}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--phases", action="store_true", help="also report a per-phase time breakdown")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: 1024 seeds per rank per step (global 1024*N); strong: a fixed global batch of "
                         "1024 split into N contiguous shards (the parity form, SURVEY §8(e))")
    ap.add_argument("--epoch-mode", default=None, metavar="SPEC",
                    help="extra measurement (not the driver's line): whole epochs through Trainer.run_epoch, "
                         "SPEC = 'c2:sage:hot=0.2:n=4' or 'c3:gcn:hot=0.2:n=4:fan=4,4:bs=10000'")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.epoch_mode:
        run_epoch_mode(args.epoch_mode)
        return

    import torch
    from paper_2311_13225_b200 import _lib
    from paper_2311_13225_b200.datagen import make_dataset
    from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer

    dist_ctx = None
    if world > 1 or os.environ.get("HG_FORCE_DIST"):  # HG_FORCE_DIST: exercise the NCCL path at N=1
        torch.cuda.set_device(_env_int("LOCAL_RANK", 0))
        from paper_2311_13225_b200.parallel import DistContext
        dist_ctx = DistContext("nccl")
        import torch.distributed as dist
        t = torch.ones(1, device="cuda")
        dist.all_reduce(t)  # NCCL warm-up outside capture
    dev = torch.device("cuda", torch.cuda.current_device())
    wl = WORKLOADS[args.workload]
    WL = wl["config"]
    ds = make_dataset(args.workload, cache_dir=CACHE)
    # report_transfers=False: the per-batch CSV bookkeeping (needed-row counting) is
    # not part of training and no report is written here
    cfg = TrainConfig(model=WL["model"], layers=WL["layers"], fanouts=tuple(WL["fanouts"]), hidden_dim=WL["hidden"],
                      batch_size=WL["batch_size"], lr=WL["lr"], strategy="case1", hot_ratio=0.0, use_graph=True,
                      seed=0, report_transfers=False)
    tr = Trainer(ds, cfg, dist=dist_ctx)
    e = tr.engine
    # instrumented copies of every set's graphs, split so CUDA events bracket the
    # dominant kernel (bottom fused gather+aggregate): it runs at the end of the
    # SAMPLE half (early_agg0: no weights involved, overlaps the previous batch's
    # training), else at the start of the train half
    early = e.early_agg0()
    parts = [e.capture_segments(split_at=("sample_agg0",) if early else ("fwd0_gemm",), set_index=k)
             for k in range(len(e.sets))]
    for ssegs, segs in parts:
        if early:
            assert [n for n, _ in ssegs] == ["start", "sample_agg0"], [n for n, _ in ssegs]
        else:
            assert [n for n, _ in segs] == ["start", "fwd0_gemm"], [n for n, _ in segs]
    K, W = args.steps, args.warmup
    strong = args.scaling == "strong"
    batches, rseeds = epoch_batches(ds, W + K, rank=rank, world=world, strong=strong)
    n_loc = int(batches[0].shape[0])  # seeds per rank per step (every shard of 1024 has the same size
    if strong and any(b.shape[0] != n_loc for b in batches):  # when world divides 1024)
        raise SystemExit("strong scaling needs equal shards (world must divide 1024)")
    if dist_ctx:
        dist_ctx.set_global_batch(1024 if strong else 1024 * world)
    # stage every step's inputs in HBM (value = device-resident inputs)
    d_seeds = torch.as_tensor(np.stack(batches).astype(np.int32), device=dev)
    bp = np.zeros((W + K, 8), dtype=np.int64)
    for i in range(W + K):
        bp[i, 0] = np.array([rseeds[i] & 0xFFFFFFFFFFFFFFFF], np.uint64).view(np.int64)[0]
        bp[i, 1], bp[i, 2], bp[i, 3], bp[i, 4] = n_loc, i, 0, -1
    d_bp = torch.as_tensor(bp, device=dev)
    n_div = 1024 if strong else 1024 * world
    d_counts = torch.tensor([n_loc, n_div], dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    from paper_2311_13225_b200.engine import stream_priorities
    ps, pt = stream_priorities()
    ss, st = torch.cuda.Stream(device=dev, priority=ps), torch.cuda.Stream(device=dev, priority=pt)
    nset = len(e.sets)
    sampled = [torch.cuda.Event() for _ in range(nset)]
    trained = [None] * nset
    ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_b = [torch.cuda.Event(enable_timing=True) for _ in range(K)]

    def sample(i, timed_idx=None, split=False):
        k = i % nset
        if trained[k] is not None:
            ss.wait_event(trained[k])
        with torch.cuda.stream(ss):
            s = e.sets[k]
            s.seeds[:n_loc].copy_(d_seeds[i], non_blocking=True)
            s.bp.copy_(d_bp[i], non_blocking=True)
            s.counts_in.copy_(d_counts, non_blocking=True)
            if split and early:  # instrumented: events bracket the bottom aggregation segment
                ssegs = parts[k][0]
                ssegs[0][1].replay()
                if timed_idx is not None:
                    ev_a[timed_idx].record(ss)
                ssegs[1][1].replay()
                if timed_idx is not None:
                    ev_b[timed_idx].record(ss)
            else:
                e.g_sample[k].replay()
            sampled[k].record(ss)

    def train(i, timed_idx=None, split=False):
        k = i % nset
        st.wait_event(sampled[k])
        with torch.cuda.stream(st):
            if split and not early:  # instrumented: CUDA events bracket the dominant kernel's graph segment
                segs = parts[k][1]
                if timed_idx is not None:
                    ev_a[timed_idx].record(st)
                segs[0][1].replay()
                if timed_idx is not None:
                    ev_b[timed_idx].record(st)
                segs[1][1].replay()
            else:
                e.g_train[k].replay()
            ev = torch.cuda.Event()
            ev.record(st)
            trained[k] = ev

    def run(lo, hi, timed=False, split=False):
        """Software pipeline: sample batch i+1 (stream ss) while batch i trains (st).
        The instrumented (split) pass runs the halves back to back instead, so
        the events bracket the dominant kernel without the other stream's work
        contending with it."""
        ss.wait_stream(stream)
        st.wait_stream(stream)
        if split:
            for i in range(lo, hi):
                if i > lo:
                    ss.wait_event(trained[(i - 1) % nset])
                sample(i, (i - lo) if timed else None, split)
                train(i, (i - lo) if timed else None, split)
        else:
            sample(lo, 0 if timed else None, split)
            for i in range(lo, hi):
                if i + 1 < hi:
                    sample(i + 1, (i + 1 - lo) if timed else None, split)
                train(i, (i - lo) if timed else None, split)
        stream.wait_stream(ss)
        stream.wait_stream(st)

    run(0, W)
    run(0, W, split=True)
    torch.cuda.synchronize()
    if dist_ctx:
        dist_ctx.barrier()
    clocks = ClockSampler(_env_int("LOCAL_RANK", 0))
    clocks.start()
    time.sleep(0.3)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t_start.record(stream)
    run(W, W + K)  # headline: one sample graph + one train graph per step
    t_end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    # instrumented pass over the same steps (train graph split around the
    # dominant kernel, CUDA events on its stream): the roofline's kernel time
    i_start = torch.cuda.Event(enable_timing=True)
    i_end = torch.cuda.Event(enable_timing=True)
    i_start.record(stream)
    run(W, W + K, timed=True, split=True)
    i_end.record(stream)
    torch.cuda.synchronize()
    if dist_ctx:
        dist_ctx.barrier()
    ms = t_start.elapsed_time(t_end)
    if dist_ctx:
        ms = dist_ctx.max_over_ranks(ms)
    global_batch = 1024 if strong else 1024 * world
    value = global_batch * K / (ms / 1000.0)
    agg_ms = float(np.mean([a.elapsed_time(b) for a, b in zip(ev_a, ev_b)]))
    # algorithmic bytes of the dominant kernel per launch:
    # unique src rows read + edge ids + per-dst metadata + [self | mean] rows written
    F = ds.feat_dim
    sizes = []
    e.cur = 0
    for i in range(min(K, 16)):
        e.seeds[:n_loc].copy_(d_seeds[W + i])
        e.bp.copy_(d_bp[W + i])
        e.counts_in.copy_(d_counts)
        e.enqueue_sample()  # full dedup of every layer (the step itself skips it for SAGE's bottom block)
        torch.cuda.synchronize()
        n_dst0 = int(e.samplers[1].n_src.item())
        n_src0 = int(e.samplers[0].n_src.item())
        E0 = int(e.samplers[0].counts[:n_dst0].sum().item())
        sizes.append((n_dst0, n_src0, E0))
    n_dst0, n_src0, E0 = (float(np.mean([s[j] for s in sizes])) for j in range(3))
    # SURVEY §8(d) "aggregate fwd" formula: unique source rows read (src prefix = dst) +
    # the mean rows written, (n_src + n_dst) * F * 4, + edge ids (4 + 4) + offsets
    alg_bytes = (n_src0 + n_dst0) * F * 4 + E0 * 8 + (n_dst0 + 1) * 8
    self_copy_bytes = n_dst0 * F * 4  # SAGE self rows written for the GEMM (implementation choice)
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = alg_bytes / (agg_ms / 1000.0) / 1e9
    # DRAM bytes per launch of the same kernel, this workload, from the committed ncu --set full capture
    traffic, kernel_name = None, "k_agg_fwd (bottom fused gather + aggregation)"
    try:
        rec = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())[args.workload]
        traffic, kernel_name = float(rec["traffic_bytes_per_launch"]), rec["kernel"]
    except Exception:
        pass
    # kernels per step (graph kernel nodes) -> launches in the timed region
    lib = _lib.load()
    per_step = 0
    sample_graphs = [g for _, g in parts[0][0]] if isinstance(parts[0][0], list) else [parts[0][0]]
    for g in sample_graphs + [g for _, g in parts[0][1]]:
        try:
            per_step += int(lib.hg_graph_kernel_count(g.raw_cuda_graph()))
        except Exception:
            per_step = -1
            break
    # ---- e2e through the public API from host seed ids ----
    e2e_K = K
    torch.cuda.synchronize()
    e2e_start = torch.cuda.Event(enable_timing=True)
    e2e_end = torch.cuda.Event(enable_timing=True)
    host_batches = [np.asarray(b, np.int64) for b in batches]
    [h() for h in tr.train_batches([(host_batches[i], rseeds[i]) for i in range(3)])]
    torch.cuda.synchronize()
    if dist_ctx:
        dist_ctx.barrier()
    wall0 = time.perf_counter()
    e2e_start.record(stream)
    handles = tr.train_batches([(host_batches[W + k], rseeds[W + k]) for k in range(e2e_K)])
    enq = time.perf_counter() - wall0
    losses = [h() for h in handles]
    e2e_end.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    e2e_event_ms = e2e_start.elapsed_time(e2e_end)
    e2e_ms = max(e2e_event_ms, wall * 1000.0)
    if dist_ctx:
        e2e_ms = dist_ctx.max_over_ranks(e2e_ms)
    e2e_value = global_batch * e2e_K / (e2e_ms / 1000.0)
    if not np.all(np.isfinite(losses)):
        raise SystemExit("non-finite loss in bench")
    phases = None
    if args.phases and rank == 0:
        phases = phase_breakdown(e, d_seeds, d_bp, d_counts, W)
    if rank != 0:
        if dist_ctx:
            dist_ctx.close()
        return
    cpu_base = None
    if not args.no_cpu_baseline and world == 1:
        budget = float(os.environ.get("HG_CPU_BASELINE_S", "20"))
        cb, steps, secs = cpu_reference_steps(ds, batches, rseeds, budget, 200, warmup=1, wl=WL)
        cpu_base = {"value": cb, "unit": UNIT, "cores": host_cores(), "kind": "port",
                    "sample": f"{steps} {args.workload.upper()} batches of 1024 seeds ({secs:.1f}s CPU) after 1 warm-up; oracle port of "
                              f"the reference path (C draw loop single-threaded, numpy/OpenBLAS on all cores); "
                              f"{cpu_model()}"}
    line = {"metric": wl["metric"], "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "ms_per_step_instrumented_serial": i_start.elapsed_time(i_end) / K,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "fp32", "data": "synthetic",
            "config": dict(WL, parallelism=f"dp{world}" if world > 1 else "single",
                           l2_flush=f"inputs > L2: {ds.num_vertices * ds.feat_dim * 4 / 1e9:.2f} GB feature table "
                                    f"+ {ds.num_edges * 4 / 1e9:.2f} GB CSR, random rows per step",
                           global_batch=global_batch, seeds_per_rank=n_loc),
            "roofline": {"bound": "hbm", "kernel": kernel_name,
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": "profiles/ncu_traffic.json",
                         "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": agg_ms,
                         "alg_bytes_formula": "SURVEY §8(d): (n_src0 + n_dst0)*F*4 + E0*8 + (n_dst0+1)*8",
                         "extra_bytes_self_rows": self_copy_bytes,
                         "kernel_timing": "CUDA events on the kernel's stream over a second pass of the same steps "
                                          "with the sample and train halves back to back (the headline pass "
                                          "overlaps them)",
                         "frac_vs_spec_8tbs": achieved / 8000.0,
                         "block0": {"n_dst": n_dst0, "n_src": n_src0, "edges": E0},
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"},
            "cpu_baseline": cpu_base,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": tr.feeder.h2d_bytes,
                    "d2h_bytes_per_step": tr.d2h_bytes_per_step,
                    "ms_per_step_device_events": e2e_event_ms / e2e_K, "ms_per_step_host_wall": wall * 1000.0 / e2e_K,
                    "ms_per_step_host_enqueue": enq * 1000.0 / e2e_K},
            "gpu_launches": per_step * K if per_step >= 0 else None,
            "kernels_per_step": per_step,
            "clocks": clk,
            "final_loss": losses[-1]}
    if args.workload == "c2":  # measured for C2's 400-byte rows
        line["roofline"]["random_row_ceiling"] = {
            "gbs_of_row_data": 4000.0,
            "source": "profiles/r01_gather_ceiling.txt (738K uniformly random 400-byte rows, no compute: "
                      "72.6-75.8 us); cost per 128-B line touched: profiles/r02s_gather_rowsize.txt; this "
                      "block's own fetch list as a pure gather: 55-61 us, profiles/r02_order_probe.txt"}
    if phases:
        line["phases_ms"] = phases
    print(json.dumps(line), flush=True)
    if dist_ctx:
        dist_ctx.close()


def run_epoch_mode(spec: str):
    """Whole training epochs (hot-embedding schedule included: queue replay,
    producer stream, store lookups/injection) through Trainer.run_epoch; reports
    seeds/s of the timed epoch, reuse statistics and full-graph accuracy."""
    import torch
    from paper_2311_13225_b200.datagen import make_dataset
    from paper_2311_13225_b200.orchestrator import TrainConfig, Trainer, evaluate
    parts = spec.split(":")
    opts = dict(p.split("=", 1) for p in parts[2:] if "=" in p)
    name, model = parts[0], parts[1]
    fan = tuple(int(x) for x in opts.get("fan", "15,10,5").split(","))
    hot = float(opts.get("hot", 0.0))
    cfg = TrainConfig(model=model, layers=len(fan), fanouts=fan, hidden_dim=int(opts.get("hidden", 64 if name != "c3" else 256)),
                      batch_size=int(opts.get("bs", 1024)), lr=float(opts.get("lr", 0.01)),
                      strategy="layer-based" if hot > 0 else "case1", hot_ratio=hot,
                      super_batch_n=int(opts.get("n", 4)), presample_rounds=int(opts.get("rounds", 2)),
                      execution=opts.get("exec", "pipelined"), seed=0, epochs=int(opts.get("epochs", 2)),
                      use_graph=bool(int(opts.get("graph", 1))))
    ds = make_dataset(name, cache_dir=CACHE)
    if "limit" in opts:  # training mask cut to its first `limit` vertices (bounded epochs on the full graph)
        from paper_2311_13225_b200.datagen import limit_train
        ds = limit_train(ds, int(opts["limit"]))
    t0 = time.perf_counter()
    tr = Trainer(ds, cfg)
    setup_s = time.perf_counter() - t0
    res = []
    first = 0
    for epoch in range(int(opts.get("epochs", 2))):
        plan = tr.build_epoch_plan(epoch, first)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        ev0.record()
        rep = tr.run_epoch(plan)
        ev1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        n_seeds = sum(b.shape[0] for b in plan.batches)
        res.append({"epoch": epoch, "batches": len(plan.batches), "seeds_per_s": n_seeds / wall,
                    "gpu_ms": ev0.elapsed_time(ev1), "wall_s": wall, "reuse_hits": rep.reuse_hits,
                    "fallbacks": rep.fallbacks, "max_gap": rep.max_gap, "first_loss": rep.losses[0],
                    "last_loss": rep.losses[-1]})
        first += len(plan.batches)
    acc = evaluate(tr)
    cpu = None
    if int(opts.get("cpu", 0)):  # the reference path on the host cores beside it (the oracle port, fp64)
        from oracle import oracle as O
        og = O.Graph(offsets=ds.offsets, targets=ds.targets.astype(np.int64))
        od = O.VertexData(features=ds.features.astype(np.float64), labels=ds.labels, train_mask=ds.train_mask,
                          val_mask=ds.val_mask, test_mask=ds.test_mask)
        kw = {k: v for k, v in cfg.to_dict().items() if k in O.DEFAULT_CFG}
        w0 = time.perf_counter()
        reps, weights, _ = O.run_training(og, od, kw, evaluate_each_epoch=False)
        cpu_s = time.perf_counter() - w0
        accs, _ = O.evaluate(og, od, cfg.model, weights)
        n_all = sum(len(r["losses"]) for r in reps) * cfg.batch_size
        cpu = {"seconds": cpu_s, "cores": host_cores(), "kind": "port",
               "seeds_per_s_incl_presampling": n_all / cpu_s, "val_accuracy": accs["val"],
               "test_accuracy": accs["test"], "max_gap": [r.get("max_gap", 0) for r in reps],
               "reuse_hits": [sum(x["reuse_hits"] for x in r["rows"]) for r in reps],
               "last_loss": reps[-1]["losses"][-1]}
    print(json.dumps({"mode": "epoch", "spec": spec, "config": cfg.to_dict(), "vertices": ds.num_vertices,
                      "edges": ds.num_edges, "hot_list": int(tr.hot_list.shape[0]), "setup_s": setup_s,
                      "epochs": res, "val_accuracy": acc["val"], "test_accuracy": acc["test"],
                      "cpu_reference": cpu}), flush=True)


def phase_breakdown(e, d_seeds, d_bp, d_counts, i0, reps=20):
    """Per-phase device time (ms) of one step run SEQUENTIALLY (sample half, then
    the train half split at every mark; no cross-batch overlap)."""
    import torch
    early = e.early_agg0()
    marks = tuple(m for m in e.MARKS if e.hot is not None or m != "fwd0_agg")  # no empty segments
    if early:  # the bottom aggregation closes the sample half; the train half starts at its GEMM
        marks = tuple(m for m in marks if m != "fwd0_gemm") + ("sample_agg0",)
    marks = marks + tuple(f"sample_l{l}" for l in range(e.L - 1))  # per-layer sampling
    gs, segs = e.capture_segments(split_at=marks)
    sample_segs = [("sample", gs)] if not isinstance(gs, list) else \
        [(f"sample_l{e.L - 1}" if n == "start" else "bottom_agg" if n == "sample_agg0" else n, g) for n, g in gs]
    segs = sample_segs + [(("train_start" if n == "start" else n), g) for n, g in segs]
    tot = {n: 0.0 for n, _ in segs}
    e.cur = 0
    for r in range(reps):
        e.seeds[:d_seeds.shape[1]].copy_(d_seeds[i0 + r % d_seeds.shape[0]])
        e.bp.copy_(d_bp[i0 + r % d_bp.shape[0]])
        e.counts_in.copy_(d_counts)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(segs) + 1)]
        evs[0].record()
        for k, (_, g) in enumerate(segs):
            g.replay()
            evs[k + 1].record()
        torch.cuda.synchronize()
        for k, (n, _) in enumerate(segs):
            tot[n] += evs[k].elapsed_time(evs[k + 1])
    return {n: v / reps for n, v in tot.items()}


if __name__ == "__main__":
    main()
