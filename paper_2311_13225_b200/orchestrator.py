"""End-to-end training driver (reference orchestrator.py:1-739) on one B200.

Keeps the reference's public surface — ``TrainConfig``, ``EpochReport``,
``run_training``, ``evaluate``, ``build_epoch_plan``, ``epsilon_monitor`` — and
its numerics contract: the same epoch shuffles, batches, batch/hot/queue
stream seeds, hot list, queues, producer versions (chunk j of super-batch g+1
pinned to version first+group[j]), double-buffered store with the 2n-1 gap
bound, injection of reused bottom-layer embeddings and epsilon trace.

What changes is where it runs: every batch is one replay of a captured CUDA
graph (engine.TrainEngine) and the hot-embedding producer runs on its own CUDA
stream gated by per-version events ("pipelined"), or inline on the training
stream ("serial"); both give bit-identical results.  The reference's
discrete-event device simulator (devsim/skeletons/presets) and its idle-time
feedback are out of scope: with no modelled CPU/GPU split the hot-set partition
keeps every queued vertex in the reuse set (hotness.partition_hot with zero
idle time, hotness.py:129), i.e. the reference with simulate_costs=False.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, dense, runplan
from .device import DeviceGraph, pad4, ptr, stream_ptr, u64_tensor
from .engine import STAGE_COUNTS, STAGE_SEEDS, BatchFeeder, HotBuffers, Pipeline, TrainEngine
from .gnnmath import init_params
from .hotness import estimate_hotness, select_hot
from .sampler import Fanouts, LayerSampler
from .store import FallbackBudgetExceeded, StalenessViolation

EXECUTIONS = ("serial", "pipelined")
STRATEGIES = ("case1", "case2", "case3", "case4", "layer-based")  # skeletons.STRATEGIES
#: the static feature cache budget of the cached-gather baselines case3/case4
#: (orchestrator.py:345-356): presets.paper_like_preset().cache_budget_bytes (presets.py:58)
STATIC_CACHE_BUDGET_BYTES = 2.0e5
REAL_SIZE = 8  # transfer.py accounting unit (8-byte reals)


class ConfigError(ValueError):
    """orchestrator.py:66-67."""


@dataclass
class TrainConfig:
    """orchestrator.py:74-146 (same fields and defaults)."""

    model: str = "gcn"
    layers: int = 3
    fanouts: tuple = (25, 10, 5)
    hidden_dim: int = 64
    batch_size: int = 1024
    super_batch_n: int = 4
    hot_ratio: float = 0.2
    strategy: str = "layer-based"
    lr: float = 0.1
    epochs: int = 1
    seed: int = 0
    optimizer: str = "sgd"
    presample_rounds: int = 20
    execution: str = "serial"
    stage_budget_frac: float = 1.0
    max_fallback_frac: float = 0.5
    # The reference's discrete-event cost simulator (devsim/presets, orchestrator.py:570-575,
    # 621-637) is out of scope: its only effect on training is the idle-time feedback that
    # moves hot vertices from "compute" to "feature cache".  Only simulate_costs=False
    # (the reference's numerics with zero idle time) is accepted; True or a preset raise
    # ConfigError instead of being silently ignored.
    simulate_costs: bool = False
    preset: object = None
    use_graph: bool = True  # replay each step as one captured CUDA graph
    report_transfers: bool = True  # per-batch needed-row accounting for the batch CSV (transfer.py:59-73)

    def validate(self) -> None:
        if self.model not in ("gcn", "sage"):
            raise ConfigError(f"model must be gcn or sage, got {self.model!r}")
        if self.layers != len(self.fanouts):
            raise ConfigError(f"layers ({self.layers}) must equal len(fanouts) ({len(self.fanouts)})")
        try:
            Fanouts(tuple(self.fanouts))
        except ValueError as exc:
            raise ConfigError(str(exc)) from exc
        if self.super_batch_n < 1:
            raise ConfigError(f"super-batch size must be >= 1, got {self.super_batch_n}")
        if self.batch_size < 1:
            raise ConfigError(f"batch size must be >= 1, got {self.batch_size}")
        if not (0.0 <= self.hot_ratio <= 1.0):
            raise ConfigError(f"hot ratio must be in [0, 1], got {self.hot_ratio}")
        if self.strategy not in STRATEGIES:
            raise ConfigError(f"strategy must be one of {STRATEGIES}, got {self.strategy!r}")
        if self.execution not in EXECUTIONS:
            raise ConfigError(f"execution must be one of {EXECUTIONS}, got {self.execution!r}")
        if self.optimizer not in ("sgd", "adam"):
            raise ConfigError(f"optimizer must be sgd or adam, got {self.optimizer!r}")
        if self.epochs < 1:
            raise ConfigError(f"epochs must be >= 1, got {self.epochs}")
        if not (0.0 < self.stage_budget_frac <= 1.0):
            raise ConfigError("stage budget fraction must be in (0, 1]")
        if self.simulate_costs:
            raise ConfigError("simulate_costs=True needs the reference's device simulator, which this "
                              "implementation does not provide (use simulate_costs=False)")
        if self.preset is not None:
            raise ConfigError("device presets belong to the reference's simulator and are not supported")

    def dims(self, feat_dim: int, num_classes: int) -> list:
        return [feat_dim] + [self.hidden_dim] * (self.layers - 1) + [num_classes]

    def to_dict(self) -> dict:
        return {"model": self.model, "layers": self.layers, "fanouts": list(self.fanouts),
                "hidden_dim": self.hidden_dim, "batch_size": self.batch_size,
                "super_batch_n": self.super_batch_n, "hot_ratio": self.hot_ratio, "strategy": self.strategy,
                "lr": self.lr, "epochs": self.epochs, "seed": self.seed, "optimizer": self.optimizer,
                "presample_rounds": self.presample_rounds, "execution": self.execution,
                "stage_budget_frac": self.stage_budget_frac, "max_fallback_frac": self.max_fallback_frac}


@dataclass
class EpochReport:
    """orchestrator.py:149-169 (simulator fields dropped)."""

    epoch: int
    losses: list = field(default_factory=list)
    batch_rows: list = field(default_factory=list)
    val_accuracy: float = 0.0
    test_accuracy: float = 0.0
    epsilon_trace: list = field(default_factory=list)
    max_weight_deltas: list = field(default_factory=list)
    max_gap: int = 0
    max_gap_batch: int = -1
    max_gap_super_batch: int = -1
    stage_seconds_measured: dict = field(default_factory=dict)
    stage_events: list = field(default_factory=list)  # (target_sb, version, count)
    warmup_computed: int = 0
    reuse_hits: int = 0
    fallbacks: int = 0


@dataclass
class EpochPlan:
    """orchestrator.py:172-181; queues live on the device, sizes on the host."""

    epoch: int
    batches: list
    groups: list
    batch_seeds: list
    first_global_batch: int
    queues: dict = field(default_factory=dict)       # g -> device int32 tensor
    queue_sizes: dict = field(default_factory=dict)  # g -> int
    hot_seeds: dict = field(default_factory=dict)    # g -> int


class HotProducer:
    """Bottom-layer embeddings for queued hot vertices (orchestrator.py:259-271,
    381-395): one-hop sample of the chunk with the super-batch's hot stream
    (sampler.sample_one_hop_hot), fused gather+aggregate, dense transform with
    the bottom weights of the pinned version, ReLU iff L > 1, then put into the
    staging table."""

    def __init__(self, engine: TrainEngine, cap_chunk: int, n_snaps: int):
        e = self.e = engine
        dev = e.device
        self.cap = max(int(cap_chunk), 1)
        # own first-occurrence table: the producer runs concurrently with the
        # training stream's samplers
        self.smp = LayerSampler(e.dg, self.cap, e.fan[0], need_nself=e.sage, need_outdeg=not e.sage,
                                minpos=e.dg.minpos.like())
        zf = lambda *s: torch.zeros(*s, dtype=torch.float32, device=dev)  # noqa: E731
        self.self_buf = zf(self.cap, e.ld[0]) if e.sage else None
        self.agg = zf(self.cap, e.ld[0])
        self.emb = zf(self.cap, e.ld[1])
        self.snaps = zf(max(n_snaps, 1), e.params.bottom_numel)
        self.img = dense.BImage(e.dims[0], e.dims[0] if e.sage else 0, e.dims[1], 1, dev)

    def snapshot(self, j: int):
        """_ParamCell.publish (orchestrator.py:281-284): copy W0 at this version."""
        self.snaps[j].copy_(self.e.params.flat[:self.e.params.bottom_numel])

    def run_chunk(self, ids: torch.Tensor, c: int, seed_dev: torch.Tensor, snap: int, version: int, stamp: int,
                  table: int, stream=None):
        e, hot = self.e, self.e.hot
        s = stream_ptr(stream)
        d0, d1 = e.dims[0], e.dims[1]
        # SAGE reads the chunk's neighbour rows by global id: draws only, no dedup
        self.smp.run(ids, None, seed_dev, 0, stream, cap_dst=c, dedup=not e.sage)
        model = 0 if e.sage else 1
        sp = e.dg.split_rows() if hasattr(e.dg, "split_rows") else None
        blk = (ptr(ids), None, c, e.fan[0], ptr(self.smp.counts), ptr(self.smp.slots), ptr(self.smp.slot_local),
               ptr(self.smp.nself), ptr(self.smp.outdeg), None, ptr(self.self_buf), e.ld[0], ptr(self.agg), e.ld[0], s)
        if sp is not None and sp["body_cols"] + sp["tail_cols"] == e.ld[0]:  # same split-row gather as the step
            _lib.call("hg_aggregate_fwd_split", model, ptr(sp["body"]), sp["body_cols"], ptr(sp["tail"]),
                      sp["tail_cols"], sp["body_cols"], e.ld[0], *blk)
        else:
            _lib.call("hg_aggregate_fwd", model, 1, ptr(e.dg.features), e.dg.feat_ld, e.ld[0], *blk)
        w = self.snaps[snap]
        act = 1 if e.L > 1 else 0
        self.img.prep(ptr(w), d1, s)
        if e.sage:
            dense.fwd(ptr(self.self_buf), e.ld[0], ptr(self.agg), e.ld[0], d0, ptr(w), d1, ptr(self.emb), e.ld[1],
                      None, c, act, s, img=self.img)
        else:
            dense.fwd(ptr(self.agg), e.ld[0], None, 0, d0, ptr(w), d1, ptr(self.emb), e.ld[1], None, c, act, s,
                      img=self.img)
        _lib.call("hg_store_put", ptr(ids), None, c, ptr(self.emb), e.ld[1], hot.H, ptr(hot.slot_of),
                  ptr(hot.tab[table]), ptr(hot.ver[table]), ptr(hot.stamp[table]), int(version), int(stamp),
                  ptr(hot.puts), s)


class Trainer:
    """State of one run_training call (orchestrator.py:183-196 _RunState)."""

    def __init__(self, ds, config: TrainConfig, device=None, hot_list=None, weights=None, dist=None):
        config.validate()
        self.cfg = config
        self.ds = ds
        given = ds if isinstance(ds, DeviceGraph) else getattr(ds, "device_graph", None)
        self.dg = given if given is not None else DeviceGraph.from_dataset(ds, device=device)
        if not hasattr(self.dg, "l2_window"):
            self.dg.persist_hot_rows()
        self.train_ids = np.nonzero(np.asarray(ds.train_mask))[0].astype(np.int64)
        self.fan = tuple(int(f) for f in config.fanouts)
        C = int(np.asarray(ds.labels).max()) + 1
        self.dims = config.dims(self.dg.feat_dim, C)
        self.dist = dist
        if weights is None:
            weights = init_params(config.model, self.dims, config.seed).weights
        self.layer_based = config.strategy == "layer-based"
        n_batches = (self.train_ids.shape[0] + config.batch_size - 1) // config.batch_size
        self.engine = TrainEngine(self.dg, config.model, self.dims, self.fan, config.batch_size, config.lr,
                                  optimizer=config.optimizer, weights=weights, max_batches=n_batches,
                                  allreduce=dist.allreduce if dist is not None else None)
        self.engine.account_rows = bool(config.report_transfers)
        self.static_cache = self._static_cache()
        if self.static_cache.size:
            flags = torch.zeros(self.dg.num_vertices, dtype=torch.uint8, device=self.dg.device)
            flags[torch.as_tensor(self.static_cache, device=self.dg.device)] = 1
            self.engine.static_cached = flags
        self.version = 0
        # ---- hot list (hotness.py:70-108 via orchestrator.py:692-702) ----
        if hot_list is None:
            hot_list = np.empty(0, np.int64)
            if self.layer_based and config.hot_ratio > 0 and config.layers > 1:
                table = estimate_hotness(self.dg, self.train_ids, Fanouts(self.fan), config.presample_rounds,
                                         config.seed, batch_size=config.batch_size, engine=self.engine)
                hot_list = select_hot(table, config.hot_ratio)
        self.hot_list = np.asarray(hot_list, np.int64)
        self.use_hot = self.layer_based and self.hot_list.size > 0 and config.layers > 1
        self.emb_dim = config.hidden_dim if config.layers > 1 else C
        dev = self.dg.device
        if self.layer_based:
            self.engine.hot = HotBuffers.create(self.dg.num_vertices, self.hot_list, self.emb_dim,
                                                config.super_batch_n, self.engine.cap_dst[0], max(n_batches, 1), dev)
        self.hot_dev = torch.as_tensor(self.hot_list.astype(np.int32), device=dev) if self.hot_list.size else None
        self.reach_tag = torch.full((self.dg.num_vertices,), -1, dtype=torch.int32, device=dev) \
            if self.use_hot else None
        self.producer = None
        self.tag_serial = 0
        self.stamp_serial = 0
        self.feeder = BatchFeeder(self.engine)
        self.pipeline = Pipeline(self.engine)
        self.prod_stream = torch.cuda.Stream(device=dev) if config.execution == "pipelined" else None
        self.batch_to_group = {}
        if config.use_graph:
            self.engine.capture()

    def _static_cache(self) -> np.ndarray:
        """The top-degree vertices of the case3/case4 static feature cache
        (orchestrator.py:345-356; accounting only: they only move rows from the
        batch CSV's raw_rows to cache_hit_rows)."""
        cfg = self.cfg
        if cfg.strategy not in ("case3", "case4"):
            return np.empty(0, np.int64)
        budget = STATIC_CACHE_BUDGET_BYTES
        if cfg.strategy == "case4":
            budget = max(0.0, budget - (self.dg.num_vertices + 1 + self.dg.num_edges) * 8.0)
        k = int(budget // (self.dg.feat_dim * REAL_SIZE))
        if k <= 0:
            return np.empty(0, np.int64)
        deg = np.diff(np.asarray(self.ds.offsets))
        return np.argsort(-deg, kind="stable")[:k].astype(np.int64)

    # ------------------------------------------------------------------
    def _new_tag(self):
        self.tag_serial += 1
        return self.tag_serial

    def build_epoch_plan(self, epoch: int, first_global_batch: int) -> EpochPlan:
        """orchestrator.py:200-229; the replay sampling and the hot-list filter run
        on the device; only the queue sizes come back to the host."""
        cfg, e = self.cfg, self.engine
        order = runplan.shuffle_epoch(self.train_ids, cfg.seed, epoch)
        batches = runplan.split_batches(order, cfg.batch_size)
        groups = runplan.super_batch_groups(len(batches), cfg.super_batch_n)
        seeds = [runplan.batch_sample_seed(cfg.seed, epoch, b) for b in range(len(batches))]
        plan = EpochPlan(epoch=epoch, batches=batches, groups=groups, batch_seeds=seeds,
                         first_global_batch=first_global_batch)
        if not self.use_hot:
            return plan
        dev = self.dg.device
        lib = _lib.load()
        n_hot = int(self.hot_list.shape[0])
        ws = torch.zeros(int(lib.hg_filter_ws_size(n_hot)), dtype=torch.int32, device=dev)
        counts = torch.zeros(len(groups), dtype=torch.int32, device=dev)
        for g in range(1, len(groups)):
            tag = self._new_tag()
            rs = runplan.queue_replay_seed(cfg.seed, epoch, g)
            for b in groups[g]:
                self.feeder.feed(batches[b], rs, 0, 0)
                # blocks L-1 .. 1 fix the bottom destinations (= layer-1 sources)
                e.enqueue_sample(layers=range(e.L - 1, 0, -1))
                fr0, n0 = e.frontier(0)
                _lib.call("hg_tag_vertices", ptr(fr0), ptr(n0), e.cap_dst[0], ptr(self.reach_tag), tag,
                          stream_ptr())
            q = torch.zeros(max(n_hot, 1), dtype=torch.int32, device=dev)
            _lib.call("hg_filter_tagged", ptr(self.hot_dev), n_hot, ptr(self.reach_tag), tag, ptr(q),
                      ptr(counts[g:g + 1]), ptr(ws), stream_ptr())
            plan.queues[g] = q
            plan.hot_seeds[g] = runplan.hot_sample_seed(cfg.seed, epoch, g)
        sizes = counts.cpu().numpy()
        for g in range(1, len(groups)):
            k = int(sizes[g])
            if cfg.stage_budget_frac < 1.0 and k:
                k = int(np.ceil(k * cfg.stage_budget_frac))
            plan.queue_sizes[g] = k
        return plan

    # ------------------------------------------------------------------
    def run_epoch(self, plan: EpochPlan) -> EpochReport:
        """orchestrator.py:330-618 (batch loop :456-545)."""
        cfg, e = self.cfg, self.engine
        hot = e.hot
        rep = EpochReport(epoch=plan.epoch)
        dev = self.dg.device
        t0 = time.perf_counter()
        nb = len(plan.batches)
        if hot is not None:
            hot.reset_counters()
        e.raw_rows_arr.zero_()
        e.cache_hit_arr.zero_()
        if self.use_hot and self.producer is None:
            cap = max([plan.queue_sizes.get(g, 0) for g in plan.queue_sizes] + [1])
            cap = (cap + cfg.super_batch_n - 1) // cfg.super_batch_n
            self.producer = HotProducer(e, max(cap, 1), cfg.super_batch_n)
        elif self.producer is not None:
            need = max([(plan.queue_sizes.get(g, 0) + cfg.super_batch_n - 1) // cfg.super_batch_n
                        for g in plan.queue_sizes] + [1])
            if need > self.producer.cap:
                self.producer = HotProducer(e, need, cfg.super_batch_n)
        hot_seed_dev = {g: u64_tensor(s, dev) for g, s in plan.hot_seeds.items()}
        main = torch.cuda.current_stream(dev)
        # store epoch reset (store.py:120-130): fresh stamps make old entries unreadable
        stamps = {}
        for g in range(len(plan.groups)):
            self.stamp_serial += 1
            stamps[g] = self.stamp_serial
        # flattened schedule: per batch its super-batch, store window parameters and
        # producer chunk (orchestrator.py:421-545)
        sched = []
        for g, group in enumerate(plan.groups):
            q_next_n = plan.queue_sizes.get(g + 1, 0) if self.use_hot else 0
            bounds = runplan.chunk_bounds(q_next_n, len(group)) if q_next_n else []
            cpu_tag = -1
            if self.use_hot and g > 0 and plan.queue_sizes.get(g, 0) > 0:
                cpu_tag = self._new_tag()
            for j, b in enumerate(group):
                gb = plan.first_global_batch + b
                self.batch_to_group[gb] = g
                chunk = bounds[j] if (bounds and bounds[j][1] > bounds[j][0]) else None
                sched.append(dict(g=g, j=j, b=b, gb=gb, cpu_tag=cpu_tag, first=j == 0, last=j == len(group) - 1,
                                  chunk=chunk, warm=1 if (self.layer_based and g == 0 and self.hot_list.size) else 0))
        pipe = self.pipeline
        state = {"prod_done": None}
        # data parallel: rank r trains the contiguous shard r of every
        # global batch; dlogits are scaled by 1/|global batch| so the all-reduced sum
        # is the union batch's gradient
        local = [self._local_seeds(bt) for bt in plan.batches]

        def feed_fn(it):
            seeds = local[it["b"]]
            n_div = int(plan.batches[it["b"]].shape[0]) if self.dist else None
            return lambda set_index: self.feeder.feed(
                seeds, plan.batch_seeds[it["b"]], it["gb"], it["b"], cpu_tag=it["cpu_tag"], table_sel=it["g"] % 2,
                cur_stamp=stamps[it["g"]], warm=it["warm"], n_div=n_div, set_index=set_index)

        def before_fn(it):
            def before(stream):
                g = it["g"]
                if it["first"]:
                    if it["cpu_tag"] >= 0:  # cpu_set of this super-batch (orchestrator.py:447-449)
                        _lib.call("hg_tag_vertices", ptr(plan.queues[g]), None, plan.queue_sizes[g],
                                  ptr(hot.cpu_tag_of), it["cpu_tag"], stream.cuda_stream)
                    if state["prod_done"] is not None:  # staging complete before use (:555-559)
                        stream.wait_event(state["prod_done"])
                        state["prod_done"] = None
                if it["chunk"] is not None:
                    lo, hi = it["chunk"]
                    c = hi - lo
                    self.producer.snapshot(it["j"])  # _ParamCell.publish: weights before this batch
                    args = (plan.queues[g + 1][lo:hi], c, hot_seed_dev[g + 1], it["j"], it["gb"], stamps[g + 1],
                            (g + 1) % 2)
                    if self.prod_stream is not None:
                        ev = torch.cuda.Event()
                        ev.record(stream)
                        self.prod_stream.wait_event(ev)
                        with torch.cuda.stream(self.prod_stream):
                            self.producer.run_chunk(*args, stream=self.prod_stream)
                    else:
                        self.producer.run_chunk(*args, stream=stream)
                    rep.stage_events.append((g + 1, it["gb"], c))
            return before

        # staleness (store.py:85-92): a violating lookup is never injected (the row is
        # computed from features) and is counted on the device; the count is copied to
        # pinned memory at every super-batch boundary and checked as soon as the copy
        # has landed (non-blocking), so a violation raises within a super-batch
        watch = []

        def poll(block=False):
            while watch and (block or watch[0][0].query()):
                ev, pin = watch.pop(0)
                ev.synchronize()
                if int(pin[0]):
                    pipe.drain()
                    torch.cuda.synchronize(dev)
                    raise StalenessViolation(f"{int(pin[0])} reuse events exceeded the 2n-1 version gap bound "
                                             f"{hot.gap_bound} (epoch {plan.epoch})")

        if sched:
            pipe.sample(0, feed_fn(sched[0]))
        for k, it in enumerate(sched):
            if k + 1 < len(sched):
                pipe.sample(k + 1, feed_fn(sched[k + 1]))
            pipe.train(k, before_fn(it))
            self.version += 1
            if it["last"] and self.prod_stream is not None and it["g"] + 1 in plan.queue_sizes \
                    and plan.queue_sizes.get(it["g"] + 1, 0) > 0:
                ev = torch.cuda.Event()
                ev.record(self.prod_stream)
                state["prod_done"] = ev
            if it["last"] and self.use_hot:
                pin = torch.zeros(1, dtype=torch.int64).pin_memory()
                with torch.cuda.stream(pipe.st):
                    pin.copy_(hot.stats[1:2], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(pipe.st)
                watch.append((ev, pin))
                poll()
        pipe.drain()
        if state["prod_done"] is not None:
            main.wait_event(state["prod_done"])
        torch.cuda.synchronize(dev)
        poll(block=True)
        e.check_numerics()
        rep.losses = e.loss_arr[:nb].double().cpu().tolist()
        if self.dist is not None:  # the union batch's mean loss from the per-shard means
            n_loc = torch.tensor([float(x.shape[0]) for x in local], dtype=torch.float64, device=dev)
            tot = e.loss_arr[:nb].double() * n_loc
            self.dist.allreduce(tot)
            rep.losses = (tot / torch.tensor([float(b.shape[0]) for b in plan.batches], dtype=torch.float64,
                                             device=dev)).cpu().tolist()
        if not np.all(np.isfinite(rep.losses)):
            raise FloatingPointError("non-finite training loss (forward aggregation or logits)")
        rep.max_weight_deltas = e.md_arr[:nb].double().cpu().tolist()
        hits = hot.batch_hits[:nb].cpu().numpy() if hot is not None else np.zeros(nb, np.int64)
        miss = hot.batch_miss[:nb].cpu().numpy() if hot is not None else np.zeros(nb, np.int64)
        raw_rows = e.raw_rows_arr[:nb].cpu().numpy()
        cache_rows = e.cache_hit_arr[:nb].cpu().numpy()
        feat_dim = self.dg.feat_dim
        # batch CSV transfer columns (orchestrator.py:505-543): raw features of the needed
        # rows; embeddings / aux move per super-batch, not per batch; the bottom weights'
        # gradient elements when the bottom layer is split off (layer-based, L > 1)
        grad_elems = (self.engine.params.bottom_numel if (self.layer_based and cfg.layers > 1) else 0)
        for g, group in enumerate(plan.groups):
            rep.epsilon_trace.append(max(rep.max_weight_deltas[b] for b in group) * 2 * cfg.super_batch_n)
            for b in group:
                rep.batch_rows.append({"epoch": plan.epoch, "batch": plan.first_global_batch + b, "super_batch": g,
                                       "loss": rep.losses[b], "reuse_hits": int(hits[b]), "fallbacks": int(miss[b]),
                                       "raw_rows": int(raw_rows[b]), "cache_hit_rows": int(cache_rows[b]),
                                       "raw_elems": int(raw_rows[b]) * feat_dim, "emb_elems": 0, "aux_elems": 0,
                                       "grad_elems": int(grad_elems), "max_weight_delta": rep.max_weight_deltas[b]})
        rep.reuse_hits, rep.fallbacks = int(hits.sum()), int(miss.sum())
        if hot is not None:
            rep.warmup_computed = int(hot.batch_warm[:nb].sum().item())
            stats = hot.stats.cpu().numpy().view(np.uint64)
            if int(stats[1]):
                raise StalenessViolation(f"{int(stats[1])} reuse events exceeded the 2n-1 gap bound")
            packed = int(stats[0])
            if packed:
                rep.max_gap = packed >> 32
                rep.max_gap_batch = 0xFFFFFFFF - (packed & 0xFFFFFFFF)
                rep.max_gap_super_batch = self.batch_to_group.get(rep.max_gap_batch, -1)
        tot = rep.reuse_hits + rep.fallbacks
        if tot > 0 and rep.fallbacks / tot > cfg.max_fallback_frac:
            raise FallbackBudgetExceeded(f"fallback fraction {rep.fallbacks / tot:.2f} exceeds configured "
                                         f"{cfg.max_fallback_frac:.2f}")
        rep.stage_seconds_measured = {"epoch": time.perf_counter() - t0}
        return rep

    def weights(self):
        return self.engine.params.to_numpy()

    def _local_seeds(self, batch: np.ndarray) -> np.ndarray:
        """This rank's contiguous shard of a global batch (all of it single-process)."""
        if self.dist is None:
            return batch
        from .parallel import shard
        return shard(batch, self.dist.world, self.dist.rank)

    # ------------------------------------------------------------------
    def train_step(self, seeds: np.ndarray, batch_seed: int, batch_in_epoch: int = 0):
        """One public training step from HOST seed ids (orchestrator._train_batch +
        the sampling call before it, orchestrator.py:461-468, 236-256): pinned H2D
        of the inputs, one graph replay, async D2H of the batch loss into a pinned
        slot.  Returns a handle; ``handle()`` synchronises and yields the loss."""
        if not hasattr(self, "_loss_pin"):
            self._loss_pin = [torch.zeros(1, dtype=torch.float32).pin_memory() for _ in range(8)]
            self._loss_k = 0
        gb = self.version
        n_div = self.dist.global_batch(seeds) if self.dist else None
        self.feeder.feed(seeds, batch_seed, gb, batch_in_epoch, n_div=n_div)
        self.engine.run_step()
        self.version += 1
        k = self._loss_k
        self._loss_k = (k + 1) % len(self._loss_pin)
        pin = self._loss_pin[k]
        pin.copy_(self.engine.d_loss, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()

        def handle():
            ev.synchronize()
            self.engine.check_numerics()  # the reference's non-finite guard (gnnmath.py:100-102)
            return float(pin.item())
        return handle

    def train_batches(self, batches):
        """Public pipelined training over HOST batches [(seed ids, batch rng seed), ...]:
        every step stages its seed ids pinned-H2D, the sample half of batch i+1
        overlaps the train half of batch i, and each step's loss is copied D2H into
        its own pinned slot.  Returns one handle per batch (call -> float loss)."""
        pipe, e = self.pipeline, self.engine
        n = len(batches)
        if n and e.g_sample is not None and os.environ.get("HG_NATIVE_LOOP", "1") != "0":
            return self._train_batches_native(batches)
        pin = torch.zeros(max(n, 1), dtype=torch.float32).pin_memory()
        v0 = self.version

        def feed(i):
            seeds, rs = batches[i]
            n_div = self.dist.global_batch(seeds) if self.dist else None
            return lambda set_index: self.feeder.feed(np.asarray(seeds), rs, v0 + i, 0, n_div=n_div,
                                                      set_index=set_index)

        done = torch.cuda.Event()
        if n:
            pipe.sample(0, feed(0))
        for i in range(n):
            if i + 1 < n:
                pipe.sample(i + 1, feed(i + 1))
            pipe.train(i)
            with torch.cuda.stream(pipe.st):
                pin[i:i + 1].copy_(e.d_loss, non_blocking=True)
        done.record(pipe.st)
        pipe.drain()
        self.version += n

        return self._handles(done, pin, n)

    def _train_batches_native(self, batches):
        """train_batches through the native step driver (hg_pipeline_run): one C
        call packs each batch's inputs into its pinned staging slot (SampleSet.stage
        layout) and enqueues that step's H2D and both half-step graphs, then the
        loss D2H — no Python work per step, and the device starts after the first
        batch is packed, not after all of them."""
        e, pipe = self.engine, self.pipeline
        n, cap = len(batches), e.batch_cap
        rec = int(e.loss_arr.numel())  # batch k records its loss at loss_arr[bp[3] = k]
        if n > rec:
            hs = []
            for i in range(0, n, rec):
                hs += self._train_batches_native(batches[i:i + rec])
            return hs
        slot = STAGE_SEEDS + 4 * cap
        prev = getattr(self, "_native_done", None)
        if prev is not None:
            prev.synchronize()  # the staging slots of the previous call may still be in flight
            self._native_fill()  # its losses leave the shared pinned buffer before it is reused
        buf = getattr(self, "_native_stage", None)
        if buf is None or buf.shape[0] < n:  # sized once for the largest call (a pinned
            # allocation costs ~ms of host time in front of the call's first launch)
            buf = torch.zeros((max(n, rec), slot), dtype=torch.uint8).pin_memory()
            self._native_stage = buf
        # per-batch host inputs; the native driver packs batch k into its pinned
        # staging slot right before launching step k
        seeds = [np.ascontiguousarray(s, dtype=np.int64) for s, _ in batches]
        n_seeds = np.fromiter((s.shape[0] for s in seeds), np.int32, n)
        if n and int(n_seeds.max()) > cap:
            raise ValueError("batch larger than the engine's capacity")
        n_div = (np.fromiter((self.dist.global_batch(s) for s in seeds), np.int32, n) if self.dist else n_seeds)
        seed_ptrs = np.fromiter((s.__array_interface__["data"][0] for s in seeds), np.int64, n)
        bp = np.zeros((n, 8), np.int64)
        bp[:, 0] = np.fromiter((int(rs) & 0xFFFFFFFFFFFFFFFF for _, rs in batches), np.uint64, n).view(np.int64)
        bp[:, 1] = n_seeds
        bp[:, 2] = self.version + np.arange(n)
        bp[:, 3] = np.arange(n)
        bp[:, 4] = -1
        bp[:, 6] = -1
        pin = getattr(self, "_native_loss", None)
        if pin is None or pin.numel() < n:
            pin = torch.zeros(max(n, rec), dtype=torch.float32).pin_memory()
            self._native_loss = pin
        execs_s = np.array([g.raw_cuda_graph_exec() for g in e.g_sample], np.int64)
        execs_t = np.array([g.raw_cuda_graph_exec() for g in e.g_train], np.int64)
        stages = np.array([st.stage.data_ptr() for st in e.sets], np.int64)
        cur = torch.cuda.current_stream(e.device)
        _lib.call("hg_pipeline_run", n, len(e.sets), execs_s.ctypes.data, execs_t.ctypes.data, cur.cuda_stream,
                  pipe.ss.cuda_stream, pipe.st.cuda_stream, stages.ctypes.data, buf.data_ptr(), slot, STAGE_COUNTS,
                  STAGE_SEEDS, bp.ctypes.data, seed_ptrs.ctypes.data, n_seeds.ctypes.data, n_div.ctypes.data,
                  ptr(e.loss_arr), pin.data_ptr())
        done = torch.cuda.Event()
        done.record(cur)
        self._native_done = done
        self.feeder.h2d_bytes = int(STAGE_SEEDS + 4 * n_seeds[0]) if n else 0
        self.version += n

        return self._handles(done, pin, n, native=True)

    def _handles(self, done, pin, n, native=False):
        """One loss handle per batch; the first handle to complete also checks the
        device numerics flags once for the whole call (gnnmath.py:100-102) and
        reads every loss of the call from the pinned buffer in one go."""
        vals = []

        def fill():
            if not vals:
                done.synchronize()
                self.engine.check_numerics()
                vals.append(pin[:n].tolist())

        def handle(i):
            def get():
                fill()
                return float(vals[0][i])
            return get
        if native:  # the next native call materialises these before reusing the pinned buffer
            self._native_fill = fill
        return [handle(i) for i in range(n)]

    @property
    def d2h_bytes_per_step(self) -> int:
        return 4


def evaluate(trainer_or_graph, weights=None, model=None) -> dict:
    """orchestrator.py:669-680: full-graph, full-neighbour inference accuracy."""
    if isinstance(trainer_or_graph, Trainer):
        t = trainer_or_graph
        dg, params, ds = t.dg, t.engine.params, t.ds
    else:
        raise TypeError("evaluate() takes a Trainer")
    acc, _ = full_graph_forward(dg, params, ds.val_mask, ds.test_mask)
    return acc


def full_graph_forward(dg: DeviceGraph, params, val_mask, test_mask, return_logits=False):
    dev = dg.device
    s = stream_ptr()
    V = dg.num_vertices
    sage = params.model == "sage"
    code = 0 if sage else 1
    outdeg = None
    if not sage:
        outdeg = torch.zeros(V, dtype=torch.int32, device=dev)
        _lib.call("hg_target_histogram", ptr(dg.targets), dg.num_edges, ptr(outdeg), s)
    h, ld = dg.features, dg.feat_ld
    nV = torch.tensor([V], dtype=torch.int32, device=dev)
    for l in range(params.L):
        d_in, d_out = params.dims[l], params.dims[l + 1]
        agg = torch.zeros((V, ld), dtype=torch.float32, device=dev)
        _lib.call("hg_full_aggregate", code, ptr(h), ld, ld, ptr(dg.offsets), ptr(dg.targets), V, ptr(outdeg),
                  ptr(agg), ld, s)
        ld_out = pad4(d_out)
        out = torch.zeros((V, ld_out), dtype=torch.float32, device=dev)
        act = 1 if l < params.L - 1 else 0
        if sage:
            dense.fwd(ptr(h), ld, ptr(agg), ld, d_in, ptr(params.view(l, 0)), d_out, ptr(out), ld_out, ptr(nV), V,
                      act, s)
        else:
            dense.fwd(ptr(agg), ld, None, 0, d_in, ptr(params.view(l, 0)), d_out, ptr(out), ld_out, ptr(nV), V, act, s)
        h, ld = out, ld_out
        del agg
    C = params.dims[-1]
    res = {}
    for name, m in (("val", val_mask), ("test", test_mask)):
        m = np.asarray(m, bool)
        if not m.any():
            res[name] = 0.0
            continue
        md = torch.as_tensor(m.astype(np.uint8), device=dev)
        corr = torch.zeros(1, dtype=torch.int64, device=dev)
        _lib.call("hg_argmax_correct", ptr(h), ld, C, V, ptr(dg.labels), ptr(md), ptr(corr), s)
        res[name] = float(int(corr.item()) / int(m.sum()))
    return res, (h[:, :C] if return_logits else None)


def run_training(graph, data=None, config: TrainConfig | None = None, device=None, hot_list=None,
                 dist=None, return_trainer=False):
    """orchestrator.py:683-725.  ``graph`` may be a datagen.Dataset (with
    ``data`` None) or a (Graph, VertexData) pair like the reference."""
    config = config or TrainConfig()
    ds = graph if data is None else _Merged(graph, data)
    tr = Trainer(ds, config, device=device, hot_list=hot_list, dist=dist)
    reports = []
    first = 0
    for epoch in range(config.epochs):
        plan = tr.build_epoch_plan(epoch, first)
        rep = tr.run_epoch(plan)
        acc = evaluate(tr)
        rep.val_accuracy, rep.test_accuracy = acc["val"], acc["test"]
        reports.append(rep)
        first += len(plan.batches)
    return (reports, tr) if return_trainer else reports


class _Merged:
    """(Graph, VertexData) viewed as one dataset object."""

    def __init__(self, graph, data):
        # an already-resident DeviceGraph (e.g. with row-sharded features) is used as is
        self.device_graph = graph if isinstance(graph, DeviceGraph) else None
        self.offsets, self.targets = graph.offsets, graph.targets
        self.features, self.labels = data.features, data.labels
        self.train_mask, self.val_mask, self.test_mask = data.train_mask, data.val_mask, data.test_mask


def epsilon_monitor(max_weight_deltas, n: int, batches_per_super_batch: int | None = None):
    """orchestrator.py:728-739."""
    size = batches_per_super_batch or n
    out = []
    for i in range(0, len(max_weight_deltas), size):
        w = max_weight_deltas[i:i + size]
        out.append(max(w) * 2 * n if w else 0.0)
    return out
