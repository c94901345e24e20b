"""The device-resident training step (the hot loop of orchestrator._run_epoch,
orchestrator.py:456-545, restated for one B200).

One step = one batch:

    sample L blocks top-down (K1-K3, sampler.py:130-147)
    -> historical-embedding lookup for the bottom destinations (store.py:67-98,
       orchestrator.py:486-500)
    -> bottom layer: fused feature gather + aggregation (K4/K5, orchestrator.py:239,
       gnnmath.py:157-179 / 105-126), dense transform (K8) + ReLU, injection of
       reused embeddings (gnnmath.py:240-245)
    -> upper layers, logits, softmax-CE (gnnmath.py:263-274)
    -> backward (gnnmath.py:250-260; dx only above the bottom layer)
    -> SGD / Adam over one flat parameter buffer + max |dw| (orchestrator.py:246-255)
    -> per-batch record (loss, max |dw|).

Every size that depends on sampling lives in device memory; buffers are sized
by static upper bounds (n_src <= n_dst*(f+1), <= V), so the whole step is
enqueued with zero host synchronisation and can be captured into a single
CUDA graph and replayed per batch.  Per-batch inputs (seed ids, the batch
rng seed and the store window parameters) are copied from pinned host memory
into fixed device buffers before each replay.
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np
import torch

from . import _lib, dense
from .device import DeviceGraph, pad4, ptr, stream_ptr
from .sampler import LayerSampler

# per-batch parameter block layout (see csrc/hg_train.cu BP_*)
BP_RNG_SEED, BP_N_SEEDS, BP_READING_BATCH, BP_BATCH_IN_EPOCH = 0, 1, 2, 3
BP_CPU_TAG, BP_TABLE_SEL, BP_CUR_STAMP, BP_WARMUP = 4, 5, 6, 7
BP_SIZE = 8


class DenseParams:
    """All layer weights in one flat fp32 device buffer (gnnmath.ModelParams,
    gnnmath.py:24-52).  GCN: [W] per layer; SAGE: [W_self, W_neigh] per layer,
    each row-major [d_in, d_out]."""

    def __init__(self, model: str, dims, weights, device):
        self.model = model
        self.dims = [int(d) for d in dims]
        self.L = len(self.dims) - 1
        self.n_mats = 1 if model == "gcn" else 2
        self.offs = []
        off = 0
        for l in range(self.L):
            row = []
            for _ in range(self.n_mats):
                row.append(off)
                off += self.dims[l] * self.dims[l + 1]
            self.offs.append(row)
        self.numel = off
        self.flat = torch.zeros(off, dtype=torch.float32, device=device)
        self.grad = torch.zeros_like(self.flat)
        if weights is not None:
            self.load(weights)

    def view(self, l: int, m: int, buf=None) -> torch.Tensor:
        buf = self.flat if buf is None else buf
        n = self.dims[l] * self.dims[l + 1]
        return buf[self.offs[l][m]:self.offs[l][m] + n].view(self.dims[l], self.dims[l + 1])

    def load(self, weights):
        for l, lw in enumerate(weights):
            for m, w in enumerate(lw):
                self.view(l, m).copy_(torch.as_tensor(np.asarray(w, dtype=np.float32)))

    def to_numpy(self, buf=None):
        return [[self.view(l, m, buf).cpu().numpy().astype(np.float64) for m in range(self.n_mats)]
                for l in range(self.L)]

    @property
    def bottom_numel(self) -> int:
        return self.n_mats * self.dims[0] * self.dims[1]


@dataclass
class HotBuffers:
    """Device embedding store (store.py:24-146): two physical tables that swap
    the roles "current" / "staging" per super-batch via BP_TABLE_SEL; entries are
    valid for reading iff their stamp equals BP_CUR_STAMP, which makes both
    advance_super_batch and reset_epoch O(1) (no clearing)."""

    slot_of: torch.Tensor      # int32 [V]: hot-list position or -1
    cpu_tag_of: torch.Tensor   # int32 [V]: membership tag of the current cpu_set
    tab: list                  # 2 x fp32 [n_hot, H]
    ver: list                  # 2 x int32 [n_hot]
    stamp: list                # 2 x int32 [n_hot]
    inj_mask: torch.Tensor     # uint8 [cap_dst0]
    inj_slot: torch.Tensor     # int32 [cap_dst0]
    batch_hits: torch.Tensor   # int32 [max_batches]
    batch_miss: torch.Tensor
    batch_warm: torch.Tensor
    stats: torch.Tensor        # uint64 as int64 [2]: packed (max gap, batch), violations
    puts: torch.Tensor         # int32 [1]
    gap_bound: int
    H: int

    @classmethod
    def create(cls, V, hot_list, H, n, cap_dst0, max_batches, device):
        n_hot = max(int(hot_list.shape[0]), 1)
        slot_of = torch.full((V,), -1, dtype=torch.int32, device=device)
        if hot_list.shape[0]:
            slot_of[torch.as_tensor(hot_list.astype(np.int64), device=device)] = torch.arange(
                hot_list.shape[0], dtype=torch.int32, device=device)
        z = lambda *s, dt=torch.int32: torch.zeros(*s, dtype=dt, device=device)  # noqa: E731
        return cls(slot_of=slot_of, cpu_tag_of=torch.full((V,), -1, dtype=torch.int32, device=device),
                   tab=[z(n_hot, H, dt=torch.float32), z(n_hot, H, dt=torch.float32)],
                   ver=[z(n_hot), z(n_hot)],
                   stamp=[torch.full((n_hot,), -1, dtype=torch.int32, device=device) for _ in range(2)],
                   inj_mask=z(max(cap_dst0, 1), dt=torch.uint8), inj_slot=z(max(cap_dst0, 1)),
                   batch_hits=z(max_batches), batch_miss=z(max_batches), batch_warm=z(max_batches),
                   stats=z(2, dt=torch.int64), puts=z(1), gap_bound=2 * n - 1, H=H)

    def reset_counters(self):
        for t in (self.batch_hits, self.batch_miss, self.batch_warm, self.puts):
            t.zero_()


def _new_graph():
    """A CUDA graph that keeps its cudaGraph_t (kernel-node counting)."""
    try:
        return torch.cuda.CUDAGraph(keep_graph=True)
    except TypeError:
        return torch.cuda.CUDAGraph()


@dataclass
class SampleSet:
    """One batch's sampled blocks plus its per-batch device inputs."""

    samplers: list
    seeds: torch.Tensor      # int32 [batch_cap]
    counts_in: torch.Tensor  # int32 [2]: n_seeds, gradient divisor (global batch)
    bp: torch.Tensor         # int64 [BP_SIZE] parameter block
    stage: torch.Tensor      # uint8: bp | counts_in | seeds as ONE buffer (one H2D copy per batch)
    # the train half's private copy of ``stage``, made by the sample half (a side
    # branch of its graph): the next H2D into ``stage`` then only has to wait for
    # this set's previous SAMPLE half, not its train half
    tstage: torch.Tensor = None
    tviews: tuple = None


STAGE_COUNTS = BP_SIZE * 8       # byte offsets inside SampleSet.stage
STAGE_SEEDS = BP_SIZE * 8 + 16


def stage_views(stage: torch.Tensor):
    """(bp int64[BP_SIZE], counts int32[2], seeds int32[...]) views of a staging buffer."""
    return (stage[:STAGE_COUNTS].view(torch.int64), stage[STAGE_COUNTS:STAGE_COUNTS + 8].view(torch.int32),
            stage[STAGE_SEEDS:].view(torch.int32))


class TrainEngine:
    """Buffers + kernel sequence of one training step for a fixed model/fanout."""

    # the current sample set's views (eager steps, capture and host planning use set `cur`)
    samplers = property(lambda self: self.sets[self.cur].samplers)
    # per-batch inputs: the staging buffer while the sample half is enqueued, the
    # train half's private copy of it while the train half is enqueued
    seeds = property(lambda self: self.sets[self.cur].tviews[2] if self._train_view else self.sets[self.cur].seeds)
    counts_in = property(lambda self: self.sets[self.cur].tviews[1] if self._train_view
                         else self.sets[self.cur].counts_in)
    bp = property(lambda self: self.sets[self.cur].tviews[0] if self._train_view else self.sets[self.cur].bp)
    _train_view = False

    def __init__(self, dg: DeviceGraph, model: str, dims, fanouts, batch_cap: int, lr: float,
                 optimizer: str = "sgd", weights=None, hot: HotBuffers | None = None, max_batches: int = 1,
                 allreduce=None, n_sets: int | None = None):
        _lib.load()
        if model not in ("gcn", "sage"):
            raise ValueError(f"unknown model {model!r}")
        self.dg, self.model = dg, model
        self.sage = model == "sage"
        self.dims = [int(d) for d in dims]
        self.fan = [int(f) for f in fanouts]
        self.L = len(self.fan)
        assert len(self.dims) == self.L + 1
        self.batch_cap = int(batch_cap)
        self.lr = float(lr)
        self.optimizer = optimizer
        self.hot = hot
        self.allreduce = allreduce  # callable(grad_tensor) for multi-GPU data parallel
        dev = self.device = dg.device
        V = dg.num_vertices
        if self.dims[0] != dg.feat_dim:
            raise ValueError("feature width mismatch")
        self.ld = [pad4(d) for d in self.dims]
        self.ld[0] = dg.feat_ld
        # ---- capacities, top-down (sampler.py:142-146) ----
        self.cap_dst = [0] * self.L
        self.cap_src = [0] * self.L
        self.cap_dst[self.L - 1] = self.batch_cap
        for l in range(self.L - 1, -1, -1):
            self.cap_src[l] = int(min(V, self.cap_dst[l] * (self.fan[l] + 1)))
            if l > 0:
                self.cap_dst[l - 1] = self.cap_src[l]
        # ---- two sample sets (blocks + per-batch inputs): batch k+1 is sampled into
        # one while batch k trains from the other (the reference's sampler/trainer
        # overlap, SPEC pipelining; sampling never reads weights, so results are
        # bit-identical to the sequential order) ----
        z32 = lambda *s: torch.zeros(*s, dtype=torch.int32, device=dev)  # noqa: E731
        zf = lambda *s: torch.zeros(*s, dtype=torch.float32, device=dev)  # noqa: E731
        # relabel halves of layers >= 1 off the sampling critical path (HG_SPLIT_RELABEL=0: in line)
        self.split_relabel = os.environ.get("HG_SPLIT_RELABEL", "1") != "0"
        self.sets = []
        # sample sets in flight (the pipeline reuses set k % n_sets after batch k - n_sets trained)
        n_sets = int(os.environ.get("HG_SETS", "2")) if n_sets is None else int(n_sets)
        for k in range(n_sets):
            mp = dg.minpos if k == 0 else dg.minpos.like()
            # layers of opposite parity use different first-occurrence tables: a
            # layer's relabel half runs on a side stream concurrently with the next
            # layer's draw + mark (enqueue_sample_part)
            mps = (mp, mp.like() if self.L > 1 and self.split_relabel else mp)
            # outdeg: GCN norm; for layers >= 1 also the per-source edge counts that
            # select the backward scatter's single-contribution fast path
            smp = [LayerSampler(dg, self.cap_dst[l], self.fan[l], need_nself=self.sage,
                                need_outdeg=(not self.sage) or l > 0, minpos=mps[l % 2]) for l in range(self.L)]
            stage = torch.zeros(STAGE_SEEDS + 4 * self.batch_cap, dtype=torch.uint8, device=dev)
            bp, counts_in, seeds = stage_views(stage)
            tstage = torch.zeros_like(stage)
            self.sets.append(SampleSet(samplers=smp, seeds=seeds, counts_in=counts_in, bp=bp, stage=stage,
                                       tstage=tstage, tviews=stage_views(tstage)))
        self.cur = 0
        # ---- parameters ----
        self.params = DenseParams(model, self.dims, weights, dev)
        if optimizer == "adam":
            self.adam_m = torch.zeros_like(self.params.flat)
            self.adam_v = torch.zeros_like(self.params.flat)
            self.adam_t = z32(1)
        # ---- activations / gradients ----
        self.self_buf = zf(self.cap_dst[0], self.ld[0]) if self.sage else None
        self.agg = [zf(self.cap_dst[l], self.ld[l]) for l in range(self.L)]
        # bottom aggregation outputs per sample set: the bottom gather+aggregate
        # needs no weights, so (without hot-embedding injection) it runs in the
        # SAMPLE half of batch k+1 while batch k trains (see early_agg0)
        self._self_bufs = [self.self_buf] + [zf(self.cap_dst[0], self.ld[0]) if self.sage else None
                                             for _ in range(n_sets - 1)]
        self._agg0s = [self.agg[0]] + [zf(self.cap_dst[0], self.ld[0]) for _ in range(n_sets - 1)]
        self.out = [zf(self.cap_dst[l], self.ld[l + 1]) for l in range(self.L)]  # out[l] = H_{l+1}
        self.dz = [zf(self.cap_dst[l], self.ld[l + 1]) for l in range(self.L)]
        self.dagg = [zf(self.cap_dst[l], self.ld[l]) if l > 0 else None for l in range(self.L)]
        self.dself = [zf(self.cap_dst[l], self.ld[l]) if (l > 0 and self.sage) else None for l in range(self.L)]
        lib = _lib.load()
        ws = max(dense.wgrad_ws_size(self.dims[l], self.dims[l + 1], self.cap_dst[l], 2 if self.sage else 1)
                 for l in range(self.L))
        self.wgrad_ws = zf(max(ws, 1))
        # two-word fixed-point accumulators (hi | lo words per row, hg_aggregate.cu)
        self.fx_acc = [torch.zeros((self.cap_src[l], 2 * self.ld[l]), dtype=torch.int64, device=dev)
                       if l > 0 else None for l in range(self.L)]
        self.fx_flags = z32(1)
        self.d_loss = zf(1)
        self.row_loss = zf(self.batch_cap + 1)  # + the loss kernel's last-block ticket
        self.d_maxdelta = z32(2)  # max |dw| bits + the fused update's last-block ticket
        self.loss_arr = zf(max(max_batches, 1))
        self.md_arr = zf(max(max_batches, 1))
        # per-batch needed bottom rows (the reference's transfer accounting,
        # transfer.py:59-73) on a side branch of the train half
        self.raw_rows_arr = z32(max(max_batches, 1))
        self.cache_hit_arr = z32(max(max_batches, 1))
        self.static_cached = None  # uint8 [V]: the case3/case4 static feature cache (accounting only)
        self.account_rows = True  # TrainConfig.report_transfers
        self.need_tag = torch.full((max(V, 1),), -1, dtype=torch.int32, device=dev)
        self.side = (torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev))
        # tensor-core B operand images, rebuilt from the current weights each step
        self.img_fwd = [dense.BImage(self.dims[l], self.dims[l] if self.sage else 0, self.dims[l + 1], 1, dev)
                        for l in range(self.L)]
        # SAGE dX: one GEMM against the stacked [W_self; W_neigh] gives [dself | dmean]
        # side by side (when d_in keeps both halves 16-byte aligned)
        self.fused_dx = [self.sage and l > 0 and self.dims[l] % 4 == 0 for l in range(self.L)]
        self.dcat = [zf(self.cap_dst[l], 2 * self.dims[l]) if self.fused_dx[l] else None for l in range(self.L)]
        self.img_dx = []
        for l in range(self.L):
            if l == 0:
                self.img_dx.append([])
            elif self.fused_dx[l]:
                self.img_dx.append([dense.BImage(self.dims[l + 1], 0, 2 * self.dims[l], 0, dev)])
            else:
                nm = 2 if self.sage else 1
                self.img_dx.append([dense.BImage(self.dims[l + 1], 0, self.dims[l], 0, dev) for _ in range(nm)])
        # the top SAGE layer's aggregate -> transform -> loss -> dX -> scatter in one kernel
        self.top_fused = (self.sage and self.L >= 2 and self.dims[self.L - 1] <= 64
                          and self.dims[self.L] <= 64 and self.fan[self.L - 1] <= 32
                          and self.fused_dx[self.L - 1] and os.environ.get("HG_TOP_FUSED", "1") != "0")
        self.graph = None
        self.g_sample = None
        self.g_train = None
        self.enqueue_weight_images()

    def _image_jobs(self):
        """(image, source weight pointer) of every tensor-core B image."""
        P = self.params
        jobs = []
        for l in range(self.L):
            jobs.append((self.img_fwd[l], ptr(P.view(l, 0))))
            for m, img in enumerate(self.img_dx[l]):
                jobs.append((img, ptr(P.view(l, m))))
        return jobs

    def _image_desc(self, jobs):
        return np.array([[w, self._ldb_of(img), img.trans_b, img.K1, img.K2, img.N, img.buf.data_ptr()]
                         for img, w in jobs], dtype=np.int64)

    def enqueue_weight_images(self, stream=None):
        """Rebuild every tensor-core B image from the current weights (one launch)."""
        s = stream_ptr(stream)
        jobs = self._image_jobs()
        for i in range(0, len(jobs), 8):
            part = jobs[i:i + 8]
            desc = self._image_desc(part)
            _lib.call("hg_gemm_tc_prep_b_many", len(part), desc.ctypes.data, s)

    def _ldb_of(self, img):
        """Row stride of the weight matrix an image is built from."""
        return img.N if img.trans_b else img.K1

    # ------------------------------------------------------------------
    def frontier(self, l):
        """(frontier ids, device count) of layer l's destinations."""
        if l == self.L - 1:
            return self.seeds, self.counts_in[0:1]
        s = self.samplers[l + 1]
        return s.src, s.n_src

    def enqueue_sample(self, stream=None, seed_ptr=None, layers=None):
        """Blocks L-1 .. 0 (sampler.py:142-146); layer l's stream is
        derive_seed(*seed, 0x5A, l), computed on device."""
        sp = self.bp if seed_ptr is None else seed_ptr
        for l in (range(self.L - 1, -1, -1) if layers is None else layers):
            fr, n = self.frontier(l)
            self.samplers[l].run(fr, n, sp, l, stream)

    #: phase boundaries enqueue_step reports through ``mark`` (for split capture / timing)
    MARKS = ("fwd0_agg", "fwd0_gemm", "fwd_upper", "loss", "bwd", "update")

    def enqueue_step(self, stream=None, mark=None):
        """One whole batch (sample + train) on one stream."""
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.enqueue_sample_part(main)
        self.enqueue_train_part(main, mark)

    def early_agg0(self) -> bool:
        """Bottom gather+aggregate in the sample half (no weights involved), also
        with hot-embedding reuse: there the rows of destinations that the train
        half's store lookup will inject are aggregated too (no skip mask yet) and
        simply overwritten after the GEMM — their dz is masked to zero, so the
        weight gradient is bit-identical — which keeps the aggregation overlapped
        with the previous batch's training.  HG_EARLY_AGG=0: in the train half,
        skipping the injected rows (HG_EARLY_AGG_HOT=0: that only with reuse)."""
        if os.environ.get("HG_EARLY_AGG", "1") == "0":
            return False
        return self.hot is None or os.environ.get("HG_EARLY_AGG_HOT", "1") != "0"

    def _bottom_bufs(self):
        """(self rows, aggregate) buffers of the bottom layer for the current set."""
        k = self.cur if self.early_agg0() else 0
        return self._self_bufs[k], self._agg0s[k]

    def _enqueue_agg0(self, s, inj=None):
        smp = self.samplers[0]
        fr, n = self.frontier(0)
        sb, ag = self._bottom_bufs()
        sh = getattr(self.dg, "shards", None)
        if sh is not None:  # feature rows spread over the box's GPUs (parallel.ShardedFeatures)
            _lib.call("hg_aggregate_fwd_sharded", 0 if self.sage else 1, sh.ptrs, sh.n_shards, sh.rows_per_shard,
                      sh.ld, self.ld[0], ptr(fr), ptr(n), self.cap_dst[0], self.fan[0], ptr(smp.counts),
                      ptr(smp.slots), ptr(smp.slot_local), ptr(smp.nself), ptr(smp.outdeg), ptr(inj),
                      ptr(sb if self.sage else None), self.ld[0], ptr(ag), self.ld[0], s)
            return
        sp = self.dg.split_rows() if hasattr(self.dg, "split_rows") else None
        if sp is not None and sp["body_cols"] + sp["tail_cols"] == self.ld[0]:  # line-aligned body + L2-held tail
            _lib.call("hg_aggregate_fwd_split", 0 if self.sage else 1, ptr(sp["body"]), sp["body_cols"],
                      ptr(sp["tail"]), sp["tail_cols"], sp["body_cols"], self.ld[0], ptr(fr), ptr(n),
                      self.cap_dst[0], self.fan[0], ptr(smp.counts), ptr(smp.slots), ptr(smp.slot_local),
                      ptr(smp.nself), ptr(smp.outdeg), ptr(inj), ptr(sb if self.sage else None), self.ld[0],
                      ptr(ag), self.ld[0], s)
            return
        _lib.call("hg_aggregate_fwd", 0 if self.sage else 1, 1, ptr(self.dg.features), self.dg.feat_ld, self.ld[0],
                  ptr(fr), ptr(n), self.cap_dst[0], self.fan[0], ptr(smp.counts), ptr(smp.slots),
                  ptr(smp.slot_local), ptr(smp.nself), ptr(smp.outdeg), ptr(inj), ptr(sb if self.sage else None),
                  self.ld[0], ptr(ag), self.ld[0], s)

    def enqueue_sample_part(self, stream=None, mark=None):
        """Blocks L-1..0 of the current set (+ the bottom aggregation when
        early_agg0); the transposed (backward) views of the CSC path are built on
        a side stream (a parallel graph branch) joined at the end."""
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        sc = self.side[1]
        forked = False
        if mark is not None:  # a mark may end a capture segment: join the side branch first
            user_mark = mark

            def mark(name):
                nonlocal forked
                if forked:
                    main.wait_stream(sc)
                    forked = False
                user_mark(name)
        else:
            mark = lambda name: None  # noqa: E731
        for l in range(self.L - 1, -1, -1):
            if l < self.L - 1:
                mark(f"sample_l{l}")
            fr, n = self.frontier(l)
            smp = self.samplers[l]
            if forked and l + 2 < self.L and self.samplers[l + 2].minpos is smp.minpos:
                main.wait_stream(sc)  # the table is still being read by layer l+2's relabel
            split = self.split_relabel and l > 0 and not self._bottom_draws_only(l)
            smp.run(fr, n, self.bp, l, main, dedup=not self._bottom_draws_only(l),
                    relabel_stream=sc if split else None)
            forked = forked or split
            if l == self.L - 1:  # the train half's copy of the batch inputs, on the side branch
                # (forked after the first kernels so the graph keeps a single root)
                sc.wait_stream(main)
                st_ = self.sets[self.cur]
                _lib.call("hg_copy_bytes", ptr(st_.tstage), ptr(st_.stage), st_.stage.numel(), sc.cuda_stream)
                forked = True
        if self.early_agg0():
            mark("sample_agg0")
            self._enqueue_agg0(main.cuda_stream)
        if forked:  # the relabel halves also overlap the bottom aggregation
            main.wait_stream(sc)

    def enqueue_train_part(self, stream=None, mark=None):
        """The train half of the current set; it reads the batch's inputs from the
        private copy the sample half made (SampleSet.tstage)."""
        self._train_view = True
        try:
            self._enqueue_train_part(stream, mark)
        finally:
            self._train_view = False

    def _enqueue_train_part(self, stream=None, mark=None):
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        s = main.cuda_stream
        L, P = self.L, self.params
        g = self.dg
        mark = mark or (lambda name: None)
        hot = self.hot
        inj = None
        if hot is not None and L > 1:
            fr0, n0 = self.frontier(0)
            _lib.call("hg_store_lookup", ptr(fr0), ptr(n0), self.cap_dst[0], ptr(self.bp), ptr(hot.cpu_tag_of),
                      ptr(hot.slot_of), ptr(hot.ver[0]), ptr(hot.ver[1]), ptr(hot.stamp[0]), ptr(hot.stamp[1]),
                      hot.gap_bound, ptr(hot.inj_mask), ptr(hot.inj_slot), ptr(hot.batch_hits),
                      ptr(hot.batch_miss), ptr(hot.batch_warm), ptr(hot.stats), s)
            inj = hot.inj_mask
        model = 0 if self.sage else 1
        # ---------------- forward ----------------
        for l in range(L):
            if l == L - 1 and self.top_fused:
                break  # folded into the fused top-layer kernel below
            smp = self.samplers[l]
            fr, n = self.frontier(l)
            d_in, d_out = self.dims[l], self.dims[l + 1]
            if l == 0:
                hin, ld_in, glob = g.features, g.feat_ld, 1
            else:
                hin, ld_in, glob = self.out[l - 1], self.ld[l], 0
            mark("fwd0_agg" if l == 0 else "fwd_upper" if l == 1 else "")
            sb0, ag0 = self._bottom_bufs()
            agg_l = ag0 if l == 0 else self.agg[l]
            if l == 0:
                if not self.early_agg0():
                    self._enqueue_agg0(s, inj)
            else:
                _lib.call("hg_aggregate_fwd", model, glob, ptr(hin), ld_in, self.ld[l], ptr(fr), ptr(n),
                          self.cap_dst[l], self.fan[l], ptr(smp.counts), ptr(smp.slots), ptr(smp.slot_local),
                          ptr(smp.nself), ptr(smp.outdeg), None, None, self.ld[0], ptr(agg_l), self.ld[l], s)
            act = 1 if l < L - 1 else 0
            mark("fwd0_gemm" if l == 0 else "")
            if self.sage:  # [h_self | mean] [W_self; W_neigh]
                a1, lda1 = (sb0, self.ld[0]) if l == 0 else (self.out[l - 1], self.ld[l])
                dense.fwd(ptr(a1), lda1, ptr(agg_l), self.ld[l], d_in, ptr(P.view(l, 0)), d_out,
                          ptr(self.out[l]), self.ld[l + 1], ptr(n), self.cap_dst[l], act, s, img=self.img_fwd[l])
            else:
                dense.fwd(ptr(agg_l), self.ld[l], None, 0, d_in, ptr(P.view(l, 0)), d_out, ptr(self.out[l]),
                          self.ld[l + 1], ptr(n), self.cap_dst[l], act, s, img=self.img_fwd[l])
            if l == 0 and inj is not None:
                _lib.call("hg_inject_rows", ptr(hot.inj_mask), ptr(hot.inj_slot), ptr(n), self.cap_dst[0],
                          ptr(self.bp), ptr(hot.tab[0]), ptr(hot.tab[1]), hot.H, ptr(self.out[0]), self.ld[1], s)
        # ---------------- loss ----------------
        mark("loss")
        C = self.dims[L]
        if self.top_fused:
            l = L - 1
            smp = self.samplers[l]
            fr, n = self.frontier(l)
            d_in = self.dims[l]
            _lib.call("hg_sage_top_fused", ptr(self.out[l - 1]), self.ld[l], d_in, ptr(fr), ptr(n), self.cap_dst[l],
                      self.fan[l], ptr(smp.counts), ptr(smp.slots), ptr(smp.slot_local), ptr(smp.nself),
                      ptr(smp.outdeg), ptr(P.view(l, 0)), C, ptr(g.labels), ptr(self.seeds),
                      ptr(self.counts_in[1:2]), ptr(self.out[l]), self.ld[L], ptr(self.dz[l]), ptr(self.agg[l]),
                      self.ld[l], ptr(self.dcat[l]), 2 * d_in, ptr(self.out[l - 1]), self.ld[l],
                      ptr(inj if l - 1 == 0 else None), ptr(self.fx_acc[l]), self.ld[l], ptr(self.dz[l - 1]),
                      self.ld[l], ptr(self.fx_flags), ptr(self.row_loss), ptr(self.d_loss), s)
        else:
            _lib.call("hg_softmax_xent", ptr(self.out[L - 1]), self.ld[L], C, ptr(self.counts_in[0:1]),
                      self.batch_cap, ptr(g.labels), ptr(self.seeds), ptr(self.counts_in[1:2]), ptr(self.dz[L - 1]),
                      self.ld[L], ptr(self.d_loss), ptr(self.row_loss), s)
        # ---------------- backward ----------------
        mark("bwd")
        # weight gradients of layer l only need dz[l]: they run on a side stream (a
        # parallel graph branch) while dX of layer l and everything below proceed
        sw = self.side[0]
        for l in range(L - 1, -1, -1):
            smp = self.samplers[l]
            fr, n = self.frontier(l)
            d_in, d_out = self.dims[l], self.dims[l + 1]
            sw.wait_stream(main)
            ws_ = sw.cuda_stream
            sb0, ag0 = self._bottom_bufs()
            agg_l = ag0 if l == 0 else self.agg[l]
            if self.sage:  # dW_self = h_self^T dz, dW_neigh = mean^T dz (gnnmath.py:190-191)
                a1, lda1 = (sb0, self.ld[0]) if l == 0 else (self.out[l - 1], self.ld[l])
                dense.wgrad(ptr(a1), lda1, ptr(agg_l), self.ld[l], d_in, ptr(self.dz[l]), self.ld[l + 1],
                            d_out, ptr(n), self.cap_dst[l], ptr(P.view(l, 0, P.grad)), ptr(P.view(l, 1, P.grad)),
                            ptr(self.wgrad_ws), ws_)
            else:  # dW = agg^T dz (gnnmath.py:135)
                dense.wgrad(ptr(agg_l), self.ld[l], None, 0, d_in, ptr(self.dz[l]), self.ld[l + 1], d_out,
                            ptr(n), self.cap_dst[l], ptr(P.view(l, 0, P.grad)), None, ptr(self.wgrad_ws), ws_)
            if l == 0:
                continue
            if l == L - 1 and self.top_fused:  # dX + scatter already ran in the fused top kernel
                _lib.call("hg_aggregate_bwd_finish", ptr(self.dcat[l]), 2 * self.dims[l], self.ld[l], ptr(n),
                          self.cap_dst[l], ptr(smp.n_src), self.cap_src[l], ptr(smp.outdeg), ptr(self.out[l - 1]),
                          self.ld[l], ptr(inj if l - 1 == 0 else None), ptr(self.fx_acc[l]), ptr(self.dz[l - 1]),
                          self.ld[l], s)
                continue
            if self.fused_dx[l]:  # [dself | dmean] = dz [W_self; W_neigh]^T in one GEMM
                dense.dx(ptr(self.dz[l]), self.ld[l + 1], d_out, ptr(P.view(l, 0)), 2 * d_in, ptr(self.dcat[l]),
                         2 * d_in, ptr(n), self.cap_dst[l], s, img=self.img_dx[l][0])
                dsp, dsl = self.dcat[l].data_ptr(), 2 * d_in
                dap, dal = dsp + 4 * d_in, 2 * d_in
            elif self.sage:  # dself = dz W_self^T, dmean = dz W_neigh^T
                dense.dx(ptr(self.dz[l]), self.ld[l + 1], d_out, ptr(P.view(l, 0)), d_in, ptr(self.dself[l]),
                         self.ld[l], ptr(n), self.cap_dst[l], s, img=self.img_dx[l][0])
                dense.dx(ptr(self.dz[l]), self.ld[l + 1], d_out, ptr(P.view(l, 1)), d_in, ptr(self.dagg[l]),
                         self.ld[l], ptr(n), self.cap_dst[l], s, img=self.img_dx[l][1])
                dsp, dsl, dap, dal = ptr(self.dself[l]), self.ld[l], ptr(self.dagg[l]), self.ld[l]
            else:
                dense.dx(ptr(self.dz[l]), self.ld[l + 1], d_out, ptr(P.view(l, 0)), d_in, ptr(self.dagg[l]),
                         self.ld[l], ptr(n), self.cap_dst[l], s, img=self.img_dx[l][0])
                dsp, dsl, dap, dal = None, 0, ptr(self.dagg[l]), self.ld[l]
            _lib.call("hg_aggregate_bwd_scatter", model, dap, dal, dsp, dsl, self.ld[l], ptr(fr), ptr(n),
                      self.cap_dst[l], self.fan[l], ptr(smp.counts), ptr(smp.slots), ptr(smp.slot_local),
                      ptr(smp.nself), ptr(smp.outdeg), ptr(smp.n_src), self.cap_src[l], ptr(self.out[l - 1]),
                      self.ld[l], ptr(inj if l - 1 == 0 else None), ptr(self.fx_acc[l]), ptr(self.dz[l - 1]),
                      self.ld[l], ptr(self.fx_flags), s)
        main.wait_stream(sw)
        if self.account_rows:  # the reference's per-batch transfer accounting (bookkeeping only)
            fr0, n0 = self.frontier(0)
            smp0 = self.samplers[0]
            _lib.call("hg_count_needed_rows", ptr(fr0), ptr(n0), self.cap_dst[0], self.fan[0], ptr(smp0.counts),
                      ptr(smp0.slots), ptr(inj), ptr(self.bp), ptr(self.static_cached), ptr(self.need_tag),
                      ptr(self.raw_rows_arr), ptr(self.cache_hit_arr), s)
        # ---------------- update ----------------
        mark("update")
        if self.allreduce is not None:
            self.allreduce(P.grad)
        jobs = self._image_jobs()
        if self.optimizer == "sgd" and len(jobs) <= 8:
            # SGD + B images of the updated weights + batch record: one launch
            desc = self._image_desc(jobs)
            _lib.call("hg_sgd_fused", ptr(P.flat), ptr(P.grad), P.numel, self.lr, len(jobs), desc.ctypes.data,
                      ptr(self.d_maxdelta), ptr(self.bp), ptr(self.d_loss), ptr(self.loss_arr), ptr(self.md_arr), s)
            return
        if self.optimizer == "sgd":
            _lib.call("hg_sgd", ptr(P.flat), ptr(P.grad), P.numel, self.lr, ptr(self.d_maxdelta), s)
        else:
            _lib.call("hg_adam", ptr(P.flat), ptr(P.grad), ptr(self.adam_m), ptr(self.adam_v), P.numel, self.lr,
                      0.9, 0.999, 1e-8, ptr(self.adam_t), ptr(self.d_maxdelta), s)
        _lib.call("hg_record_batch", ptr(self.bp), ptr(self.d_loss), ptr(self.d_maxdelta), ptr(self.loss_arr),
                  ptr(self.md_arr), s)
        # tensor-core B images of the updated weights, ready for the next step
        self.enqueue_weight_images(main)

    # ------------------------------------------------------------------
    def _warmup(self, stream):
        """Run one eager step outside capture (lazy module loads, smem attributes),
        then undo its side effects."""
        saved = self._save_state()
        stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(stream):
            for k in range(len(self.sets)):
                self.cur = k
                self.enqueue_step(stream)
        self.cur = 0
        torch.cuda.current_stream(self.device).wait_stream(stream)
        torch.cuda.synchronize(self.device)
        self._restore_state(saved)

    def capture(self, stream: torch.cuda.Stream | None = None):
        """Capture enqueue_step (set 0) into one CUDA graph, and the sample /
        train halves of every set into separate graphs for pipelined replay."""
        stream = stream or torch.cuda.Stream(device=self.device)
        self._warmup(stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            self.enqueue_step()
        self.g_sample, self.g_train = [], []
        for k in range(len(self.sets)):
            self.cur = k
            gs, gt = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(gs, stream=stream):
                self.enqueue_sample_part()
            with torch.cuda.graph(gt, stream=stream):
                self.enqueue_train_part()
            self.g_sample.append(gs)
            self.g_train.append(gt)
        self.cur = 0
        torch.cuda.synchronize(self.device)
        self.graph = g
        return g

    def capture_segments(self, split_at=(), stream: torch.cuda.Stream | None = None, set_index: int = 0):
        """Capture the halves of set ``set_index`` as consecutive graphs split
        before the marks in ``split_at`` (so a caller can record CUDA events between
        segments, e.g. around the dominant kernel).  Returns (sample, [(first_mark,
        graph), ...]) where sample is one graph, or a [(mark, graph), ...] list when
        a mark split the sample half too."""
        stream = stream or torch.cuda.Stream(device=self.device)
        if self.g_sample is None:
            self._warmup(stream)
        self.cur = set_index
        ssegs = []
        scur = {"g": _new_graph(), "name": "start"}

        def smark(name):
            if name in split_at:
                scur["g"].capture_end()
                ssegs.append((scur["name"], scur["g"]))
                scur["g"], scur["name"] = _new_graph(), name
                scur["g"].capture_begin()

        with torch.cuda.stream(stream):
            scur["g"].capture_begin()
            self.enqueue_sample_part(mark=smark)
            scur["g"].capture_end()
            ssegs.append((scur["name"], scur["g"]))
        gs = ssegs[0][1] if len(ssegs) == 1 else ssegs
        segs = []
        cur = {"g": _new_graph(), "name": "start"}

        def mark(name):
            if name in split_at:
                cur["g"].capture_end()
                segs.append((cur["name"], cur["g"]))
                cur["g"], cur["name"] = _new_graph(), name
                cur["g"].capture_begin()

        with torch.cuda.stream(stream):
            cur["g"].capture_begin()
            self.enqueue_train_part(mark=mark)
            cur["g"].capture_end()
            segs.append((cur["name"], cur["g"]))
        self.cur = 0
        for g in [g for _, g in ssegs] + [g for _, g in segs]:
            if hasattr(g, "instantiate"):
                try:
                    g.instantiate()
                except RuntimeError:
                    pass
        torch.cuda.synchronize(self.device)
        return gs, segs

    def _bottom_draws_only(self, l: int) -> bool:
        """SAGE's bottom block is consumed by global source id only (fused gather
        of feature rows; no transposed aggregation below layer 0, gnnmath.py:256),
        so the training step skips its dedup/relabel pass (HG_BOTTOM_DEDUP=1 keeps
        it).  GCN needs the block-local out-degrees (gnnmath.py:96)."""
        return l == 0 and self.sage and os.environ.get("HG_BOTTOM_DEDUP", "0") != "1"

    def check_numerics(self):
        """Raise like the reference's non-finite guard (gnnmath.py:100-102) if a
        backward scatter saw a non-finite value (flag bit 0), or a contribution
        outdeg * |v| >= 2^42 that the fixed-point accumulator cannot hold (bit 1)."""
        f = int(self.fx_flags.item())
        if f:
            self.fx_flags.zero_()
            if f & 1:
                raise FloatingPointError("non-finite gradient in the transposed aggregation")
            raise FloatingPointError("gradient magnitude beyond the fixed-point accumulator range (2^42)")

    def _save_state(self):
        st = {"flat": self.params.flat.clone(), "md": self.d_maxdelta.clone(),
              "loss": self.loss_arr.clone(), "mdarr": self.md_arr.clone()}
        if self.optimizer == "adam":
            st.update(m=self.adam_m.clone(), v=self.adam_v.clone(), t=self.adam_t.clone())
        if self.hot is not None:
            h = self.hot
            st.update(hits=h.batch_hits.clone(), miss=h.batch_miss.clone(), warm=h.batch_warm.clone(),
                      stats=h.stats.clone())
        return st

    def _restore_state(self, st):
        """The warm-up pass ran one real update; undo it so capture is side-effect free."""
        self.params.flat.copy_(st["flat"])
        self.fx_flags.zero_()  # the warm-up ran on unfed (empty) sample sets
        self.need_tag.fill_(-1)  # ... and tagged vertices for the row accounting
        self.raw_rows_arr.zero_()
        self.cache_hit_arr.zero_()
        self.d_maxdelta.copy_(st["md"])
        self.loss_arr.copy_(st["loss"])
        self.md_arr.copy_(st["mdarr"])
        if self.optimizer == "adam":
            self.adam_m.copy_(st["m"])
            self.adam_v.copy_(st["v"])
            self.adam_t.copy_(st["t"])
        if self.hot is not None:
            h = self.hot
            h.batch_hits.copy_(st["hits"])
            h.batch_miss.copy_(st["miss"])
            h.batch_warm.copy_(st["warm"])
            h.stats.copy_(st["stats"])
        self.enqueue_weight_images()
        torch.cuda.synchronize(self.device)

    def run_step(self, stream=None):
        """Sequential step on the current stream (set 0)."""
        if self.graph is not None:
            self.graph.replay()
        else:
            self.cur = 0
            self.enqueue_step(stream)


class Pipeline:
    """Two-stream software pipeline over batches: the sample half of batch k+1
    runs on ``ss`` while the train half of batch k runs on ``st``; sample set
    k % 2 is reused only after batch k-2 finished training."""

    def __init__(self, engine: TrainEngine):
        self.e = engine
        dev = engine.device
        ps, pt = stream_priorities()
        self.ss = torch.cuda.Stream(device=dev, priority=ps)
        self.st = torch.cuda.Stream(device=dev, priority=pt)
        n = len(engine.sets)
        self.sampled = [torch.cuda.Event() for _ in range(n)]
        self.trained = [None] * n

    def sample(self, k: int, feed):
        """``feed(set_index)`` stages batch k's inputs (on the sampling stream)."""
        e, st = self.e, k % len(self.e.sets)
        self.ss.wait_stream(torch.cuda.current_stream(e.device))
        if self.trained[st] is not None:
            self.ss.wait_event(self.trained[st])
        with torch.cuda.stream(self.ss):
            feed(st)
            if e.g_sample is not None:
                e.g_sample[st].replay()
            else:
                e.cur = st
                e.enqueue_sample_part(self.ss)
                e.cur = 0
            self.sampled[st].record(self.ss)

    def train(self, k: int, before=None):
        """Train batch k; ``before(stream)`` enqueues work that must precede it on
        the training stream (store tags, weight snapshots)."""
        e, st = self.e, k % len(self.e.sets)
        self.st.wait_event(self.sampled[st])
        with torch.cuda.stream(self.st):
            if before is not None:
                before(self.st)
            if e.g_train is not None:
                e.g_train[st].replay()
            else:
                e.cur = st
                e.enqueue_train_part(self.st)
                e.cur = 0
            ev = torch.cuda.Event()
            ev.record(self.st)
            self.trained[st] = ev

    def drain(self):
        torch.cuda.current_stream(self.e.device).wait_stream(self.st)
        torch.cuda.current_stream(self.e.device).wait_stream(self.ss)


def stream_priorities():
    """(sample stream, train stream) priorities of the two-stream pipeline: env
    HG_STREAM_PRIO = "train" gives the training half the higher priority (lower
    number), "sample" the sampling half, default none."""
    mode = os.environ.get("HG_STREAM_PRIO", "")
    hi = torch.cuda.Stream.priority_range()[1] if torch.cuda.is_available() else 0
    if mode == "train":
        return 0, hi
    if mode == "sample":
        return hi, 0
    return 0, 0


class BatchFeeder:
    """Pinned-host -> device staging of per-batch inputs (seed ids, counts and the
    parameter block), ring-buffered so the host never overwrites a slot whose
    copy has not completed."""

    def __init__(self, engine: TrainEngine, slots: int = 4):
        self.e = engine
        cap = engine.batch_cap
        # pinned images of SampleSet.stage (bp | counts | seeds): one H2D copy per batch
        self.stage = [torch.zeros(STAGE_SEEDS + 4 * cap, dtype=torch.uint8).pin_memory() for _ in range(slots)]
        views = [stage_views(t) for t in self.stage]
        self.bp = [v[0] for v in views]
        self.counts = [v[1] for v in views]
        self.seeds = [v[2] for v in views]
        self.events = [None] * slots
        self.k = 0
        self.h2d_bytes = 0

    def feed(self, seeds: np.ndarray, rng_seed: int, reading_batch: int, batch_in_epoch: int, cpu_tag: int = -1,
             table_sel: int = 0, cur_stamp: int = -1, warm: int = 0, n_div: int | None = None,
             set_index: int | None = None):
        k = self.k
        self.k = (k + 1) % len(self.seeds)
        if self.events[k] is not None:
            self.events[k].synchronize()
        n = int(seeds.shape[0])
        if n > self.e.batch_cap:
            raise ValueError("batch larger than the engine's capacity")
        self.seeds[k].numpy()[:n] = seeds
        self.counts[k].numpy()[:] = (n, n if n_div is None else n_div)
        rs = int(rng_seed) & 0xFFFFFFFFFFFFFFFF
        self.bp[k].numpy()[:] = np.array([rs], dtype=np.uint64).view(np.int64)[0], n, reading_batch, \
            batch_in_epoch, cpu_tag, table_sel, cur_stamp, warm
        e = self.e.sets[self.e.cur if set_index is None else set_index]
        nb = STAGE_SEEDS + 4 * n
        e.stage[:nb].copy_(self.stage[k][:nb], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.events[k] = ev
        self.h2d_bytes = nb
