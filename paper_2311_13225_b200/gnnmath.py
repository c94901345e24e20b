"""GCN / mean-SAGE layer math on the GPU (reference gnnmath.py:1-347).

The functional API keeps the reference's signatures (numpy in, numpy out) so
it is a drop-in for parity tests; each call runs the library's kernels:
aggregation K5 (``hg_aggregate_fwd``), transposed aggregation K6
(``hg_aggregate_bwd_scatter``: deterministic fixed-point scatter), dense
transforms K8 on the tensor cores (``hg_gemm_tc`` / ``hg_wgrad_tc``), loss K9
and updates K10.  Arithmetic is
fp32 on device (the reference is fp64); tolerances are stated in the tests.
The training engine (engine.py) runs the same kernels device-resident.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, dense
from .device import pad4, ptr, require_cuda, stream_ptr
from .seeds import derive_seed


class ShapeError(ValueError):
    """gnnmath.py:20-21."""


@dataclass
class ModelParams:
    """gnnmath.py:24-52 (host copy; the engine keeps the device master)."""

    model: str
    dims: list
    weights: list
    version: int = 0

    @property
    def num_layers(self) -> int:
        return len(self.weights)

    def copy(self) -> "ModelParams":
        return ModelParams(self.model, list(self.dims), [[w.copy() for w in l] for l in self.weights], self.version)

    def bottom_weights(self):
        return [w.copy() for w in self.weights[0]]

    def num_elements(self) -> int:
        return sum(w.size for l in self.weights for w in l)


def init_params(model: str, dims, seed: int) -> ModelParams:
    """gnnmath.py:55-71: Glorot uniform from Philox(derive_seed(seed, 7, l, m)).
    Host-side planning: consuming numpy's Philox keeps the initial weights
    identical to the reference's."""
    if model not in ("gcn", "sage"):
        raise ShapeError(f"unknown model {model!r}")
    weights = []
    for l in range(len(dims) - 1):
        fi, fo = dims[l], dims[l + 1]
        lim = np.sqrt(6.0 / (fi + fo))
        layer = []
        for m in range(1 if model == "gcn" else 2):
            gen = np.random.Generator(np.random.Philox(key=derive_seed(seed, 7, l, m)))
            layer.append(gen.uniform(-lim, lim, size=(fi, fo)))
        weights.append(layer)
    return ModelParams(model=model, dims=list(dims), weights=weights)


# ---------------------------------------------------------------------------
# numpy Block -> device slot form
# ---------------------------------------------------------------------------

class DeviceBlock:
    """A reference Block (edges sorted by (dst, src)) in the kernels' slot form."""

    def __init__(self, block, device):
        es = np.asarray(block.edge_src, np.int64)
        ed = np.asarray(block.edge_dst, np.int64)
        n_dst, n_src = int(block.n_dst), int(block.n_src)
        self.n_dst, self.n_src = n_dst, n_src
        cnt = np.bincount(ed, minlength=n_dst).astype(np.int64) if ed.size else np.zeros(n_dst, np.int64)
        f = max(int(cnt.max()) if n_dst else 1, 1)
        starts = np.concatenate([[0], np.cumsum(cnt)[:-1]]) if n_dst else np.zeros(0, np.int64)
        pos = ed * f + (np.arange(ed.size) - starts[ed]) if ed.size else np.zeros(0, np.int64)
        slot_local = np.zeros(max(n_dst * f, 1), np.int32)
        slot_g = np.zeros(max(n_dst * f, 1), np.int32)
        slot_local[pos] = es
        src_g = np.asarray(block.src_vertices, np.int64)
        dst_g = np.asarray(block.dst_vertices, np.int64)
        slot_g[pos] = src_g[es]
        nself = np.bincount(ed[src_g[es] != dst_g[ed]], minlength=n_dst) if ed.size else np.zeros(n_dst)
        outdeg = np.bincount(es, minlength=n_src) if es.size else np.zeros(n_src)
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=device)  # noqa: E731
        self.f = f
        self.counts = t(np.maximum(cnt, 0) if n_dst else [0])
        self.slot_local, self.slot_g = t(slot_local), t(slot_g)
        self.nself, self.outdeg = t(nself if n_dst else [0]), t(outdeg if n_src else [0])
        self.dst = t(dst_g if n_dst else [0])
        self.d_n_dst = t([n_dst])
        self.d_n_src = t([n_src])


def _dev_rows(x, device, ld=None):
    x = np.asarray(x, dtype=np.float32)
    ld = ld or pad4(x.shape[1])
    t = torch.zeros((max(x.shape[0], 1), ld), dtype=torch.float32, device=device)
    t[:x.shape[0], :x.shape[1]] = torch.as_tensor(x, device=device)
    return t


@dataclass
class LayerActivations:
    """gnnmath.py:74-86 (device tensors)."""

    dblock: DeviceBlock
    h_in: torch.Tensor
    agg: torch.Tensor
    out: torch.Tensor
    activation: bool
    d_in: int
    d_out: int
    injected_rows: np.ndarray = None
    inj_dev: torch.Tensor = field(default=None)


def _model_code(model):
    if model not in ("gcn", "sage"):
        raise ShapeError(f"unknown model {model!r}")
    return 0 if model == "sage" else 1


def layer_forward(model: str, block, h_in, layer_weights, activation: bool):
    """gnnmath.py:203-208 -> (h_out numpy float64, cache)."""
    dev = require_cuda()
    h_in_np = np.asarray(h_in)
    if h_in_np.shape[0] != block.n_src:
        raise ShapeError(f"{model} layer: input rows {h_in_np.shape[0]} != block src count {block.n_src}")
    d_in = h_in_np.shape[1]
    if layer_weights[0].shape[0] != d_in or (model == "sage" and layer_weights[1].shape[0] != d_in):
        raise ShapeError(f"{model} layer: weight input dim mismatch")
    d_out = layer_weights[0].shape[1]
    db = DeviceBlock(block, dev)
    hin = _dev_rows(h_in_np, dev)
    out, cache = _layer_forward_dev(model, db, hin, d_in, d_out,
                                    [torch.as_tensor(np.asarray(w, np.float32), device=dev) for w in layer_weights],
                                    activation)
    h = out[:block.n_dst, :d_out].double().cpu().numpy()
    if not np.all(np.isfinite(h)):
        raise FloatingPointError(f"non-finite values in {model} layer output")
    return h, cache


def _layer_forward_dev(model, db, hin, d_in, d_out, W, activation, inj=None):
    dev = hin.device
    s = stream_ptr()
    ld_in, ld_out = hin.shape[1], pad4(d_out)
    n = max(db.n_dst, 1)
    agg = torch.zeros((n, ld_in), dtype=torch.float32, device=dev)
    out = torch.zeros((n, ld_out), dtype=torch.float32, device=dev)
    code = _model_code(model)
    if db.n_dst:
        _lib.call("hg_aggregate_fwd", code, 0, ptr(hin), ld_in, ld_in, ptr(db.dst), ptr(db.d_n_dst), db.n_dst, db.f,
                  ptr(db.counts), ptr(db.slot_g), ptr(db.slot_local), ptr(db.nself), ptr(db.outdeg), ptr(inj), None,
                  0, ptr(agg), ld_in, s)
        if code == 0:  # [h_self | mean] [W_self; W_neigh]
            wst = torch.cat([W[0], W[1]], 0).contiguous()
            dense.fwd(ptr(hin), ld_in, ptr(agg), ld_in, d_in, ptr(wst), d_out, ptr(out), ld_out, ptr(db.d_n_dst),
                      db.n_dst, int(activation), s)
        else:
            dense.fwd(ptr(agg), ld_in, None, 0, d_in, ptr(W[0]), d_out, ptr(out), ld_out, ptr(db.d_n_dst), db.n_dst,
                      int(activation), s)
    cache = LayerActivations(dblock=db, h_in=hin, agg=agg, out=out, activation=activation, d_in=d_in, d_out=d_out)
    return out, cache


def forward_batch(stack, inputs, params: ModelParams, model: str | None = None, inject=None):
    """gnnmath.py:219-247: bottom-up; ``inject`` overwrites bottom OUTPUT rows."""
    dev = require_cuda()
    model = model or params.model
    L = len(stack.blocks)
    if params.num_layers != L:
        raise ShapeError(f"stack has {L} blocks but params {params.num_layers} layers")
    inputs = np.asarray(inputs)
    if inputs.shape[0] != stack.blocks[0].n_src:
        raise ShapeError(f"{model} layer: input rows {inputs.shape[0]} != block src count {stack.blocks[0].n_src}")
    h = _dev_rows(inputs, dev)
    d = inputs.shape[1]
    caches = []
    for l, blk in enumerate(stack.blocks):
        W = [torch.as_tensor(np.asarray(w, np.float32), device=dev) for w in params.weights[l]]
        if W[0].shape[0] != d:
            raise ShapeError(f"{model} layer: weight input dim {W[0].shape[0]} != feature dim {d}")
        db = DeviceBlock(blk, dev)
        if h.shape[0] < blk.n_src:
            raise ShapeError(f"{model} layer: input rows {h.shape[0]} != block src count {blk.n_src}")
        out, c = _layer_forward_dev(model, db, h, d, W[0].shape[1], W, l < L - 1)
        if l == 0 and inject is not None and len(inject[0]):
            idx = np.asarray(inject[0], np.int64)
            vals = np.asarray(inject[1], np.float32)
            out[torch.as_tensor(idx, device=dev), :vals.shape[1]] = torch.as_tensor(vals, device=dev)
            m = np.zeros(blk.n_dst, bool)
            m[idx] = True
            c.injected_rows = m
            c.inj_dev = torch.as_tensor(m.astype(np.uint8), device=dev)
        caches.append(c)
        h = out
        d = W[0].shape[1]
    logits = h[:stack.blocks[-1].n_dst, :d].double().cpu().numpy()
    if not np.all(np.isfinite(logits)):
        raise FloatingPointError("non-finite values in logits")
    return logits, caches


def backward_batch(caches, dlogits, params: ModelParams):
    """gnnmath.py:250-260: reverse mode; dx only above the bottom layer."""
    dev = require_cuda()
    s = stream_ptr()
    L = len(caches)
    d = _dev_rows(np.asarray(dlogits), dev)
    grads = [None] * L
    for l in range(L - 1, -1, -1):
        c = caches[l]
        db = c.dblock
        code = _model_code(params.model)
        W = [torch.as_tensor(np.asarray(w, np.float32), device=dev) for w in params.weights[l]]
        dz = d
        if c.activation:  # d_out * (z > 0): the mask is folded in when d was produced (below)
            pass
        ld_in, ld_out = c.h_in.shape[1], dz.shape[1]
        nsrc = 2 if code == 0 else 1
        g = [torch.zeros((c.d_in, c.d_out), dtype=torch.float32, device=dev) for _ in range(nsrc)]
        ws = torch.zeros(max(dense.wgrad_ws_size(c.d_in, c.d_out, db.n_dst, nsrc), 1), dtype=torch.float32,
                         device=dev)
        if code == 0:  # dW_self = h_self^T dz, dW_neigh = mean^T dz
            dense.wgrad(ptr(c.h_in), ld_in, ptr(c.agg), ld_in, c.d_in, ptr(dz), ld_out, c.d_out, ptr(db.d_n_dst),
                        db.n_dst, ptr(g[0]), ptr(g[1]), ptr(ws), s)
        else:
            dense.wgrad(ptr(c.agg), ld_in, None, 0, c.d_in, ptr(dz), ld_out, c.d_out, ptr(db.d_n_dst), db.n_dst,
                        ptr(g[0]), None, ptr(ws), s)
        grads[l] = [x.double().cpu().numpy() for x in g]
        if l == 0:
            break
        n = max(db.n_dst, 1)
        dagg = torch.zeros((n, ld_in), dtype=torch.float32, device=dev)
        dself = torch.zeros((n, ld_in), dtype=torch.float32, device=dev) if code == 0 else None
        if code == 0:
            dense.dx(ptr(dz), ld_out, c.d_out, ptr(W[0]), c.d_in, ptr(dself), ld_in, ptr(db.d_n_dst), db.n_dst, s)
            dense.dx(ptr(dz), ld_out, c.d_out, ptr(W[1]), c.d_in, ptr(dagg), ld_in, ptr(db.d_n_dst), db.n_dst, s)
        else:
            dense.dx(ptr(dz), ld_out, c.d_out, ptr(W[0]), c.d_in, ptr(dagg), ld_in, ptr(db.d_n_dst), db.n_dst, s)
        below = caches[l - 1]
        dx = torch.zeros((max(db.n_src, 1), ld_in), dtype=torch.float32, device=dev)
        acc = torch.zeros((max(db.n_src, 1), 2 * ld_in), dtype=torch.int64, device=dev)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("hg_aggregate_bwd_scatter", code, ptr(dagg), ld_in, ptr(dself), ld_in, ld_in, ptr(db.dst),
                  ptr(db.d_n_dst), db.n_dst, db.f, ptr(db.counts), ptr(db.slot_g), ptr(db.slot_local),
                  ptr(db.nself), ptr(db.outdeg), ptr(db.d_n_src), db.n_src,
                  ptr(below.out) if below.activation else None, ld_in, ptr(below.inj_dev), ptr(acc), ptr(dx), ld_in,
                  ptr(flags), s)
        if int(flags.item()):  # gnnmath.py:100-102 (non-finite), or the fixed-point range guard
            raise FloatingPointError(f"{params.model} backward: transposed aggregation flagged {int(flags.item())}")
        d = dx
    return grads


def loss_and_grad(logits, labels):
    """gnnmath.py:263-274 on device (fp32): (mean CE, dlogits)."""
    dev = require_cuda()
    lg = np.asarray(logits)
    n, C = lg.shape
    z = _dev_rows(lg, dev)
    lab = torch.as_tensor(np.asarray(labels, np.int32), device=dev)
    dl = torch.zeros_like(z)
    loss = torch.zeros(1, dtype=torch.float32, device=dev)
    rows = torch.zeros(max(n, 1) + 1, dtype=torch.float32, device=dev)
    _lib.call("hg_softmax_xent", ptr(z), z.shape[1], C, None, n, ptr(lab), None, None, ptr(dl), z.shape[1], ptr(loss),
              ptr(rows), stream_ptr())
    return float(loss.item()), dl[:n, :C].double().cpu().numpy()


def sgd_step(params: ModelParams, grads, lr: float) -> ModelParams:
    """gnnmath.py:277-283 (device update of each matrix, version += 1)."""
    dev = require_cuda()
    for lw, lg in zip(params.weights, grads):
        for i, (w, g) in enumerate(zip(lw, lg)):
            dw = torch.as_tensor(np.asarray(w, np.float32).ravel(), device=dev)
            dg = torch.as_tensor(np.asarray(g, np.float32).ravel(), device=dev)
            _lib.call("hg_sgd", ptr(dw), ptr(dg), dw.numel(), float(lr), None, stream_ptr())
            lw[i] = dw.double().cpu().numpy().reshape(w.shape)
    params.version += 1
    return params


@dataclass
class AdamState:
    """gnnmath.py:286-290."""

    m: list = field(default_factory=list)
    v: list = field(default_factory=list)
    t: int = 0


def adam_step(params: ModelParams, grads, lr: float, state: AdamState, beta1=0.9, beta2=0.999, eps=1e-8):
    """gnnmath.py:293-312 on device."""
    dev = require_cuda()
    if not state.m:
        state.m = [[np.zeros_like(w) for w in l] for l in params.weights]
        state.v = [[np.zeros_like(w) for w in l] for l in params.weights]
    state.t += 1
    t_dev = torch.tensor([state.t - 1], dtype=torch.int32, device=dev)
    for li, (lw, lg) in enumerate(zip(params.weights, grads)):
        for wi, (w, g) in enumerate(zip(lw, lg)):
            f = lambda a: torch.as_tensor(np.asarray(a, np.float32).ravel(), device=dev)  # noqa: E731
            dw, dg, dm, dv = f(w), f(g), f(state.m[li][wi]), f(state.v[li][wi])
            t_dev.fill_(state.t - 1)
            _lib.call("hg_adam", ptr(dw), ptr(dg), ptr(dm), ptr(dv), dw.numel(), float(lr), beta1, beta2, eps,
                      ptr(t_dev), None, stream_ptr())
            lw[wi] = dw.double().cpu().numpy().reshape(w.shape)
            state.m[li][wi] = dm.double().cpu().numpy().reshape(w.shape)
            state.v[li][wi] = dv.double().cpu().numpy().reshape(w.shape)
    params.version += 1
    return params
