"""Per-layer execution-mode protocol of the reference (unet.py:430-663), device-backed.

`UNet.forward(latent, t, text_emb, mode)` calls only `mode.conv / mode.norm /
mode.self_attn / mode.cross_attn` per layer (unet.py:434-458), exactly like the
reference, so callers that drive single steps with DenseMode / ControlledMode /
SparseMode (e.g. the reference's test_unet.py) work unchanged. Each method runs
the libfisedit kernels through the op-level API (`ops.py`) with reference
semantics on full maps; the glue between layers (time-bias add, SiLU, residual
adds, 2x2 average pool, nearest upsample, skip concat) runs on the GPU too.

This is the API-compatible per-layer path. The fast path — `generate_dense` /
`detect_mask` / `edit` — executes the same math as whole-step CUDA graphs with
select-on-read (engine.py).
"""

from __future__ import annotations

import math
from collections import defaultdict

import numpy as np
import torch

from . import _lib as L
from . import ops
from .cache import Role
from .engine import DRef, _pad
from .errors import ContractViolation
from .model import NORM_EPS
from .sparse import SparseLayerContext
from .tensors import ConvWeights, macs_attention, macs_conv, macs_linear


class _MacsCounter:
    def __init__(self):
        self.per_layer = defaultdict(int)

    def add(self, layer_id, macs):
        self.per_layer[layer_id] += macs

    @property
    def total(self):
        return sum(self.per_layer.values())


# ---------------------------------------------------------------------------
# layer objects with the reference's attributes (unet.py:262-288)
# ---------------------------------------------------------------------------

class ConvLayer:
    def __init__(self, info, w, b):
        self.info, self.weights = info, ConvWeights(w, b, padding=1)


class NormLayer:
    def __init__(self, info, gamma, beta):
        self.info, self.gamma, self.beta = info, gamma, beta


class SelfAttnLayer:
    def __init__(self, info, wq, wk, wv):
        self.info, self.wq, self.wk, self.wv = info, wq, wk, wv
        self.scale = 1.0 / math.sqrt(info.channels)


class CrossAttnLayer:
    def __init__(self, info, wq, wk_text, wv_text):
        self.info, self.wq, self.wk_text, self.wv_text = info, wq, wk_text, wv_text
        self.scale = 1.0 / math.sqrt(info.channels)


def make_layers(host_layers):
    out = {}
    for hl in host_layers:
        i, p = hl.info, hl.params
        if i.kind == "conv":
            out[i.layer_id] = ConvLayer(i, p["weight"], p["bias"])
        elif i.kind == "norm":
            out[i.layer_id] = NormLayer(i, p["gamma"], p["beta"])
        elif i.kind == "self_attn":
            out[i.layer_id] = SelfAttnLayer(i, p["wq"], p["wk"], p["wv"])
        else:
            out[i.layer_id] = CrossAttnLayer(i, p["wq"], p["wk_text"], p["wv_text"])
    return out


# ---------------------------------------------------------------------------
# glue on device (unet.py:291-302,435,446,456-457)
# ---------------------------------------------------------------------------

def _dev(x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def silu(x: np.ndarray) -> np.ndarray:
    v = _dev(x).double()
    return (v / (1.0 + torch.exp(-v))).float().cpu().numpy()


def add(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    return (_dev(a) + _dev(b)).cpu().numpy()


def avgpool2(x: np.ndarray) -> np.ndarray:
    t = _dev(x)
    s = (t[:, :, 0::2, 0::2] + t[:, :, 0::2, 1::2]) + (t[:, :, 1::2, 0::2] + t[:, :, 1::2, 1::2])
    return (s * 0.25).cpu().numpy()


def upsample_concat(x: np.ndarray, skip: np.ndarray) -> np.ndarray:
    u = _dev(x).repeat_interleave(2, dim=2).repeat_interleave(2, dim=3)
    return torch.cat([u, _dev(skip)], dim=1).cpu().numpy()


def text_kv(layer: CrossAttnLayer, text_emb: np.ndarray):
    """unet.py:476-479 (f32 GEMMs on device)."""
    e = _dev(text_emb.astype(np.float32))
    lz = ops._lz()
    nt = text_emb.shape[0]
    c = layer.info.channels
    k = torch.empty((nt, c), dtype=torch.float32, device="cuda")
    v = torch.empty((nt, c), dtype=torch.float32, device="cuda")
    lz.gemm(nt, c, e.shape[1], a=DRef(e), b=DRef(_dev(layer.wk_text.T.copy())), d=DRef(k), splits=1)
    lz.gemm(nt, c, e.shape[1], a=DRef(e), b=DRef(_dev(layer.wv_text.T.copy())), d=DRef(v), splits=1)
    return k.cpu().numpy(), v.cpu().numpy()


def _cross_macs(layer, q_tokens, n_text, text_dim):
    c = layer.info.channels
    return macs_linear(q_tokens, c, c) + 2 * macs_linear(n_text, text_dim, c) + macs_attention(q_tokens, n_text, c)


# ---------------------------------------------------------------------------
# modes
# ---------------------------------------------------------------------------

class DenseMode:
    """unet.py:491-536; optionally records activations via recorder(layer_id, role, payload)."""

    def __init__(self, groups: int, macs=None, recorder=None):
        self.groups, self.macs, self.recorder = groups, macs, recorder

    def _record(self, lid, role, payload):
        if self.recorder is not None:
            self.recorder(lid, role, payload)

    def conv(self, layer, x):
        y = ops.conv2d(x, layer.weights)
        if self.macs:
            self.macs.add(layer.info.layer_id, macs_conv(layer.weights, y.shape[2] * y.shape[3]))
        self._record(layer.info.layer_id, Role.LAYER_OUTPUT, y)
        return y

    def norm(self, layer, x):
        y, mean, var = ops.group_norm(x, self.groups, layer.gamma, layer.beta, NORM_EPS)
        self._record(layer.info.layer_id, Role.NORM_MEAN, mean)
        self._record(layer.info.layer_id, Role.NORM_VAR, var)
        self._record(layer.info.layer_id, Role.LAYER_OUTPUT, y)
        return y

    def self_attn(self, layer, x):
        y = ops.dense_self_attention(x, layer.wq, layer.wk, layer.wv, layer.scale)
        if self.macs:
            hw, c = layer.info.h * layer.info.w, layer.info.channels
            self.macs.add(layer.info.layer_id, 3 * macs_linear(hw, c, c) + macs_attention(hw, hw, c))
        self._record(layer.info.layer_id, Role.LAYER_OUTPUT, y)
        return y

    def cross_attn(self, layer, x, text_emb):
        k, v = text_kv(layer, text_emb)
        y, scores = ops.dense_cross_attention(x, k, v, layer.wq, layer.scale)
        if self.macs:
            self.macs.add(layer.info.layer_id,
                          _cross_macs(layer, layer.info.h * layer.info.w, text_emb.shape[0], text_emb.shape[1]))
        self._record(layer.info.layer_id, Role.CROSS_ATTN_MAP, scores)
        self._record(layer.info.layer_id, Role.LAYER_OUTPUT, y)
        return y


class ControlledMode(DenseMode):
    """Shared-token columns pinned to the cached maps, rows renormalised (unet.py:539-575);
    the pinning runs in fis_softmax."""

    def __init__(self, config, cached_maps, shared, n_new, macs=None):
        super().__init__(config.groups, macs=macs)
        self.cached_maps, self.shared, self.n_new = cached_maps, shared, n_new

    def cross_attn(self, layer, x, text_emb):
        k, v = text_kv(layer, text_emb)
        cached = np.ascontiguousarray(self.cached_maps[layer.info.layer_id], dtype=np.float32)
        n, c, h, w = x.shape
        lz = ops._lz()
        nt = k.shape[0]
        verbatim = len(self.shared.pairs) == self.n_new and self.n_new == cached.shape[1]
        q = ops._proj(ops._nhwc(x), None, h * w, ops._dev2d(layer.wq.T))
        S = torch.empty((h * w, nt), dtype=torch.float32, device="cuda")
        P = torch.zeros((h * w, _pad(nt)), dtype=torch.float32, device="cuda")
        lz.gemm(h * w, nt, c, a=DRef(q), b=DRef(ops._dev2d(k)), d=DRef(S))
        cached_d = ops._dev2d(cached)
        pairs = None
        if self.shared.pairs and not verbatim:
            po = torch.tensor([p[0] for p in self.shared.pairs], dtype=torch.int32, device="cuda")
            pn = torch.tensor([p[1] for p in self.shared.pairs], dtype=torch.int32, device="cuda")
            pairs = (po, pn)
        lz.softmax(h * w, nt, _pad(nt), DRef(S), layer.scale, DRef(P), None, cached=DRef(cached_d),
                   verbatim=verbatim, pairs=pairs)
        out = ops._apply(P, ops._vt(ops._dev2d(v), nt), h * w, nt)
        if self.macs:
            self.macs.add(layer.info.layer_id, _cross_macs(layer, h * w, text_emb.shape[0], text_emb.shape[1]))
        return ops._nchw(out, c, h, w)


class SparseMode:
    """Gated layers run the sparse ops against their pyramid level; others run dense (unet.py:578-663)."""

    def __init__(self, config, pyramid, plans, contexts, macs=None, pool=None):
        self.config, self.pyramid, self.plans, self.contexts = config, pyramid, plans, contexts
        self.macs, self.pool = macs, pool

    def _mask(self, info):
        return self.pyramid.levels[info.level]

    def conv(self, layer, x):
        info = layer.info
        if not info.gated:
            if self.macs:
                self.macs.add(info.layer_id, macs_conv(layer.weights, info.h * info.w))
            return ops.conv2d(x, layer.weights)
        plan = self.plans[info.level]
        y = ops.sparse_conv(x, layer.weights, plan, self.contexts[info.layer_id], self._mask(info), pool=self.pool)
        if self.macs:
            self.macs.add(info.layer_id, macs_conv(layer.weights, plan.cost))
        return y

    def norm(self, layer, x):
        info = layer.info
        if not info.gated:
            y, _, _ = ops.group_norm(x, self.config.groups, layer.gamma, layer.beta, NORM_EPS)
            return y
        return ops.sparse_group_norm(x, self.contexts[info.layer_id], layer.gamma, layer.beta, NORM_EPS,
                                     self._mask(info))

    def self_attn(self, layer, x):
        info = layer.info
        if not info.gated:
            if self.macs:
                hw, c = info.h * info.w, info.channels
                self.macs.add(info.layer_id, 3 * macs_linear(hw, c, c) + macs_attention(hw, hw, c))
            return ops.dense_self_attention(x, layer.wq, layer.wk, layer.wv, layer.scale)
        mask = self._mask(info)
        y = ops.sparse_self_attention(x, layer.wq, layer.wk, layer.wv, layer.scale, self.contexts[info.layer_id], mask)
        if self.macs:
            a, c = mask.active_count, info.channels
            self.macs.add(info.layer_id, 3 * macs_linear(a, c, c) + macs_attention(a, a, c))
        return y

    def cross_attn(self, layer, x, text_emb):
        info = layer.info
        k, v = text_kv(layer, text_emb)
        if not info.gated:
            y, _ = ops.dense_cross_attention(x, k, v, layer.wq, layer.scale)
            if self.macs:
                self.macs.add(info.layer_id, _cross_macs(layer, info.h * info.w, text_emb.shape[0], text_emb.shape[1]))
            return y
        mask = self._mask(info)
        y = ops.sparse_cross_attention(x, k, v, layer.wq, layer.scale, self.contexts[info.layer_id], mask)
        if self.macs:
            self.macs.add(info.layer_id, _cross_macs(layer, mask.active_count, text_emb.shape[0], text_emb.shape[1]))
        return y


def sparse_contexts(unet, store, t):
    """Per gated layer: cached output and (norm) statistics of step t (unet.py:781-797)."""
    contexts = {}
    for info in unet.layers:
        if not info.gated:
            continue
        ctx = SparseLayerContext(step=t, layer_id=info.layer_id,
                                 cached_output=store.get((t, info.layer_id, Role.LAYER_OUTPUT)),
                                 mask_level=info.level, resolution_gate=True)
        if info.kind == "norm":
            ctx.cached_mean = store.get((t, info.layer_id, Role.NORM_MEAN))
            ctx.cached_var = store.get((t, info.layer_id, Role.NORM_VAR))
        contexts[info.layer_id] = ctx
    return contexts


def forward(unet, latent: np.ndarray, t: int, text_emb: np.ndarray, mode) -> np.ndarray:
    """One denoiser evaluation through the per-layer mode protocol (unet.py:430-458)."""
    cfg = unet.config
    if not 1 <= t <= cfg.steps:
        raise ContractViolation(f"step {t} outside 1..{cfg.steps}")
    Ls = unet.layer_objects()
    topo = unet.topo
    x = mode.conv(Ls[topo["stem"]], latent)
    x = add(x, unet.time_bias[t][None, :, None, None])
    skips = []

    def block(blk, x):
        y = mode.conv(Ls[blk["conv"]], x)
        y = silu(mode.norm(Ls[blk["norm"]], y))
        y = add(y, mode.self_attn(Ls[blk["self_attn"]], y))
        return add(y, mode.cross_attn(Ls[blk["cross_attn"]], y, text_emb))

    for l in range(cfg.levels):
        for blk in topo["enc"][l]:
            x = block(blk, x)
        if l < cfg.levels - 1:
            skips.append(x)
            x = mode.conv(Ls[topo["down"][l]], avgpool2(x))
    for l in range(cfg.levels - 2, -1, -1):
        x = mode.conv(Ls[topo["fuse"][l]], upsample_concat(x, skips[l]))
        for blk in topo["dec"][l]:
            x = block(blk, x)
    return mode.conv(Ls[topo["out"]], x)
