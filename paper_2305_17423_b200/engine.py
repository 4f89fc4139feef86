"""Device engine: weights in HBM, the per-generation HBM arena, and the dense and
sparse (select-on-read) step programs launched through libfisedit.

Layout: every feature map is NHWC-flattened `[pixels, C]`
(channels contiguous). Per-step cache slabs are `[T+1, pixels, C]` tensors; a
kernel addresses slab[t] as `base + t*stride` with t read from a device step
counter, so a captured CUDA graph of one step replays every step.

Sparse step: at a gated level the fresh values of a feature
live only at the level's active pixels, in a compact `[n_active, C]` buffer in
row-major active order; a read of pixel q selects `index[q] >= 0 ? fresh :
cache[t][q]`. Nothing is ever copied from the cache; the cache is never
mutated by an edit (no compaction, cache.py:538-579 is a numerical no-op).
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .errors import CacheMissError, ContractViolation
from .model import (NORM_EPS, UNetConfig, build_registry, embed_ids, initial_latent_np, lcs_pairs, step_program,
                    step_scale)

_ESIZE = {torch.float32: 4, torch.bfloat16: 2}
PRECISIONS = ("fp32", "tf32x3", "bf16")


class DRef:
    """A device buffer as the kernels see it: base (+byte offset) and a per-step stride."""

    __slots__ = ("t", "ss", "off", "ld")

    def __init__(self, t: torch.Tensor, ss: int = 0, off: int = 0, ld: int | None = None):
        self.t, self.ss, self.off = t, ss, off
        self.ld = ld if ld is not None else (t.stride(-2) if t.dim() >= 2 else 1)

    def ref(self) -> L.Ref:
        return L.Ref(self.t.data_ptr() + self.off, self.ss, self.ld, L.dt(self.t))

    def cols(self, c0: int) -> "DRef":
        """View starting at column c0 (same ld)."""
        return DRef(self.t, self.ss, self.off + c0 * _ESIZE[self.t.dtype], self.ld)


def slab(t: torch.Tensor, prev: bool = False) -> DRef:
    """Per-step slab [T+1, ...] addressed as slab[t] (or slab[t-1] with prev=True)."""
    ss = t.stride(0) * t.element_size()
    return DRef(t[0], ss, -ss if prev else 0, ld=t.stride(1) if t.dim() >= 3 else 1)


NULL = L.Ref(None, 0, 0, 0)


def _r(x):
    return x.ref() if x is not None else NULL


@dataclass
class FeatVal:
    """Runtime value of a feature: full map (index None) or compact fresh rows + select-on-read cache."""

    fresh: DRef
    level: int
    c: int
    index: torch.Tensor | None = None
    cache: DRef | None = None


class Weights:
    """Device copies of the seeded parameters in GEMM-ready layouts."""

    def __init__(self, layers, topo, config: UNetConfig, act: torch.dtype, dev):
        self.conv, self.norm, self.sa, self.ca = {}, {}, {}, {}
        f32 = torch.float32
        for hl in layers:
            i, p = hl.info, hl.params
            if i.kind == "conv":
                w = p["weight"]  # (co, ci, 3, 3) -> B[co, (ky,kx,ci)]
                b = torch.from_numpy(np.ascontiguousarray(w.transpose(0, 2, 3, 1).reshape(w.shape[0], -1)))
                self.conv[i.layer_id] = (b.to(dev, act), torch.from_numpy(p["bias"]).to(dev, f32), hl.c_in)
            elif i.kind == "norm":
                self.norm[i.layer_id] = (torch.from_numpy(p["gamma"]).to(dev, f32), torch.from_numpy(p["beta"]).to(dev, f32))
            elif i.kind == "self_attn":
                # scores reassociated: (s wq)(s wk)^T = (s (wq wk^T)) s^T, so the projection GEMM makes
                # Q' = s (wq wk^T) and V only (B = [(wq wk^T)^T; wv^T], [2C, C]; the product in f64) and
                # the keys are s itself: 2/3 of the QKV weights and FLOPs
                mqk = (p["wq"].astype(np.float64) @ p["wk"].astype(np.float64).T).T
                wqv = np.concatenate([mqk, p["wv"].T.astype(np.float64)], axis=0).astype(np.float32)  # [2C, C]
                self.sa[i.layer_id] = (torch.from_numpy(np.ascontiguousarray(wqv)).to(dev, act),
                                       1.0 / math.sqrt(i.channels))
            else:
                # wq [C_in, C_out] as the reference stores it (q = g . wq): the per-edit score matrix
                # M^T = K . wq^T... see Engine.text_kv
                # text K / V weights: fp32 in the fp32 / tf32x3 modes; bf16 (like every other weight)
                # in bf16 mode so the per-edit text K / V GEMMs run on the tensor cores
                wt = f32 if act == f32 else act
                self.ca[i.layer_id] = (torch.from_numpy(np.ascontiguousarray(p["wq"])).to(dev, act),
                                       torch.from_numpy(np.ascontiguousarray(p["wk_text"].T)).to(dev, wt),
                                       torch.from_numpy(np.ascontiguousarray(p["wv_text"].T)).to(dev, wt),
                                       1.0 / math.sqrt(i.channels))
        self.time_bias = torch.from_numpy(topo["time_bias"]).to(dev, f32)


def _pad(n, m=16):
    return (n + m - 1) // m * m


class Launcher:
    """Kernel launch helpers (GEMM / softmax / GN / pool / materialise) independent of a model."""

    def __init__(self, precision: str = "fp32", device=None):
        L.require_cuda()
        if precision not in PRECISIONS:
            raise ContractViolation(f"precision must be one of {PRECISIONS}, got {precision!r}")
        self.precision = precision
        self.dev = torch.device(device or "cuda")
        # fp32: fp32 operands, SIMT FFMA (the reference numerics, parity mode); tf32x3: fp32 operands on
        # the tensor cores as 3xTF32 (big*big + big*small + small*big, fp32 accumulate); bf16: perf mode
        self.act = torch.bfloat16 if precision == "bf16" else torch.float32
        self.gemm_impl = {"fp32": 1, "tf32x3": 3, "bf16": 0}[precision]
        self.sms = L.lib().fis_device_sm_count()
        # namespace of the request being driven: requests that run concurrently (one CUDA stream
        # each) own separate scratch activations, split-K workspaces and step counters
        self.ns = 0
        self._ns_state = {}
        # stacked images of the step being launched (BatchedSparsePlan: R requests as one batch)
        self.batch = 1
        self.launches = 0
        # when a list: every launch appends {"op", "kernels", ...shape} (bench.py maps profiled
        # kernels of a step back to ops with it)
        self.op_log: list | None = None
        self._scratch = {}
        # tcgen05 fused attention (csrc/fis_attn.cu: TMA-fed, log2 softmax, resident S for <= 256
        # keys, P shared across value slices) instead of S GEMM -> softmax -> P.V GEMM: C2 sparse
        # step 1.416 vs 1.506 ms, dense step 2.83 vs 3.30 ms (r01). Stacked requests always use it
        # (segments); FIS_FUSED_ATTN=0 restores the three-launch path for single sequences.
        self.fused_attn = os.environ.get("FIS_FUSED_ATTN", "1") == "1"
        # gather lists (rows / pixel->row maps) are written once per edit, before any step runs
        # (DevicePlan syncs), so GEMMs may read them before the programmatic-launch wait
        self.static_meta = False
        self.groups = 1
        self.step_scale_value = 1.0
        self._kv_graphs = {}  # (n_text, text_dim) -> (graph, embedding buffer, outputs) of text_kv
        self._kv_seen = {}    # prompt shapes seen once (captured on the second use)

    def _call(self, name, args, b_static=False):
        L.call(name, args)

    def _count(self, name, kernels=1, **info):
        self.launches += kernels
        if self.op_log is not None:
            self.op_log.append(dict(op=name, kernels=kernels, **info))

    def _state(self):
        st = self._ns_state.get(self.ns)
        if st is None:
            st = {"step": torch.zeros(1, dtype=torch.int32, device=self.dev),
                  "ws": torch.zeros(1, dtype=torch.float32, device=self.dev),
                  "counters": torch.zeros(1 << 16, dtype=torch.int32, device=self.dev)}
            self._ns_state[self.ns] = st
        return st

    @property
    def step_dev(self) -> torch.Tensor:
        """Device step counter t of the current namespace (kernels read the step from it)."""
        return self._state()["step"]

    @property
    def _ws(self) -> torch.Tensor:
        return self._state()["ws"]

    @property
    def _counters(self) -> torch.Tensor:
        return self._state()["counters"]

    def scratch(self, name, shape, dtype=None, zero=False):
        key = (self.ns, name, tuple(shape), dtype or self.act)
        t = self._scratch.get(key)
        if t is None:
            t = (torch.zeros if zero else torch.empty)(shape, dtype=dtype or self.act, device=self.dev)
            self._scratch[key] = t
        return t


    WS_FLOATS = (1 << 25) + 1024  # 128 MB split-K workspace per namespace; the split choice respects ws_floats

    def _ensure_ws(self, floats):
        # allocated once at its cap and never replaced: captured CUDA graphs hold its raw pointer
        if self._ws.numel() < self.WS_FLOATS:
            self._state()["ws"] = torch.empty(self.WS_FLOATS, dtype=torch.float32, device=self.dev)

    def _splits(self, m, n, k):
        tiles = ((m + 63) // 64) * ((n + 63) // 64)
        ktiles = (k + 15) // 16
        if tiles >= self.sms or ktiles < 32:
            return 1
        s = min(max(1, (2 * self.sms) // tiles), ktiles // 16, 32)
        return max(1, s)

    def gemm(self, m, n, k, *, a=None, rows=None, srcs=None, out_hw=None, b: DRef, d: DRef, alpha=1.0, bias=None,
             bias2=None, pre=None, epi=L.EPI_NONE, gn=None, lat=None, res=None, d_trans=False, splits=None,
             n_split=0, d2=None, d2_trans=False, b_static=False, d_rows=None, m_halo=False, log_level=None):
        """b_static: B is not produced inside the step (weights, per-edit text K/V)."""
        if m == 0:
            return
        g = L.GemmArgs()
        g.m, g.n, g.k = m, n, k
        if srcs is not None:
            g.a_mode = L.A_CONV3X3
            g.nsrc = len(srcs)
            for i, s in enumerate(srcs):
                g.src[i] = s
            g.out_h, g.out_w = out_hw
        else:
            g.a_mode = L.A_ROWS
            g.a = a.ref()
        g.rows = L.ptr(rows)
        g.d_rows = L.ptr(d_rows)
        g.m_halo = 1 if m_halo else 0
        g.b = b.ref()
        g.alpha = alpha
        g.bias = L.ptr(bias)
        g.bias2 = _r(bias2)
        g.pre = _r(pre)
        g.epi = epi
        if gn is not None:
            mean, var, gamma, beta, groups = gn
            g.gn_mean, g.gn_var = mean.ref(), var.ref()
            g.gamma, g.beta, g.groups, g.eps = L.ptr(gamma), L.ptr(beta), groups, NORM_EPS
        g.lat = _r(lat)
        g.step_scale = self.step_scale_value
        g.res = _r(res)
        g.d = d.ref()
        g.d_trans = 1 if d_trans else 0
        if n_split:
            g.n_split, g.d2, g.d2_trans = n_split, d2.ref(), 1 if d2_trans else 0
        s = 0 if splits is None else splits  # 0: the library picks split-K from the tile shape
        self._ensure_ws((32 if s == 0 else s) * m * n)
        g.ws, g.ws_floats = L.ptr(self._ws), self._ws.numel()
        g.counters = L.ptr(self._counters)
        g.splits = s
        g.step = L.ptr(self.step_dev)
        g.impl = self.gemm_impl
        g.static_meta = 1 if self.static_meta else 0
        self.last_gemm = g  # inspected by tests (fis_gemm_kernel_kind)
        self._call("fis_gemm", g, b_static)
        self._count("fis_gemm", m=m, n=n, k=k, gathered=rows is not None and srcs is not None, conv=srcs is not None,
                    level=log_level, halo=bool(m_halo))

    def softmax(self, rows, cols, pad_cols, s: DRef, scale, p: DRef, map_: DRef | None = None, cached=None,
                verbatim=False, pairs=None):
        a = L.SoftmaxArgs()
        a.rows, a.cols, a.pad_cols = rows, cols, pad_cols
        a.s, a.scale, a.p, a.map = s.ref(), scale, p.ref(), _r(map_)
        a.cached = _r(cached)
        a.verbatim = 1 if verbatim else 0
        if pairs is not None and not verbatim:
            po, pn = pairs
            a.npairs, a.pair_old, a.pair_new = po.numel(), L.ptr(po), L.ptr(pn)
        a.step = L.ptr(self.step_dev)
        self._call("fis_softmax", a)
        self._count("fis_softmax", rows=rows, cols=cols)

class Engine(Launcher):
    """One model (config + precision) resident on one GPU."""

    def __init__(self, config: UNetConfig, precision: str = "fp32", device=None):
        super().__init__(precision, device)
        self.static_meta = True
        self.config = config
        self.groups = config.groups
        self.step_scale_value = float(step_scale(config))
        self.layers, self.topo = build_registry(config)
        self.info = {hl.info.layer_id: hl.info for hl in self.layers}
        self.prog, self.feats = step_program(config, self.topo)
        self.W = Weights(self.layers, self.topo, config, self.act, self.dev)
        self.gated = [config.latent_h * config.latent_w >> (2 * l) >= config.gate_fraction * config.latent_h * config.latent_w
                      for l in range(config.levels)]

    # ------------------------------------------------------------------ helpers
    def hw(self, level):
        return (self.config.latent_h >> level) * (self.config.latent_w >> level)

    def cap(self, level):
        """Row capacity of a level's activations: its pixels times the stacked images."""
        return self.hw(level) * self.batch

    def grid(self, level):
        return self.config.latent_h >> level, self.config.latent_w >> level

    def src(self, fv: FeatVal, up=False):
        h, w = self.grid(fv.level)
        if fv.index is not None and fv.cache is None:
            raise CacheMissError("?", "?", "feature cache")
        return L.Src(fv.fresh.ref(), _r(fv.cache) if fv.index is not None else NULL,
                     L.ptr(fv.index) if fv.index is not None else None, h, w, fv.c, 1 if up else 0)

    # ------------------------------------------------------------ text K/V
    def text_kv(self, text_emb: np.ndarray):
        """Per cross layer, once per prompt: text K [n_text, C] and V^T [C, pad16(n_text)]
        (unet.py:476-479) and the score matrix M^T = K . wq^T [n_text, C].

        Cross attention reassociates its scores: (x wq) K^T = x (wq K^T) = x M, so the step feeds
        the layer input x straight into the attention kernel with M^T as its key matrix and skips
        the per-step query projection (one launch and a C x C GEMM per cross layer and step).

        From the second prompt of a given length on, the 3 GEMMs x cross layers run as one captured
        CUDA graph per prompt length (the Python launch overhead of ~42 GEMM calls was ~4.5 ms of
        every edit); every call copies the new embeddings in, replays, and returns fresh copies."""
        emb_h = torch.from_numpy(np.ascontiguousarray(text_emb, dtype=np.float32))
        if os.environ.get("FIS_KV_GRAPH", "1") == "0":
            return self._text_kv(emb_h.to(self.dev))
        key = tuple(emb_h.shape)
        ent = self._kv_graphs.get(key)
        if ent is None and self._kv_seen.get(key, 0) == 0:
            # first prompt of this length: eager (a one-off length does not pay a capture)
            self._kv_seen[key] = 1
            return self._text_kv(emb_h.to(self.dev))
        if ent is None:
            emb_buf = emb_h.to(self.dev)
            self._text_kv(emb_buf)  # warm-up outside the capture
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            import gc
            gc_on = gc.isenabled()
            gc.disable()
            try:
                # capture_begin / capture_end directly: torch.cuda.graph() empties the caching
                # allocator before every capture (cudaFree of every cached block: up to ~0.5 s
                # with a large arena resident, measured in edit_batch)
                with torch.cuda.stream(s):
                    g.capture_begin()
                    try:
                        _, flat = self._text_kv(emb_buf, want_flat=True)
                    finally:
                        g.capture_end()
            finally:
                if gc_on:
                    gc.enable()
            torch.cuda.current_stream().wait_stream(s)
            ent = self._kv_graphs[key] = (g, emb_buf, flat)
        g, emb_buf, flat = ent
        emb_buf.copy_(emb_h)
        g.replay()
        # the outputs live in one flat buffer: one copy gives the caller its own K / V^T / M^T (the
        # next replay overwrites the graph's buffer; 48 per-tensor clones cost ~1 ms per edit)
        return self._kv_views(flat.clone(), emb_h.shape[0])

    def _kv_layout(self, nt):
        """Element offsets of every cross layer's K [nt, C], V^T [C, pad16(nt)] and M^T [nt, C] in
        one flat buffer (each view 128-byte aligned), and the buffer's length."""
        lay, off = [], 0
        for lid, (wq, _, _, _) in self.W.ca.items():
            c = wq.shape[0]
            views = []
            for shape in ((nt, c), (c, _pad(nt)), (nt, c)):
                views.append((off, shape))
                off += (shape[0] * shape[1] + 63) // 64 * 64
            lay.append((lid, views))
        return lay, off

    def _kv_views(self, flat, nt):
        out = {}
        for lid, views in self._kv_layout(nt)[0]:
            k, vt, mt = (flat[o:o + sh[0] * sh[1]].view(sh) for o, sh in views)
            out[lid] = (k, vt, None, mt)
        return out

    def _text_kv(self, emb: torch.Tensor, want_flat: bool = False):
        nt = emb.shape[0]
        # bf16 mode: the embeddings as bf16 operands -> tcgen05 split-K GEMMs (fp32 embeddings would
        # take the SIMT kernel: ~100 us per layer GEMM); fp32 / tf32x3 keep the unsplit fp32 path
        bf = self.act == torch.bfloat16
        if bf:
            emb = emb.to(torch.bfloat16)
        sp = None if bf else 1
        # every output in one zeroed flat buffer (V^T's pad columns stay zero)
        flat = torch.zeros(self._kv_layout(nt)[1], dtype=self.act, device=self.dev)
        out = self._kv_views(flat, nt)
        for lid, (wq, wk, wv, scale) in self.W.ca.items():
            c = wq.shape[0]
            k, vt, _, mt = out[lid]
            self.gemm(nt, c, emb.shape[1], a=DRef(emb), b=DRef(wk), d=DRef(k), splits=sp)
            self.gemm(nt, c, emb.shape[1], a=DRef(emb), b=DRef(wv), d=DRef(vt), d_trans=True, splits=sp)
            self.gemm(nt, c, c, a=DRef(k), b=DRef(wq), d=DRef(mt), splits=sp)
        return (out, flat) if want_flat else out

    def text_kv_stacked(self, text_embs):
        """Text K / V^T of R prompts computed as ONE GEMM pair per cross layer over the stacked
        embeddings (each prompt padded to pad16(max tokens) zero rows, so the pad keys are zero):
        returns ({lid: (K [R*ks, C], V^T [C, R*ks], None)}, key segments int32 [2R], max tokens)."""
        R = len(text_embs)
        nts = [e.shape[0] for e in text_embs]
        ks = _pad(max(nts))
        emb = np.zeros((R * ks, text_embs[0].shape[1]), dtype=np.float32)
        for r, e in enumerate(text_embs):
            emb[r * ks: r * ks + nts[r]] = e
        emb_d = torch.from_numpy(emb).to(self.dev)
        if self.act == torch.bfloat16:  # tensor-core GEMMs with the bf16 text K / V weights
            emb_d = emb_d.to(torch.bfloat16)
        out = {}
        for lid, (wq, wk, wv, scale) in self.W.ca.items():
            c = wq.shape[0]
            k = torch.empty((R * ks, c), dtype=self.act, device=self.dev)
            vt = torch.empty((c, R * ks), dtype=self.act, device=self.dev)
            mt = torch.empty((R * ks, c), dtype=self.act, device=self.dev)
            self.gemm(R * ks, c, emb.shape[1], a=DRef(emb_d), b=DRef(wk), d=DRef(k))
            self.gemm(R * ks, c, emb.shape[1], a=DRef(emb_d), b=DRef(wv), d=DRef(vt), d_trans=True)
            self.gemm(R * ks, c, c, a=DRef(k), b=DRef(wq), d=DRef(mt))
            out[lid] = (k, vt, None, mt)
        kseg = torch.tensor([v for r in range(R) for v in (r * ks, r * ks + nts[r])], dtype=torch.int32,
                            device=self.dev)
        return out, kseg, max(nts)

    # ------------------------------------------------------------ building blocks
    def attn_self(self, lid, m, s: DRef, y1: DRef, level, tag, pre=None, segs=None):
        """y1 = s + softmax(s Wq (s Wk)^T * scale) (s Wv) over m tokens (sparse.py:265-300/341-349),
        computed as softmax(Q' s^T * scale) (s Wv) with Q' = s (Wq Wk^T) (Weights.sa).

        segs (batched requests): (q_seg, nseg, max_q) -- each request's rows attend to its own rows."""
        wqv, scale = self.W.sa[lid]
        c = wqv.shape[1]
        cap = self.cap(level)
        mp = _pad(cap)
        qk = self.scratch(f"q2{tag}", (cap, c))
        vt = self.scratch(f"vt{tag}", (c, mp), zero=True)
        # one GEMM for Q' (row-major) and V (stored transposed as the PV B operand)
        self.gemm(m, 2 * c, c, a=s, b=DRef(wqv), d=DRef(qk), n_split=c, d2=DRef(vt, ld=mp), d2_trans=True,
                  b_static=True)
        qr = DRef(qk)
        if segs is not None:
            qseg, nseg, maxq = segs
            self.attn(m, m, c, qr, s, DRef(vt, ld=mp), scale, s, y1, pre, segs=(qseg, qseg, nseg, maxq, maxq))
            return
        if self.use_fused_attn(c, m, m, pre):
            # S = Q' s^T, softmax and P.V (+ residual) in one tcgen05 kernel (fis_attn)
            self.attn(m, m, c, qr, s, DRef(vt, ld=mp), scale, s, y1, pre)
            return
        S = self.scratch(f"S{tag}", (cap, cap), torch.float32)  # unfused path only (cap^2)
        P = self.scratch(f"P{tag}", (cap, mp), zero=True)
        self.gemm(m, m, c, a=qr, b=s, d=DRef(S, ld=_pad(m)))
        self.softmax(m, m, _pad(m), DRef(S, ld=_pad(m)), scale, DRef(P, ld=_pad(m)))
        self.gemm(m, c, m, a=DRef(P, ld=_pad(m)), b=DRef(vt, ld=mp), d=y1, res=s, pre=pre)

    def attn_cross(self, lid, m, x: DRef, out: DRef, level, tag, kv, pre=None, map_=None, ctrl=None, segs=None):
        """out = x + softmax(x Wq K_text^T * scale) V_text (sparse.py:303-338/352-361, unet.py:555-566).

        segs (batched requests): (q_seg, k_seg, nseg, max_q) -- each request's rows attend to its
        own prompt's keys (stacked K / V^T of all requests)."""
        wq, _, _, scale = self.W.ca[lid]
        k, vt, v, mt = kv[lid]
        c, nt = wq.shape[0], k.shape[0]
        ntp = vt.shape[1]
        cap = self.cap(level)
        # scores x (wq K^T) = x M: the layer input is the query, M^T (per edit) the key matrix
        if segs is not None:
            self.attn(m, nt, c, x, DRef(mt), DRef(vt), scale, x, out, pre, segs=segs)
            return
        if ctrl is None and map_ is None and self.use_fused_attn(c, m, nt, pre) and not x.ss:
            self.attn(m, nt, c, x, DRef(mt), DRef(vt), scale, x, out, pre)
            return
        S = self.scratch(f"Sx{tag}", (cap, ntp), torch.float32)  # ld padded: 16-byte aligned rows
        P = self.scratch(f"Px{tag}", (cap, ntp), zero=True)
        self.gemm(m, nt, c, a=x, b=DRef(mt), d=DRef(S), b_static=True)  # M^T: per edit
        if ctrl is not None:
            cached, verbatim, pairs = ctrl
            self.softmax(m, nt, ntp, DRef(S), scale, DRef(P), map_, cached=cached, verbatim=verbatim, pairs=pairs)
        else:
            self.softmax(m, nt, ntp, DRef(S), scale, DRef(P), map_)
        self.gemm(m, c, ntp, a=DRef(P), b=DRef(vt), d=out, res=x, pre=pre, b_static=True)  # text V^T

    def use_fused_attn(self, d, m=None, n_keys=None, pre=None):
        if self.act != torch.bfloat16 or d % 64:
            return False
        return self.fused_attn

    def attn(self, m, n_keys, d, q: DRef, k: DRef, vt: DRef, scale, res: DRef, out: DRef, pre=None, segs=None):
        if self.act != torch.bfloat16:
            raise ContractViolation("fused attention (fis_attn) runs on bf16 operands only")
        a = L.AttnArgs(m, n_keys, d, d, q.ref(), k.ref(), vt.ref(), float(scale), _r(res), _r(pre), out.ref(),
                       L.ptr(self.step_dev))
        maxk = n_keys
        if segs is not None:
            qseg, kseg, nseg, maxq, maxk = segs
            a.nseg, a.max_seg_q, a.q_seg, a.k_seg = nseg, maxq, L.ptr(qseg), L.ptr(kseg)
        # workspace: the P scratch of value slices sharing one P per query tile, or the split-KV
        # partials (+ completion counters, zeroed once and reset by the kernel)
        nbytes = int(L.lib().fis_attn_ws_bytes(m, maxk, d))
        ws = self.scratch("attn_ws", (nbytes,), torch.uint8, zero=True)
        a.max_seg_k, a.ws, a.ws_bytes = maxk, L.ptr(ws), nbytes
        self._call("fis_attn", a)
        # kernels (2 when P is shared)
        self._count("fis_attn", max(1, L.lib().fis_attn_launches(C.byref(a))), m=m, n_keys=n_keys, d=d,
                    segs=segs is not None)

    def gn_stats(self, x: DRef, hw, c, mean: DRef, var: DRef, n_img=1):
        a = L.GnStatsArgs(hw, c, self.groups, x.ref(), mean.ref(), var.ref(), L.ptr(self.step_dev), n_img)
        self._call("fis_gn_stats", a)
        self._count("fis_gn_stats", rows=hw, c=c)

    def gn_apply(self, lid, x: DRef, rows, c, mean: DRef, var: DRef, y_norm: DRef | None, y_silu: DRef | None,
                 fused_stats: bool = False, img_rows=0, row_img=None):
        gamma, beta = self.W.norm[lid]
        a = L.GnApplyArgs()
        a.img_rows, a.row_img = img_rows, L.ptr(row_img)
        a.rows, a.c, a.groups, a.eps = rows, c, self.groups, NORM_EPS
        a.x, a.mean, a.var = x.ref(), mean.ref(), var.ref()
        a.gamma, a.beta = L.ptr(gamma), L.ptr(beta)
        a.y_norm, a.y_silu = _r(y_norm), _r(y_silu)
        a.step = L.ptr(self.step_dev)
        self._call("fis_gn" if fused_stats else "fis_gn_apply", a)
        nk = max(1, L.lib().fis_gn_launches(C.byref(a))) if fused_stats else 1
        self._count("fis_gn" if fused_stats else "fis_gn_apply", nk, rows=rows, c=c)

    def pool(self, fv: FeatVal, rows, n, out: DRef):
        a = L.PoolArgs()
        a.n, a.c, a.src, a.rows, a.out = n, fv.c, self.src(fv), L.ptr(rows), out.ref()
        a.step = L.ptr(self.step_dev)
        self._call("fis_pool2", a)
        self._count("fis_pool2", rows=n, c=fv.c)

    def up2(self, fv: FeatVal, n, out: DRef):
        a = L.PoolArgs()
        a.n, a.c, a.src, a.rows, a.out = n, fv.c, self.src(fv), None, out.ref()
        a.step = L.ptr(self.step_dev)
        self._call("fis_up2", a)
        self._count("fis_up2", rows=n, c=fv.c)

    def materialize(self, fv: FeatVal, out: DRef, n_img: int = 1):
        src = self.src(fv)
        src.h *= n_img  # stacked images: a per-pixel op over n_img * h * w pixels
        a = L.MaterializeArgs(fv.c, src, out.ref(), L.ptr(self.step_dev))
        self._call("fis_materialize", a)
        self._count("fis_materialize", c=fv.c)

    # ------------------------------------------------------------ one UNet step
    def run_step(self, plan: "StepPlan"):
        """Launch one UNet forward + step update (unet.py:430-458,693) for the current device step."""
        vals = {}
        cfg = self.config
        self.batch = plan.batch
        for ins in self.prog:
            op = ins[0]
            if op == "stem":
                lid, f = ins[1], ins[2]
                self._conv(plan, lid, [(plan.latent_in(), False)], plan.out_buf(f), 0, bias2=slab(self.W.time_bias),
                           pre=plan.record(lid, 0))
                vals[f.key] = plan.value(f)
            elif op == "block":
                blk, fi, fo = ins[1], ins[2], ins[3]
                self._block(plan, blk, vals[fi.key], fo)
                vals[fo.key] = plan.value(fo)
            elif op == "down":
                lid, fi, fp, fo = ins[1], ins[2], ins[3], ins[4]
                lv = fp.level
                rows, n = plan.rows(lv)
                self.pool(vals[fi.key], rows, n, plan.out_buf(fp))
                pv = plan.value(fp)
                self._conv(plan, lid, [(pv, False)], plan.out_buf(fo), lv, pre=plan.record(lid, 0))
                vals[fo.key] = plan.value(fo)
            elif op == "fuse":
                lid, fu, fs, fo = ins[1], ins[2], ins[3], ins[4]
                up = vals[fu.key]
                if not plan.sparse(fo.level) and up.index is None and self.act == torch.bfloat16:
                    # dense level: materialise the 2x upsample once so the fuse conv's A operand is a
                    # dense map the GEMM stages with TMA (one 4-D box per tap)
                    buf = DRef(self.scratch(f"up{fo.level}", (self.cap(fo.level), fu.channels)))
                    self.up2(up, self.cap(fo.level), buf)
                    srcs = [(FeatVal(buf, fo.level, fu.channels), False), (vals[fs.key], False)]
                else:
                    srcs = [(up, True), (vals[fs.key], False)]
                self._conv(plan, lid, srcs, plan.out_buf(fo), fo.level, pre=plan.record(lid, 0))
                vals[fo.key] = plan.value(fo)
            else:  # out conv + step update
                lid, fi = ins[1], ins[2]
                self._conv(plan, lid, [(vals[fi.key], False)], plan.latent_out(), 0, epi=L.EPI_STEP,
                           lat=plan.latent_prev_rows(), pre=plan.record(lid, 0))
        return vals

    def _conv(self, plan, lid, inputs, out: DRef, level, **kw):
        b, bias, cin = self.W.conv[lid]
        rows, m = plan.rows(level)
        srcs = [self.src(fv, up) for fv, up in inputs]
        # halo-mode epilogues: bias (+ time bias) or the out conv's step update (no GN, no recording)
        plain = all(v is None or k_ in ("epi", "lat", "bias2") for k_, v in kw.items()) and \
            kw.get("epi", L.EPI_NONE) in (L.EPI_NONE, L.EPI_STEP)
        halo = plan.halo_rows(level) if plain and self.act == torch.bfloat16 else None
        if halo is not None and all(fv.c % 64 == 0 for fv, _ in inputs):
            # stacked sparse level: rows as framed runs of adjacent pixels, staged once per kernel row
            # (csrc/fis_gemm_halo.cu); framing rows are computed but not stored (d_rows = -1)
            pix, outi, mh = halo
            self.gemm(mh, b.shape[0], b.shape[1], rows=pix, srcs=srcs, out_hw=self.grid(level), b=DRef(b), d=out,
                      bias=bias, b_static=True, d_rows=outi, m_halo=True, log_level=level,
                      **{k_: v for k_, v in kw.items() if v is not None})
            return
        self.gemm(m, b.shape[0], b.shape[1], rows=rows, srcs=srcs, out_hw=self.grid(level), b=DRef(b), d=out,
                  bias=bias, b_static=True, log_level=level, **kw)

    def _block(self, plan, blk, x: FeatVal, fo):
        """conv -> GN -> SiLU -> +self-attn -> +cross-attn (unet.py:452-458)."""
        level, c = fo.level, fo.channels
        cap = self.cap(level)
        rows, m = plan.rows(level)
        tag = f"L{level}"
        s = DRef(self.scratch(f"s{tag}", (cap, c)))
        nl = blk["norm"]
        if plan.batch > 1:
            # stacked requests: GN statistics per image, so the norm runs after the conv
            co = DRef(self.scratch(f"co{tag}", (cap, c), zero=True))  # padding rows stay finite (halo convs)
            self._conv(plan, blk["conv"], [(x, False)], co, level)
            mean, var = plan.stats(nl)
            if plan.sparse(level):  # cached statistics of each row's request
                self.gn_apply(nl, co, m, c, mean, var, None, s, row_img=plan.row_img(level))
            else:
                # statistics per image + normalise + SiLU in one launch (fis_gn)
                self.gn_apply(nl, co, m, c, mean, var, None, s, fused_stats=True, img_rows=self.hw(level))
        elif plan.sparse(level):
            mean, var = plan.stats(nl)
            gamma, beta = self.W.norm[nl]
            self._conv(plan, blk["conv"], [(x, False)], s, level, epi=L.EPI_GN_SILU,
                       gn=(mean, var, gamma, beta, self.config.groups))
        else:
            co = plan.record(blk["conv"], 0) or DRef(self.scratch(f"co{tag}", (cap, c)))
            self._conv(plan, blk["conv"], [(x, False)], co, level)
            mean, var = plan.stats(nl)
            # statistics + normalisation (+ SiLU) of each group in one launch (fis_gn)
            self.gn_apply(nl, co, cap, c, mean, var, plan.record(nl, 0), s, fused_stats=True)
        y1 = DRef(self.scratch(f"y1{tag}", (cap, c)))
        qs = plan.segments(level)
        self.attn_self(blk["self_attn"], m, s, y1, level, tag, pre=plan.record(blk["self_attn"], 0), segs=qs)
        lid = blk["cross_attn"]
        xs = None if qs is None else (qs[0], plan.key_segments(), qs[1], qs[2], plan.max_keys())
        self.attn_cross(lid, m, y1, plan.out_buf(fo), level, tag, plan.kv, pre=plan.record(lid, 0),
                        map_=plan.record(lid, 3), ctrl=plan.ctrl(lid), segs=xs)


# ---------------------------------------------------------------------------
# HBM arena of one cached generation
# ---------------------------------------------------------------------------

class Arena:
    """Per-step HBM slabs of one generation (replaces the CacheStore tiers, cache.py:281-679).

    engine features: FEATURE/POOLED maps of gated levels, gated-norm stats, cross-attention
    maps, step latents. `full=True` also keeps every reference role (LAYER_OUTPUT of all
    layers, all norm stats) for API-level `store.get` parity.
    """

    def __init__(self, eng: Engine, n_text: int, full: bool, batch: int = 1):
        """batch > 1: a stacked arena of `batch` generations (image r = rows [r*hw, (r+1)*hw) of
        every level, statistics [T+1, batch, groups]); `view(r)` is generation r's arena."""
        cfg = eng.config
        T = cfg.steps
        dev, f32 = eng.dev, torch.float32
        if batch > 1 and full:
            raise ContractViolation("a stacked arena records the engine roles only")
        self.eng, self.n_text, self.full, self.T, self.batch = eng, n_text, full, T, batch
        self.latent = torch.empty((T + 1, batch * eng.hw(0), cfg.latent_channels), dtype=f32, device=dev)
        self.feature = {}
        for key, f in eng.feats.items():
            if eng.gated[f.level]:
                self.feature[key] = torch.empty((T + 1, batch * eng.hw(f.level), f.channels), dtype=eng.act,
                                                device=dev)
        self.stats = {}
        self.maps = {}
        self.outputs = {}
        sshape = (T + 1, cfg.groups) if batch == 1 else (T + 1, batch, cfg.groups)
        for hl in eng.layers:
            i = hl.info
            if i.kind == "norm" and (i.gated or full):
                self.stats[i.layer_id] = (torch.empty(sshape, dtype=f32, device=dev),
                                          torch.empty(sshape, dtype=f32, device=dev))
            if i.kind == "cross_attn" and batch == 1:  # stacked: each view owns its maps
                self.maps[i.layer_id] = torch.empty((T + 1, eng.hw(i.level), n_text), dtype=f32, device=dev)
            if full:
                self.outputs[i.layer_id] = torch.empty((T + 1, eng.hw(i.level), i.channels), dtype=f32, device=dev)

    def view(self, r: int, n_text: int) -> "Arena":
        """Arena of stacked generation r (prompt of n_text tokens): strided views of the stacked
        slabs, own cross-attention maps."""
        v = Arena.__new__(Arena)
        v.eng, v.n_text, v.full, v.T, v.batch = self.eng, n_text, False, self.T, 1
        v.stacked, v.index = self, r
        hw = self.eng.hw
        v.latent = self.latent[:, r * hw(0):(r + 1) * hw(0)]
        v.feature = {k: t[:, r * hw(self.eng.feats[k].level):(r + 1) * hw(self.eng.feats[k].level)]
                     for k, t in self.feature.items()}
        v.stats = {k: (m[:, r], s[:, r]) for k, (m, s) in self.stats.items()}
        v.maps = {i.layer_id: torch.empty((self.T + 1, hw(i.level), n_text), dtype=torch.float32,
                                          device=self.eng.dev)
                  for i in self.eng.info.values() if i.kind == "cross_attn"}
        v.outputs = {}
        return v

    def map_tensors(self, fn) -> "Arena":
        """A copy of this arena with every slab replaced by fn(slab) (host <-> device tiering)."""
        a = Arena.__new__(Arena)
        a.__dict__.update({k: v for k, v in self.__dict__.items()
                           if k not in ("latent", "feature", "stats", "maps", "outputs")})
        a.latent = fn(self.latent)
        a.feature = {k: fn(t) for k, t in self.feature.items()}
        a.stats = {k: (fn(m), fn(v)) for k, (m, v) in self.stats.items()}
        a.maps = {k: fn(t) for k, t in self.maps.items()}
        a.outputs = {k: fn(t) for k, t in self.outputs.items()}
        return a

    def slabs(self):
        """(name, tensor) of every slab in a fixed order (the spill sidecar's record order)."""
        out = [(("latent",), self.latent)]
        out += [(("feature", *k), t) for k, t in self.feature.items()]
        for k, (m, v) in self.stats.items():
            out += [(("mean", k), m), (("var", k), v)]
        out += [(("map", k), t) for k, t in self.maps.items()]
        out += [(("out", k), t) for k, t in self.outputs.items()]
        return out

    def nbytes(self):
        ts = [self.latent, *self.feature.values(), *self.maps.values(), *self.outputs.values()]
        ts += [x for p in self.stats.values() for x in p]
        return sum(t.numel() * t.element_size() for t in ts)


# ---------------------------------------------------------------------------
# step plans: where each instruction reads and writes
# ---------------------------------------------------------------------------

class StepPlan:
    """Dense plan: full maps at every level. Records into an arena when given."""

    batch = 1  # stacked images per step

    def segments(self, level):
        """Attention query segments (q_seg, nseg, max_q) of stacked requests; None: one sequence."""
        return None

    def __init__(self, eng: Engine, kv, latents: torch.Tensor, arena: Arena | None = None, ctrl=None):
        self.eng, self.kv, self.arena, self._ctrl = eng, kv, arena, ctrl
        self.latents = latents  # [T+1, HW, Cl] f32 slab: [t-1] in, [t] out

    def sparse(self, level):
        return False

    def rows(self, level):
        return None, self.eng.cap(level)

    def halo_rows(self, level):
        """(pixel per GEMM row, output row or -1, rows) of a halo-mode conv at this level, or None."""
        return None

    def latent_in(self) -> FeatVal:
        return FeatVal(slab(self.latents, prev=True), 0, self.eng.config.latent_channels)

    def latent_out(self) -> DRef:
        return slab(self.latents)

    def latent_prev_rows(self) -> DRef:
        return slab(self.latents, prev=True)

    def out_buf(self, f) -> DRef:
        if self.arena is not None and f.key in self.arena.feature:
            return slab(self.arena.feature[f.key])
        return DRef(self.eng.scratch(f"feat{f.key}", (self.eng.cap(f.level), f.channels)))

    def value(self, f) -> FeatVal:
        return FeatVal(self.out_buf(f), f.level, f.channels)

    def record(self, lid, role):
        a = self.arena
        if a is None:
            return None
        if role == 3:
            return slab(a.maps[lid]) if lid in a.maps else None
        if a.full and role == 0:
            return slab(a.outputs[lid])
        return None

    def stats(self, nl):
        a = self.arena
        if a is not None and nl in a.stats:
            m, v = a.stats[nl]
            return slab(m), slab(v)
        g = self.eng.config.groups
        return (DRef(self.eng.scratch(f"mean{nl}", (self.batch, g), torch.float32)),
                DRef(self.eng.scratch(f"var{nl}", (self.batch, g), torch.float32)))

    def ctrl(self, lid):
        if self._ctrl is None:
            return None
        arena, verbatim, pairs = self._ctrl
        return slab(arena.maps[lid]), verbatim, pairs


class SparsePlan(StepPlan):
    """Select-on-read plan over a cached generation (the edit's sparse steps)."""

    def __init__(self, eng: Engine, kv, arena: Arena, lists, lat_rows: torch.Tensor):
        super().__init__(eng, kv, arena.latent, None)
        self.src_arena = arena
        self.lists = lists  # level -> (rows int32 [n], index int32 [hw], n)
        self.lat_rows = lat_rows  # [n0, Cl] f32 fresh latent rows (updated in place)

    def sparse(self, level):
        return self.eng.gated[level]

    def rows(self, level):
        if self.sparse(level):
            r, _, n = self.lists[level]
            return r, n
        return None, self.eng.cap(level)

    def latent_in(self) -> FeatVal:
        _, idx, _ = self.lists[0]
        return FeatVal(DRef(self.lat_rows), 0, self.eng.config.latent_channels, idx,
                       slab(self.src_arena.latent, prev=True))

    def latent_out(self) -> DRef:
        return DRef(self.lat_rows)

    def latent_prev_rows(self) -> DRef:
        return DRef(self.lat_rows)

    def out_buf(self, f) -> DRef:
        if self.sparse(f.level):
            # zeroed once: rows that pad each stacked request's run are never written by halo-mode
            # convs and must stay finite (attention multiplies them by P = 0)
            return DRef(self.eng.scratch(f"sfeat{f.key}", (self.eng.cap(f.level), f.channels), zero=True))
        return DRef(self.eng.scratch(f"feat{f.key}", (self.eng.cap(f.level), f.channels)))

    def value(self, f) -> FeatVal:
        if self.sparse(f.level):
            _, idx, _ = self.lists[f.level]
            return FeatVal(self.out_buf(f), f.level, f.channels, idx, slab(self.src_arena.feature[f.key]))
        return FeatVal(self.out_buf(f), f.level, f.channels)

    def record(self, lid, role):
        return None

    def stats(self, nl):
        if self.eng.info[nl].gated:
            m, v = self.src_arena.stats[nl]
            return slab(m), slab(v)
        return super().stats(nl)


class BatchedSparsePlan(SparsePlan):
    """R edit requests stepped as one stacked batch (the per-GPU shard of requests).

    Rows of all requests are concatenated per gated level (each request's run padded to a
    multiple of 16 rows, so attention segments start 16-byte aligned); dense levels stack the
    R full maps. Every GEMM of the step then runs once over all requests' rows, reading each
    weight once per step for R requests. Attention is block-diagonal (each request's queries
    see only its own rows / its own prompt's keys) and GroupNorm uses each image's statistics.
    """

    def __init__(self, eng: Engine, kv, arena: Arena, lists, lat_rows: torch.Tensor, qsegs, kseg, row_img,
                 max_keys: int = 256, halo=None):
        super().__init__(eng, kv, arena, lists, lat_rows)
        self._halo = halo or {}  # gated level -> (pixel per GEMM row, output row / -1, rows) (halo_lists)
        self._max_keys = max_keys  # longest prompt (text keys of one request)
        self.batch = arena.batch
        self._qsegs = qsegs      # level -> (int32 [2R] device, R, max rows per request)
        self._kseg = kseg        # int32 [2R] device: each request's text keys in the stacked K / V^T
        self._row_img = row_img  # gated level -> int32 [rows] device: request of each compact row

    def segments(self, level):
        return self._qsegs[level]

    def halo_rows(self, level):
        return self._halo.get(level) if self.sparse(level) else None

    def key_segments(self):
        return self._kseg

    def max_keys(self):
        return self._max_keys

    def row_img(self, level):
        return self._row_img[level]


def halo_lists(pixels: np.ndarray, out_rows: np.ndarray, h: int, w: int):
    """GEMM rows of a halo-mode conv (fis_gemm_args.m_halo): the active pixels (stacked ids
    img * h * w + y * w + x, row-major per image) grouped into runs of horizontally adjacent
    pixels, each run framed by its left / right neighbour (-1 at the image border) as a row that
    is computed but not stored. Returns (pixel per row, output row per row or -1)."""
    pixels = np.asarray(pixels, np.int64)
    out_rows = np.asarray(out_rows, np.int64)
    if pixels.size == 0:
        return np.zeros(0, np.int32), np.zeros(0, np.int32)
    x = pixels % w
    brk = np.ones(pixels.size, bool)
    brk[1:] = (pixels[1:] != pixels[:-1] + 1) | (x[1:] == 0)
    starts = np.flatnonzero(brk)
    ends = np.append(starts[1:], pixels.size) - 1
    n_runs = starts.size
    total = pixels.size + 2 * n_runs
    pix = np.empty(total, np.int64)
    out = np.full(total, -1, np.int64)
    # position of each pixel in the framed sequence: its index + 2 * (run ordinal) + 1
    run_id = np.cumsum(brk) - 1
    pos = np.arange(pixels.size) + 2 * run_id + 1
    pix[pos] = pixels
    out[pos] = out_rows
    lpos = starts + 2 * np.arange(n_runs)
    rpos = ends + 2 * np.arange(n_runs) + 2
    pix[lpos] = np.where(x[starts] > 0, pixels[starts] - 1, -1)
    pix[rpos] = np.where(x[ends] < w - 1, pixels[ends] + 1, -1)
    return pix.astype(np.int32), out.astype(np.int32)
