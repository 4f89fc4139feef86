"""CPU ORACLE — test infrastructure, never product code.

A numpy restatement of the reference `sparsedit` 0.1.0 algorithm for the sparse
edit path (cached generation, mask detection, sparse UNet forward). Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / reference
legs may import this module, and only as the checker or the timed CPU
baseline. The product path (`paper_2305_17423_b200`) never imports it.

Parity pinning: `tests/test_oracle_golden.py` checks every function here against
golden vectors produced by the real reference package
(`tests/golden/make_golden.py`, run in the build container where
`/root/reference` exists; the vectors are committed under `tests/golden/`).

Numerics follow the reference exactly: float64 accumulation with one float32
rounding per op output (`tensors.py:76-94,129-207`), group-norm statistics
rounded to float32 before normalising (`tensors.py:143-145`), softmax weights
rounded to float32 (`tensors.py:183-192`), SiLU in float64 (`unet.py:291-293`),
float32 avg-pool (`unet.py:296-298`), step rule latent - f32(1/T)*delta
(`unet.py:676-677,693`). All randomness uses the same numpy PCG64/SeedSequence
streams as `unet.py:151-158,325-396,669-673` so weights and latents are
bit-identical to the reference for a given numpy.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# Role ids of the reference cache (cache.py:40-46)
LAYER_OUTPUT, NORM_MEAN, NORM_VAR, CROSS_ATTN_MAP, STEP_LATENT = 0, 1, 2, 3, 4
NORM_EPS = 1e-5  # unet.py:69
OTSU_BINS = 256  # masks.py:18


# ---------------------------------------------------------------------------
# configuration and seeded parameters (unet.py:73-138, 312-399)
# ---------------------------------------------------------------------------

DEFAULTS = dict(latent_h=64, latent_w=64, latent_channels=4, channels=(8, 16, 32),
                blocks_per_level=1, groups=4, steps=20, t1=5, t2=10, gate_fraction=0.25,
                dilation_radius=1, text_dim=16, vocab_size=512, seed=0)


def cfg_of(c) -> dict:
    """Accept a dict, or any object with to_json(), and fill defaults."""
    d = c.to_json() if hasattr(c, "to_json") else dict(c)
    out = dict(DEFAULTS)
    out.update(d)
    out["channels"] = tuple(int(v) for v in out["channels"])
    return out


def _stream(*words):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(words))))


@dataclass
class Layer:
    lid: int
    name: str
    kind: str
    level: int
    h: int
    w: int
    c: int
    gated: bool
    c_in: int = 0
    p: dict = field(default_factory=dict)


@dataclass
class Net:
    cfg: dict
    layers: list
    time_bias: np.ndarray
    stem: int = 0
    enc: list = field(default_factory=list)   # enc[l] = list of block dicts kind->lid
    down: list = field(default_factory=list)
    fuse: dict = field(default_factory=dict)
    dec: dict = field(default_factory=dict)
    out: int = 0


def build_net(cfg) -> Net:
    """Layer registry + seeded weights in construction order (unet.py:312-399)."""
    cfg = cfg_of(cfg)
    H, W = cfg["latent_h"], cfg["latent_w"]
    area = H * W
    layers: list[Layer] = []

    def add(name, kind, level, c, c_in=0):
        h, w = H >> level, W >> level
        L = Layer(len(layers), name, kind, level, h, w, c, (h * w) >= cfg["gate_fraction"] * area, c_in)
        layers.append(L)
        g = _stream(cfg["seed"], 1000, L.lid)
        if kind == "conv":
            wt = g.standard_normal((c, c_in, 3, 3)).astype(np.float32)
            wt *= np.float32(1.0 / math.sqrt(c_in * 9))
            L.p = dict(w=wt, b=(0.01 * g.standard_normal(c)).astype(np.float32))
        elif kind == "norm":
            L.p = dict(gamma=(1.0 + 0.1 * g.standard_normal(c)).astype(np.float32),
                       beta=(0.1 * g.standard_normal(c)).astype(np.float32))
        elif kind == "self_attn":
            s = np.float32(1.0 / math.sqrt(c))
            L.p = {k: (g.standard_normal((c, c)) * s).astype(np.float32) for k in ("wq", "wk", "wv")}
        else:  # cross_attn
            s = np.float32(1.0 / math.sqrt(c))
            st = np.float32(1.0 / math.sqrt(cfg["text_dim"]))
            wq = (g.standard_normal((c, c)) * s).astype(np.float32)
            wk = (g.standard_normal((cfg["text_dim"], c)) * st).astype(np.float32)
            wv = (g.standard_normal((cfg["text_dim"], c)) * st).astype(np.float32)
            L.p = dict(wq=wq, wk_text=wk, wv_text=wv)
        if kind in ("self_attn", "cross_attn"):
            L.p["scale"] = 1.0 / math.sqrt(c)
        return L.lid

    def block(tag, level, c):
        return {k: add(f"{tag}.{k}", k, level, c, c if k == "conv" else 0)
                for k in ("conv", "norm", "self_attn", "cross_attn")}

    ch = cfg["channels"]
    nl = len(ch)
    net = Net(cfg, layers, None)
    net.stem = add("stem", "conv", 0, ch[0], cfg["latent_channels"])
    net.enc = [[block(f"enc{l}.b{b}", l, ch[l]) for b in range(cfg["blocks_per_level"])] for l in range(nl)]
    net.down = [add(f"down{l}", "conv", l + 1, ch[l + 1], ch[l]) for l in range(nl - 1)]
    for l in range(nl - 2, -1, -1):
        net.fuse[l] = add(f"fuse{l}", "conv", l, ch[l], ch[l + 1] + ch[l])
        net.dec[l] = [block(f"dec{l}.b{b}", l, ch[l]) for b in range(cfg["blocks_per_level"])]
    net.out = add("out", "conv", 0, cfg["latent_channels"], ch[0])
    net.time_bias = (0.1 * _stream(cfg["seed"], 17).standard_normal((cfg["steps"] + 1, ch[0]))).astype(np.float32)
    net.layers = layers
    return net


def embed(ids, cfg) -> np.ndarray:
    """unet.py:151-158"""
    cfg = cfg_of(cfg)
    table = _stream(cfg["seed"], 13).standard_normal((cfg["vocab_size"], cfg["text_dim"])).astype(np.float32)
    return table[list(ids)]


def init_latent(cfg) -> np.ndarray:
    """unet.py:669-673"""
    cfg = cfg_of(cfg)
    return _stream(cfg["seed"], 11).standard_normal(
        (1, cfg["latent_channels"], cfg["latent_h"], cfg["latent_w"]), dtype=np.float32)


def step_scale(cfg) -> np.float32:
    """unet.py:676-677"""
    return np.float32(1.0) / np.float32(cfg_of(cfg)["steps"])


def lcs_pairs(a, b):
    """Shared-token pairs by longest common subsequence (unet.py:174-195)."""
    la, lb = len(a), len(b)
    tab = [[0] * (lb + 1) for _ in range(la + 1)]
    for i in range(la):
        for j in range(lb):
            tab[i + 1][j + 1] = tab[i][j] + 1 if a[i] == b[j] else max(tab[i][j + 1], tab[i + 1][j])
    out, i, j = [], la, lb
    while i and j:
        if a[i - 1] == b[j - 1]:
            out.append((i - 1, j - 1)); i -= 1; j -= 1
        elif tab[i - 1][j] >= tab[i][j - 1]:
            i -= 1
        else:
            j -= 1
    return tuple(out[::-1])


# ---------------------------------------------------------------------------
# dense kernels (tensors.py:76-207, unet.py:291-302)
# ---------------------------------------------------------------------------

def conv3x3(x, w, b) -> np.ndarray:
    """Same-size 3x3 cross-correlation, f64 accumulation per tap, bias last (tensors.py:76-113)."""
    n, ci, h, ww = x.shape
    xp = np.zeros((n, ci, h + 2, ww + 2))
    xp[:, :, 1:h + 1, 1:ww + 1] = x
    w64 = w.astype(np.float64)
    acc = np.zeros((n, w.shape[0], h * ww))
    for ky in range(3):
        for kx in range(3):
            acc += w64[:, :, ky, kx] @ xp[:, :, ky:ky + h, kx:kx + ww].reshape(n, ci, h * ww)
    acc += b.astype(np.float64)[None, :, None]
    return acc.reshape(n, w.shape[0], h, ww).astype(np.float32)


def conv3x3_at(x, w, b, pix) -> np.ndarray:
    """3x3 conv evaluated only at flat pixel indices `pix` -> (len(pix), c_out) f32.

    Same value the reference's gathered-block valid conv produces at those
    pixels (sparse.py:143-223) up to f64 reassociation.
    """
    _, ci, h, ww = x.shape
    xp = np.zeros((ci, h + 2, ww + 2))
    xp[:, 1:h + 1, 1:ww + 1] = x[0]
    ys, xs = np.divmod(np.asarray(pix, dtype=np.int64), ww)
    w64 = w.astype(np.float64)
    acc = np.zeros((len(ys), w.shape[0]))
    for ky in range(3):
        for kx in range(3):
            acc += xp[:, ys + ky, xs + kx].T @ w64[:, :, ky, kx].T
    acc += b.astype(np.float64)[None, :]
    return acc.astype(np.float32)


def gn_stats(x, groups):
    """Group statistics in f64 rounded to f32 (tensors.py:129-146)."""
    n, c, h, w = x.shape
    xg = x.reshape(n, groups, c // groups, h, w).astype(np.float64)
    return xg.mean(axis=(2, 3, 4)).astype(np.float32), xg.var(axis=(2, 3, 4)).astype(np.float32)


def gn_apply(x, mean, var, gamma, beta, eps=NORM_EPS):
    """tensors.py:149-180"""
    n, c, h, w = x.shape
    g = mean.shape[1]
    xg = x.reshape(n, g, c // g, h, w).astype(np.float64)
    y = (xg - mean.astype(np.float64)[:, :, None, None, None]) / np.sqrt(
        var.astype(np.float64)[:, :, None, None, None] + float(eps))
    y = y.reshape(n, c, h, w) * gamma.astype(np.float64)[None, :, None, None] \
        + beta.astype(np.float64)[None, :, None, None]
    return y.astype(np.float32)


def silu(x):
    """unet.py:291-293"""
    v = x.astype(np.float64)
    return (v / (1.0 + np.exp(-v))).astype(np.float32)


def avgpool2(x):
    """unet.py:296-298 (float32 mean)"""
    n, c, h, w = x.shape
    return x.reshape(n, c, h // 2, 2, w // 2, 2).mean(axis=(3, 5)).astype(np.float32)


def upsample2(x):
    """unet.py:301-302"""
    return x.repeat(2, axis=2).repeat(2, axis=3)


def proj(tok, w):
    """sparse.py:261-262"""
    return (tok.astype(np.float64) @ w.astype(np.float64)).astype(np.float32)


def attn_weights(q, k, scale):
    """tensors.py:183-192"""
    s = (q.astype(np.float64) @ k.astype(np.float64).T) * float(scale)
    s = np.exp(s - s.max(axis=1, keepdims=True))
    return (s / s.sum(axis=1, keepdims=True)).astype(np.float32)


def attn_apply(p, v):
    """tensors.py:195-200"""
    return (p.astype(np.float64) @ v.astype(np.float64)).astype(np.float32)


def tokens_of(x):
    n, c, h, w = x.shape
    return x[0].reshape(c, h * w).T


def from_tokens(tok, shape):
    return np.ascontiguousarray(tok.T).reshape(shape)


def text_kv(L: Layer, text):
    """unet.py:476-479"""
    return proj(text, L.p["wk_text"]), proj(text, L.p["wv_text"])


# ---------------------------------------------------------------------------
# MAC accounting (tensors.py:210-224, unet.py:404-426,482-488)
# ---------------------------------------------------------------------------

def conv_macs(L: Layer, px):
    return px * L.c * L.c_in * 9


def sa_macs(L: Layer, a):
    return 3 * a * L.c * L.c + 2 * a * a * L.c


def ca_macs(L: Layer, a, n_text, text_dim):
    return a * L.c * L.c + 2 * n_text * text_dim * L.c + 2 * a * n_text * L.c


def dense_step_macs(net: Net, n_text):
    out = {}
    for L in net.layers:
        hw = L.h * L.w
        out[L.lid] = {"conv": conv_macs(L, hw), "norm": 0, "self_attn": sa_macs(L, hw),
                      "cross_attn": ca_macs(L, hw, n_text, net.cfg["text_dim"])}[L.kind]
    return out


# ---------------------------------------------------------------------------
# UNet forward with pluggable per-layer ops (unet.py:430-458)
# ---------------------------------------------------------------------------

def forward(net: Net, latent, t, text, ops):
    L = net.layers
    x = ops.conv(L[net.stem], latent)
    x = x + net.time_bias[t][None, :, None, None]
    skips = []
    nl = len(net.cfg["channels"])
    for l in range(nl):
        for blk in net.enc[l]:
            x = _block(net, blk, x, text, ops)
        if l < nl - 1:
            skips.append(x)
            x = ops.conv(L[net.down[l]], avgpool2(x))
    for l in range(nl - 2, -1, -1):
        x = ops.conv(L[net.fuse[l]], np.concatenate([upsample2(x), skips[l]], axis=1))
        for blk in net.dec[l]:
            x = _block(net, blk, x, text, ops)
    return ops.conv(L[net.out], x)


def _block(net, blk, x, text, ops):
    L = net.layers
    y = silu(ops.norm(L[blk["norm"]], ops.conv(L[blk["conv"]], x)))
    y = y + ops.self_attn(L[blk["self_attn"]], y)
    return y + ops.cross_attn(L[blk["cross_attn"]], y, text)


class DenseOps:
    """unet.py:491-536; `rec(lid, role, payload)` records into a cache."""

    def __init__(self, net, rec=None, macs=None):
        self.net, self.rec, self.macs = net, rec, macs

    def _r(self, lid, role, v):
        if self.rec is not None:
            self.rec(lid, role, v)

    def _m(self, lid, v):
        if self.macs is not None:
            self.macs[lid] = self.macs.get(lid, 0) + v

    def conv(self, L, x):
        y = conv3x3(x, L.p["w"], L.p["b"])
        self._m(L.lid, conv_macs(L, L.h * L.w))
        self._r(L.lid, LAYER_OUTPUT, y)
        return y

    def norm(self, L, x):
        mean, var = gn_stats(x, self.net.cfg["groups"])
        y = gn_apply(x, mean, var, L.p["gamma"], L.p["beta"])
        self._r(L.lid, NORM_MEAN, mean)
        self._r(L.lid, NORM_VAR, var)
        self._r(L.lid, LAYER_OUTPUT, y)
        return y

    def self_attn(self, L, x):
        tok = tokens_of(x)
        p = attn_weights(proj(tok, L.p["wq"]), proj(tok, L.p["wk"]), L.p["scale"])
        y = from_tokens(attn_apply(p, proj(tok, L.p["wv"])), x.shape)
        self._m(L.lid, sa_macs(L, L.h * L.w))
        self._r(L.lid, LAYER_OUTPUT, y)
        return y

    def cross_attn(self, L, x, text):
        k, v = text_kv(L, text)
        p = self._ca_weights(L, x, k)
        y = from_tokens(attn_apply(p, v), x.shape)
        self._m(L.lid, ca_macs(L, L.h * L.w, text.shape[0], text.shape[1]))
        self._r(L.lid, CROSS_ATTN_MAP, p)
        self._r(L.lid, LAYER_OUTPUT, y)
        return y

    def _ca_weights(self, L, x, k):
        return attn_weights(proj(tokens_of(x), L.p["wq"]), k, L.p["scale"])


class ControlledOps(DenseOps):
    """Shared-token columns pinned to the cached map, rows renormalised (unet.py:539-575)."""

    def __init__(self, net, maps, pairs, n_new, macs=None):
        super().__init__(net, None, macs)
        self.maps, self.pairs, self.n_new = maps, pairs, n_new

    def _ca_weights(self, L, x, k):
        cached = self.maps[L.lid]
        if len(self.pairs) == self.n_new and self.n_new == cached.shape[1]:
            return cached
        p = super()._ca_weights(L, x, k)
        for oc, nc in self.pairs:
            p[:, nc] = cached[:, oc]
        s = p.sum(axis=1, keepdims=True)
        return (p.astype(np.float64) / s.astype(np.float64)).astype(np.float32)

    def cross_attn(self, L, x, text):
        k, v = text_kv(L, text)
        p = self._ca_weights(L, x, k)
        self._m(L.lid, ca_macs(L, L.h * L.w, text.shape[0], text.shape[1]))
        return from_tokens(attn_apply(p, v), x.shape)


class SparseOps:
    """Mask-restricted execution over cached outputs (unet.py:578-663, sparse.py:184-338)."""

    def __init__(self, net, pyr, plans, cache, t, macs=None):
        self.net, self.pyr, self.plans, self.cache, self.t = net, pyr, plans, cache, t
        self.macs = macs

    def _m(self, lid, v):
        if self.macs is not None:
            self.macs[lid] = self.macs.get(lid, 0) + v

    def _base(self, L, shape):
        c = self.cache.get((self.t, L.lid, LAYER_OUTPUT))
        if c is None:
            raise KeyError(f"cache miss: step={self.t} layer={L.lid} role=layer_output")
        return c.copy()

    def conv(self, L, x):
        if not L.gated:
            self._m(L.lid, conv_macs(L, L.h * L.w))
            return conv3x3(x, L.p["w"], L.p["b"])
        mask = self.pyr[L.level]
        pix = np.flatnonzero(mask.ravel())
        out = self._base(L, (1, L.c, L.h, L.w))
        if pix.size:
            vals = conv3x3_at(x, L.p["w"], L.p["b"], pix)
            out.reshape(L.c, -1)[:, pix] = vals.T
        self._m(L.lid, conv_macs(L, self.plans[L.level]["cost"]))
        return out

    def norm(self, L, x):
        if not L.gated:
            mean, var = gn_stats(x, self.net.cfg["groups"])
            return gn_apply(x, mean, var, L.p["gamma"], L.p["beta"])
        mean = self.cache[(self.t, L.lid, NORM_MEAN)]
        var = self.cache[(self.t, L.lid, NORM_VAR)]
        y = gn_apply(x, mean, var, L.p["gamma"], L.p["beta"])
        mask = self.pyr[L.level]
        if mask.all():
            return y
        out = self._base(L, x.shape)
        out[:, :, mask] = y[:, :, mask]
        return out

    def _scatter(self, L, x, pix, tok):
        out = np.empty_like(x) if pix.size == x.shape[2] * x.shape[3] else self._base(L, x.shape)
        out[0].reshape(x.shape[1], -1)[:, pix] = tok.T
        return out

    def self_attn(self, L, x):
        if not L.gated:
            self._m(L.lid, sa_macs(L, L.h * L.w))
            return DenseOps.self_attn(DenseOps(self.net), L, x)
        pix = np.flatnonzero(self.pyr[L.level].ravel())
        self._m(L.lid, sa_macs(L, pix.size))
        if pix.size == 0:
            return self._base(L, x.shape)
        g = tokens_of(x)[pix]
        p = attn_weights(proj(g, L.p["wq"]), proj(g, L.p["wk"]), L.p["scale"])
        return self._scatter(L, x, pix, attn_apply(p, proj(g, L.p["wv"])))

    def cross_attn(self, L, x, text):
        k, v = text_kv(L, text)
        if not L.gated:
            self._m(L.lid, ca_macs(L, L.h * L.w, text.shape[0], text.shape[1]))
            p = attn_weights(proj(tokens_of(x), L.p["wq"]), k, L.p["scale"])
            return from_tokens(attn_apply(p, v), x.shape)
        pix = np.flatnonzero(self.pyr[L.level].ravel())
        self._m(L.lid, ca_macs(L, pix.size, text.shape[0], text.shape[1]))
        if pix.size == 0:
            return self._base(L, x.shape)
        p = attn_weights(proj(tokens_of(x)[pix], L.p["wq"]), k, L.p["scale"])
        return self._scatter(L, x, pix, attn_apply(p, v))


# ---------------------------------------------------------------------------
# masks and gather plans (masks.py:117-222, sparse.py:81-140)
# ---------------------------------------------------------------------------

def accumulate_diff(xs, ys, t1, t2):
    """Returns (values f32 (H,W), degenerate) — masks.py:117-144."""
    acc = None
    for t in range(t1 - 1, t2):
        d = np.abs(xs[t].astype(np.float64) - ys[t].astype(np.float64)).mean(axis=(0, 1))
        acc = d if acc is None else acc + d
    lo, hi = float(acc.min()), float(acc.max())
    if hi == lo:
        return np.zeros(acc.shape, np.float32), True
    v = ((acc - lo) / (hi - lo)).astype(np.float32)
    np.clip(v, 0.0, 1.0, out=v)
    return v, False


def otsu(values, degenerate=False):
    """Returns (epsilon, objective, mask, no_edit) — masks.py:147-177."""
    if degenerate:
        return 1.0, 0.0, np.zeros(values.shape, bool), True
    v = values.ravel().astype(np.float64)
    n = v.size
    eps = (np.arange(OTSU_BINS, dtype=np.float64) + 0.5) / OTSU_BINS
    above = v[None, :] >= eps[:, None]
    n2 = above.sum(axis=1)
    n1 = n - n2
    ok = (n1 > 0) & (n2 > 0)
    if not ok.any():
        return 1.0, 0.0, np.zeros(values.shape, bool), True
    s2 = (v[None, :] * above).sum(axis=1)
    s1 = (v[None, :] * ~above).sum(axis=1)
    m1 = np.divide(s1, n1, out=np.zeros_like(s1), where=ok)
    m2 = np.divide(s2, n2, out=np.zeros_like(s2), where=ok)
    obj = np.full(OTSU_BINS, -np.inf)
    obj[ok] = (n1[ok] * n2[ok]) / float(n) ** 2 * (m1[ok] - m2[ok]) ** 2
    i = int(np.argmax(obj))
    return float(eps[i]), float(obj[i]), values >= eps[i], False


def dilate(bits, r):
    """Square dilation, side 2r+1 (masks.py:180-192)."""
    if r == 0:
        return bits.copy()
    h, w = bits.shape
    p = np.pad(bits, r)
    out = np.zeros((h, w), bool)
    for dy in range(2 * r + 1):
        for dx in range(2 * r + 1):
            out |= p[dy:dy + h, dx:dx + w]
    return out


def orpool2(bits):
    h, w = bits.shape
    return bits.reshape(h // 2, 2, w // 2, 2).any(axis=(1, 3))


def pyramid(bits, levels):
    """masks.py:195-210"""
    out = [np.asarray(bits, bool)]
    for _ in range(levels - 1):
        out.append(orpool2(out[-1]))
    return out


def centered_square(h, w, f):
    """masks.py:213-222"""
    side = max(1, min(int(round((f * h * w) ** 0.5)), h, w))
    top, left = (h - side) // 2, (w - side) // 2
    b = np.zeros((h, w), bool)
    b[top:top + side, left:left + side] = True
    return b


def gather_plan(bits, kernel=(3, 3), candidates=(2, 4, 8, 16, 32)):
    """argmin over blocks of tile_area*active_tiles, ties to smaller area/h/w (sparse.py:91-140)."""
    kh, kw = kernel
    pairs = [(a, b) for a in sorted(candidates) for b in sorted(candidates) if a >= kh and b >= kw]
    if not pairs:
        raise ValueError("no block candidate fits the kernel")
    h, w = bits.shape
    if not bits.any():
        a, b = min(pairs, key=lambda p: (p[0] * p[1], p[0], p[1]))
        return dict(block=(a, b), tile=(a - kh + 1, b - kw + 1), origins=[], cost=0)
    best = None
    for a, b in pairs:
        th, tw = a - kh + 1, b - kw + 1
        ny, nx = -(-h // th), -(-w // tw)
        pad = np.zeros((ny * th, nx * tw), bool)
        pad[:h, :w] = bits
        grid = pad.reshape(ny, th, nx, tw).any(axis=(1, 3))
        key = (th * tw * int(grid.sum()), a * b, a, b)
        if best is None or key < best[0]:
            best = (key, (a, b), (th, tw), grid)
    key, blk, tile, grid = best
    org = [(int(y) * tile[0], int(x) * tile[1]) for y, x in np.argwhere(grid)]
    return dict(block=blk, tile=tile, origins=org, cost=tile[0] * tile[1] * len(org))


# ---------------------------------------------------------------------------
# pipeline (unet.py:680-899)
# ---------------------------------------------------------------------------

def generate(cfg, ids, net=None, record=True):
    """Dense generation recording every role (unet.py:680-696). Returns (final, cache)."""
    net = net or build_net(cfg)
    text = embed(ids, net.cfg)
    lat = init_latent(net.cfg)
    sc = step_scale(net.cfg)
    cache = {}
    for t in range(1, net.cfg["steps"] + 1):
        rec = (lambda lid, role, v, _t=t: cache.__setitem__((_t, lid, role), v)) if record else None
        lat = lat - sc * forward(net, lat, t, text, DenseOps(net, rec))
        if record:
            cache[(t, 0, STEP_LATENT)] = lat
    return lat, cache


def detect(net, cache, old_ids, new_ids, t1, t2, macs=None):
    """Controlled steps 1..t2, diff, Otsu, dilation (unet.py:709-752).

    Returns dict(no_edit, mask, epsilon, control_latent)."""
    cfg = net.cfg
    text = embed(new_ids, cfg)
    pairs = lcs_pairs(tuple(old_ids), tuple(new_ids))
    lat = init_latent(cfg)
    sc = step_scale(cfg)
    ys = []
    cross = [L.lid for L in net.layers if L.kind == "cross_attn"]
    for t in range(1, t2 + 1):
        maps = {lid: cache[(t, lid, CROSS_ATTN_MAP)] for lid in cross}
        lat = lat - sc * forward(net, lat, t, text, ControlledOps(net, maps, pairs, len(new_ids), macs))
        ys.append(lat)
    xs = [cache[(t, 0, STEP_LATENT)] for t in range(1, t2 + 1)]
    vals, degen = accumulate_diff(xs, ys, t1, t2)
    eps, obj, m, no_edit = otsu(vals, degen)
    if no_edit:
        return dict(no_edit=True, mask=None, epsilon=eps, control_latent=lat, diff=vals)
    return dict(no_edit=False, mask=dilate(m, cfg["dilation_radius"]), epsilon=eps,
                control_latent=lat, diff=vals, raw_mask=m)


def edit(cfg, cache, old_ids, new_ids, user_mask=None, t1=None, t2=None, net=None):
    """Sparse regeneration for the edited prompt (unet.py:823-899).

    Returns dict(latent, mask, no_edit, macs: per-layer sparse MACs, dense_step, plans).
    """
    net = net or build_net(cfg)
    cfg = net.cfg
    t1 = cfg["t1"] if t1 is None else t1
    t2 = cfg["t2"] if t2 is None else t2
    T = cfg["steps"]
    text = embed(new_ids, cfg)
    sc = step_scale(cfg)
    macs1, macs2 = {}, {}
    if user_mask is not None:
        det = dict(no_edit=not user_mask.any(), mask=np.asarray(user_mask, bool), control_latent=None)
        user = True
    else:
        det = detect(net, cache, old_ids, new_ids, t1, t2, macs1)
        user = False
    res = dict(mask=det["mask"], no_edit=det["no_edit"], plans={},
               dense_step=dense_step_macs(net, len(new_ids)))
    if det["no_edit"]:
        res.update(latent=cache[(T, 0, STEP_LATENT)].copy(), macs=macs1, phase2=0)
        return res
    mask = det["mask"]
    if user:
        start, lat = 1, init_latent(cfg)
    else:
        start = t2 + 1
        lat = np.where(mask, det["control_latent"], cache[(t2, 0, STEP_LATENT)])
    full = bool(mask.all())
    pyr = plans = None
    if not full:
        pyr = pyramid(mask, len(cfg["channels"]))
        levels = sorted({L.level for L in net.layers if L.gated})
        plans = {lv: gather_plan(pyr[lv]) for lv in levels}
        res["plans"] = plans
    for t in range(start, T + 1):
        ops = DenseOps(net, None, macs2) if full else SparseOps(net, pyr, plans, cache, t, macs2)
        lat = lat - sc * forward(net, lat, t, text, ops)
    tot = dict(macs1)
    for k, v in macs2.items():
        tot[k] = tot.get(k, 0) + v
    res.update(latent=lat, macs=tot, phase1=sum(macs1.values()), phase2=sum(macs2.values()))
    return res
