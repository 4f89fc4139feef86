"""UNet configuration, layer registry, seeded host parameters and the step program.

The registry order and the seeded numpy streams follow the reference exactly
(unet.py:73-138 config, :312-399 registry + weights, :151-158 embeddings,
:669-673 initial latent) so device results can be compared with the CPU
reference on identical inputs. The "step program" is the topology of one UNet
forward (unet.py:430-458) flattened into instructions that the dense and the
sparse device engines both execute.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import functools

import numpy as np

from .errors import ConfigError, ContractViolation

ALLOWED_LATENT = (32, 64, 96, 128)  # unet.py:64
SEED_INIT, SEED_TOKENS, SEED_TIME, SEED_LAYER = 11, 13, 17, 1000  # unet.py:65-68
NORM_EPS = 1e-5


@dataclass(frozen=True)
class UNetConfig:
    """Same fields, defaults and validation as sparsedit UNetConfig (unet.py:73-138)."""

    latent_h: int = 64
    latent_w: int = 64
    latent_channels: int = 4
    channels: tuple = (8, 16, 32)
    blocks_per_level: int = 1
    groups: int = 4
    steps: int = 20
    t1: int = 5
    t2: int = 10
    gate_fraction: float = 0.25
    dilation_radius: int = 1
    text_dim: int = 16
    vocab_size: int = 512
    seed: int = 0

    def __post_init__(self):
        if self.latent_h not in ALLOWED_LATENT or self.latent_w not in ALLOWED_LATENT:
            raise ConfigError(f"latent dims must be one of {ALLOWED_LATENT}, got {(self.latent_h, self.latent_w)}")
        object.__setattr__(self, "channels", tuple(int(c) for c in self.channels))
        if not self.channels:
            raise ConfigError("at least one channel level required")
        for c in self.channels:
            if c % self.groups != 0:
                raise ConfigError(f"channels {self.channels} must be divisible by groups {self.groups}")
        f = 2 ** (self.levels - 1)
        if self.latent_h % f or self.latent_w % f:
            raise ConfigError(f"latent dims {(self.latent_h, self.latent_w)} not divisible by {f}")
        if not (1 <= self.t1 <= self.t2 <= min(10, self.steps)):
            raise ConfigError(f"need 1 <= t1 <= t2 <= min(10, steps), got t1={self.t1} t2={self.t2} steps={self.steps}")
        if self.steps < 1:
            raise ConfigError("steps must be >= 1")
        if not (0.0 < self.gate_fraction <= 1.0):
            raise ConfigError(f"gate_fraction must be in (0, 1], got {self.gate_fraction}")
        if self.dilation_radius < 0:
            raise ConfigError("dilation_radius must be >= 0")

    @property
    def levels(self) -> int:
        return len(self.channels)

    def to_json(self) -> dict:
        return {k: (list(v) if k == "channels" else v) for k, v in self.__dict__.items()}

    @classmethod
    def from_json(cls, data: dict) -> "UNetConfig":
        unknown = set(data) - set(cls.__dataclass_fields__)
        if unknown:
            raise ConfigError(f"unknown config fields: {sorted(unknown)}")
        return cls(**data)

    def key(self):
        return tuple(sorted((k, tuple(v) if isinstance(v, list) else v) for k, v in self.to_json().items()))


@dataclass(frozen=True)
class LayerInfo:
    layer_id: int
    name: str
    kind: str  # conv | norm | self_attn | cross_attn
    level: int
    h: int
    w: int
    channels: int
    gated: bool


def _rng(*words):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(words))))


@dataclass
class HostLayer:
    info: LayerInfo
    c_in: int = 0
    params: dict = field(default_factory=dict)


def build_registry(config: UNetConfig, with_params: bool = True):
    """Layer registry in construction order, with seeded host params (unet.py:312-399).

    Returns (layers, topo) where topo holds stem/enc/down/fuse/dec/out layer ids.
    """
    area = config.latent_h * config.latent_w
    layers: list[HostLayer] = []

    def add(name, kind, level, c, c_in=0):
        h, w = config.latent_h >> level, config.latent_w >> level
        info = LayerInfo(len(layers), name, kind, level, h, w, c, (h * w) >= config.gate_fraction * area)
        L = HostLayer(info, c_in)
        layers.append(L)
        if with_params:
            g = _rng(config.seed, SEED_LAYER, info.layer_id)
            if kind == "conv":
                w_ = g.standard_normal((c, c_in, 3, 3)).astype(np.float32)
                w_ *= np.float32(1.0 / math.sqrt(c_in * 9))
                L.params = {"weight": w_, "bias": (0.01 * g.standard_normal(c)).astype(np.float32)}
            elif kind == "norm":
                L.params = {"gamma": (1.0 + 0.1 * g.standard_normal(c)).astype(np.float32),
                            "beta": (0.1 * g.standard_normal(c)).astype(np.float32)}
            elif kind == "self_attn":
                s = np.float32(1.0 / math.sqrt(c))
                L.params = {k: (g.standard_normal((c, c)) * s).astype(np.float32) for k in ("wq", "wk", "wv")}
            else:
                s = np.float32(1.0 / math.sqrt(c))
                st = np.float32(1.0 / math.sqrt(config.text_dim))
                L.params = {"wq": (g.standard_normal((c, c)) * s).astype(np.float32),
                            "wk_text": (g.standard_normal((config.text_dim, c)) * st).astype(np.float32),
                            "wv_text": (g.standard_normal((config.text_dim, c)) * st).astype(np.float32)}
        return info.layer_id

    def block(tag, level, c):
        return {k: add(f"{tag}.{k}", k, level, c, c if k == "conv" else 0)
                for k in ("conv", "norm", "self_attn", "cross_attn")}

    ch = config.channels
    topo = {"stem": add("stem", "conv", 0, ch[0], config.latent_channels)}
    topo["enc"] = [[block(f"enc{l}.b{b}", l, ch[l]) for b in range(config.blocks_per_level)]
                   for l in range(config.levels)]
    topo["down"] = [add(f"down{l}", "conv", l + 1, ch[l + 1], ch[l]) for l in range(config.levels - 1)]
    topo["fuse"], topo["dec"] = {}, {}
    for l in range(config.levels - 2, -1, -1):
        topo["fuse"][l] = add(f"fuse{l}", "conv", l, ch[l], ch[l + 1] + ch[l])
        topo["dec"][l] = [block(f"dec{l}.b{b}", l, ch[l]) for b in range(config.blocks_per_level)]
    topo["out"] = add("out", "conv", 0, config.latent_channels, ch[0])
    time_bias = None
    if with_params:
        time_bias = (0.1 * _rng(config.seed, SEED_TIME).standard_normal((config.steps + 1, ch[0]))).astype(np.float32)
    topo["time_bias"] = time_bias
    return layers, topo


def embed_ids(ids, config: UNetConfig) -> np.ndarray:
    """unet.py:151-158"""
    for i in ids:
        if not 0 <= i < config.vocab_size:
            raise ConfigError(f"token id {i} outside vocabulary [0, {config.vocab_size})")
    return _token_table(config.seed, config.vocab_size, config.text_dim)[list(ids)]


@functools.lru_cache(maxsize=2)
def _token_table(seed: int, vocab: int, dim: int) -> np.ndarray:
    """The seeded (vocab, text_dim) embedding table.  The reference regenerates it on every call
    (unet.py:151-158, 38 M normal samples at SD shape); it is a pure function of (seed, vocab, dim),
    so it is generated once per process and kept read-only."""
    table = _rng(seed, SEED_TOKENS).standard_normal((vocab, dim)).astype(np.float32)
    table.flags.writeable = False
    return table


def initial_latent_np(config: UNetConfig) -> np.ndarray:
    """unet.py:669-673"""
    return _rng(config.seed, SEED_INIT).standard_normal(
        (1, config.latent_channels, config.latent_h, config.latent_w), dtype=np.float32)


def step_scale(config: UNetConfig) -> np.float32:
    """unet.py:676-677"""
    return np.float32(1.0) / np.float32(config.steps)


# ---------------------------------------------------------------------------
# step program: the forward topology as instructions (unet.py:430-458)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Feature:
    """An activation that feeds a convolution: produced by `key`, lives at `level`."""

    key: tuple
    level: int
    channels: int


def step_program(config: UNetConfig, topo):
    """Instructions: ("stem", lid, out) / ("block", blk, in, out) / ("down", lid, in, pooled, out)
    / ("fuse", lid, up, skip, out) / ("out", lid, in). Features are keyed by their producer."""
    ch = config.channels
    prog = []
    feats = {}

    def feat(key, level, c):
        f = Feature(key, level, c)
        feats[key] = f
        return f

    x = feat(("x0", topo["stem"]), 0, ch[0])
    prog.append(("stem", topo["stem"], x))
    skips = []
    for l in range(config.levels):
        for blk in topo["enc"][l]:
            y = feat(("blk", blk["cross_attn"]), l, ch[l])
            prog.append(("block", blk, x, y))
            x = y
        if l < config.levels - 1:
            skips.append(x)
            d = topo["down"][l]
            pooled = feat(("pool", d), l + 1, ch[l])
            y = feat(("down", d), l + 1, ch[l + 1])
            prog.append(("down", d, x, pooled, y))
            x = y
    for l in range(config.levels - 2, -1, -1):
        fz = topo["fuse"][l]
        y = feat(("fuse", fz), l, ch[l])
        prog.append(("fuse", fz, x, skips[l], y))
        x = y
        for blk in topo["dec"][l]:
            y = feat(("blk", blk["cross_attn"]), l, ch[l])
            prog.append(("block", blk, x, y))
            x = y
    prog.append(("out", topo["out"], x))
    return prog, feats


def lcs_pairs(old_ids, new_ids):
    """(old index, new index) pairs of the longest common subsequence (unet.py:174-195)."""
    la, lb = len(old_ids), len(new_ids)
    # plain Python rows (numpy scalar indexing made this ~2 ms for 77 x 77 tokens)
    dp = [[0] * (lb + 1) for _ in range(la + 1)]
    for i in range(1, la + 1):
        a, prev, row = old_ids[i - 1], dp[i - 1], dp[i]
        for j in range(1, lb + 1):
            row[j] = prev[j - 1] + 1 if a == new_ids[j - 1] else (prev[j] if prev[j] >= row[j - 1] else row[j - 1])
    pairs, i, j = [], la, lb
    while i > 0 and j > 0:
        if old_ids[i - 1] == new_ids[j - 1]:
            pairs.append((i - 1, j - 1))
            i, j = i - 1, j - 1
        elif dp[i - 1][j] >= dp[i][j - 1]:
            i -= 1
        else:
            j -= 1
    return tuple(reversed(pairs))


def require_tensor4(arr, name="tensor"):
    if not isinstance(arr, np.ndarray) or arr.ndim != 4:
        raise ContractViolation(f"{name} must be a rank-4 ndarray, got {getattr(arr, 'shape', type(arr))}")
    if arr.dtype != np.float32:
        raise ContractViolation(f"{name} must be float32, got {arr.dtype}")
    return arr
