"""Dense ops, MAC accounting and the FT4 fixture format (reference tensors.py:1-303).

The dense ops (conv2d, conv2d_valid, group_norm, normalize_with_group_stats,
attention_scores, apply_attention, attention) take and return float32 NCHW /
2-D numpy arrays like the reference, and run on the GPU through libfisedit
(`ops.py`). MAC accounting is analytic host arithmetic (tensors.py:210-276).
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

import numpy as np

from .errors import ContractViolation
from .model import require_tensor4

FIXTURE_MAGIC = b"FT4\x00"


@dataclass(frozen=True)
class ConvWeights:
    """Stride-1 conv weights (c_out, c_in, kh, kw) + bias, odd kernels (tensors.py:41-73)."""

    weight: np.ndarray
    bias: np.ndarray
    padding: int

    def __post_init__(self):
        if self.weight.ndim != 4:
            raise ContractViolation(f"conv weight must be rank 4, got shape {self.weight.shape}")
        c_out, _, kh, kw = self.weight.shape
        if kh % 2 == 0 or kw % 2 == 0:
            raise ContractViolation(f"kernel sides must be odd, got ({kh}, {kw})")
        if self.bias.shape != (c_out,):
            raise ContractViolation(f"bias must have shape ({c_out},), got {self.bias.shape}")
        if self.padding < 0:
            raise ContractViolation("padding must be non-negative")

    c_out = property(lambda self: self.weight.shape[0])
    c_in = property(lambda self: self.weight.shape[1])
    kernel = property(lambda self: (self.weight.shape[2], self.weight.shape[3]))


def macs_conv(weights: ConvWeights, active_output_pixels: int) -> int:
    if active_output_pixels < 0:
        raise ContractViolation("active_output_pixels must be >= 0")
    kh, kw = weights.kernel
    return active_output_pixels * weights.c_out * weights.c_in * kh * kw


def macs_attention(q_tokens: int, kv_tokens: int, dim: int) -> int:
    return 2 * q_tokens * kv_tokens * dim


def macs_linear(tokens: int, d_in: int, d_out: int) -> int:
    return tokens * d_in * d_out


@dataclass
class LayerMacs:
    layer_id: int
    kind: str
    dense_macs: int
    sparse_macs: int

    def __post_init__(self):
        if self.sparse_macs > self.dense_macs:
            raise ContractViolation(
                f"layer {self.layer_id}: sparse MACs {self.sparse_macs} exceed dense {self.dense_macs}")


@dataclass
class MacsReport:
    layers: list = field(default_factory=list)

    @property
    def dense_total(self) -> int:
        return sum(l.dense_macs for l in self.layers)

    @property
    def sparse_total(self) -> int:
        return sum(l.sparse_macs for l in self.layers)

    @property
    def ratio(self) -> float:
        s = self.sparse_total
        return math.inf if s == 0 else self.dense_total / s

    def to_json(self) -> dict:
        return {"layers": [dict(layer_id=l.layer_id, kind=l.kind, dense_macs=l.dense_macs, sparse_macs=l.sparse_macs)
                           for l in self.layers],
                "dense_total": self.dense_total, "sparse_total": self.sparse_total,
                "ratio": None if math.isinf(self.ratio) else self.ratio}


def save_tensor(path, arr: np.ndarray) -> None:
    """FT4: magic, 4 little-endian u64 dims, f32 payload (tensors.py:279-290)."""
    require_tensor4(arr, "save_tensor input")
    with open(path, "wb") as f:
        f.write(FIXTURE_MAGIC)
        f.write(struct.pack("<4Q", *arr.shape))
        f.write(np.ascontiguousarray(arr, dtype="<f4").tobytes())


def load_tensor(path) -> np.ndarray:
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != FIXTURE_MAGIC:
            raise ContractViolation(f"bad fixture magic in {path}: {magic!r}")
        dims = struct.unpack("<4Q", f.read(32))
        count = int(np.prod(dims))
        buf = f.read(count * 4)
        if len(buf) != count * 4:
            raise ContractViolation(f"truncated fixture payload in {path}")
    return np.frombuffer(buf, dtype="<f4").reshape(dims).astype(np.float32)


def __getattr__(name):
    # device-backed dense ops live in ops.py; re-exported lazily to avoid import cycles
    if name in ("conv2d", "conv2d_valid", "group_norm", "normalize_with_group_stats", "attention_scores",
                "apply_attention", "attention"):
        from . import ops
        return getattr(ops, name)
    raise AttributeError(name)
