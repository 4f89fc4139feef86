"""Gather plans and mask-restricted ops (reference sparse.py:1-361).

`select_gather_plan` keeps the reference's APSC argmin contract. For 3x3
kernels with the default candidates the argmin is always the 2x2-tile grid
(every coarser candidate grid is refined by it), so the plan
is produced by the device mask-plan kernel; other kernels / candidate sets run
the general host search. The sparse ops themselves are device-backed (ops.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, ContractViolation
from .masks import BinaryMask, DevicePlan, _mask_dev

BLOCK_CANDIDATES = (2, 4, 8, 16, 32)


@dataclass(frozen=True)
class GatherPlan:
    block: tuple
    tile: tuple
    kernel: tuple
    origins: tuple
    cost: int
    image: tuple

    def to_json(self) -> dict:
        return {"block": list(self.block), "tile": list(self.tile), "kernel": list(self.kernel),
                "active_tiles": len(self.origins), "cost": self.cost, "origins": [list(o) for o in self.origins]}


@dataclass
class SparseLayerContext:
    step: int
    layer_id: int
    cached_output: object = None
    cached_mean: object = None
    cached_var: object = None
    mask_level: int = 0
    resolution_gate: bool = True


def _pairs(kernel, candidates):
    kh, kw = kernel
    return [(a, b) for a in sorted(candidates) for b in sorted(candidates) if a >= kh and b >= kw]


def _host_search(bits, kernel, pairs):
    kh, kw = kernel
    h, w = bits.shape
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
    _, blk, tile, grid = best
    org = tuple((int(y) * tile[0], int(x) * tile[1]) for y, x in np.argwhere(grid))
    return blk, tile, org


def select_gather_plan(mask: BinaryMask, kernel, candidates=BLOCK_CANDIDATES) -> GatherPlan:
    """argmin over blocks of tile_area * active_tiles; ties to smaller area, h, w (sparse.py:91-140)."""
    kernel = tuple(kernel)
    pairs = _pairs(kernel, candidates)
    if not pairs:
        raise ConfigError(f"no block candidate in {candidates} fits kernel {kernel}")
    if mask.is_empty():
        a, b = min(pairs, key=lambda p: (p[0] * p[1], p[0], p[1]))
        return GatherPlan((a, b), (a - kernel[0] + 1, b - kernel[1] + 1), kernel, (), 0, mask.shape)
    if kernel == (3, 3) and (4, 4) in pairs and all(a % 2 == 0 and b % 2 == 0 for a, b in pairs):
        # every candidate tile side (block - 2) is even, so the 2x2-tile grid refines all of
        # them and has the smallest block area: the argmin is (4,4) — computed on device
        dp = DevicePlan(_mask_dev(mask), mask.h, mask.w, 1)
        org = dp.origins(0)
        return GatherPlan((4, 4), (2, 2), kernel, org, 4 * len(org), mask.shape)
    blk, tile, org = _host_search(mask.bits, kernel, pairs)
    return GatherPlan(blk, tile, kernel, org, tile[0] * tile[1] * len(org), mask.shape)


def __getattr__(name):
    if name in ("gather_blocks", "sparse_conv", "sparse_group_norm", "sparse_self_attention",
                "sparse_cross_attention", "dense_self_attention", "dense_cross_attention"):
        from . import ops
        return getattr(ops, name)
    raise AttributeError(name)
