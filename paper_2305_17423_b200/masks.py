"""Edit-mask types and mask generation (reference masks.py:1-243), device-backed.

The value types (BinaryMask, DiffMap, OtsuResult, MaskPyramid) are host objects
at the API boundary exactly as in the reference. Every computation on mask
data runs in the fused K1 kernels of libfisedit (fis_mask_detect /
fis_mask_plan): diff accumulation, Otsu, dilation, OR-pool pyramid, active
pixel / tile lists.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .errors import ContractViolation
from .model import require_tensor4

OTSU_CANDIDATES = 256


@dataclass(frozen=True, eq=False)
class BinaryMask:
    """Immutable per-pixel edit indicator (masks.py:22-71)."""

    bits: np.ndarray

    def __post_init__(self):
        b = np.ascontiguousarray(self.bits, dtype=bool)
        if b.ndim != 2:
            raise ContractViolation(f"mask must be 2-D, got shape {b.shape}")
        b.setflags(write=False)
        object.__setattr__(self, "bits", b)

    @classmethod
    def full(cls, h, w):
        return cls(np.ones((h, w), bool))

    @classmethod
    def empty(cls, h, w):
        return cls(np.zeros((h, w), bool))

    shape = property(lambda self: self.bits.shape)
    h = property(lambda self: self.bits.shape[0])
    w = property(lambda self: self.bits.shape[1])
    active_count = property(lambda self: int(self.bits.sum()))
    sparsity = property(lambda self: self.active_count / self.bits.size)

    def all_active(self) -> bool:
        return bool(self.bits.all())

    def is_empty(self) -> bool:
        return not bool(self.bits.any())

    def __eq__(self, other):
        if not isinstance(other, BinaryMask):
            return NotImplemented
        return np.array_equal(self.bits, other.bits)


@dataclass(frozen=True)
class DiffMap:
    """Accumulated latent difference normalised to [0, 1] (masks.py:75-93)."""

    values: np.ndarray
    degenerate: bool

    def __post_init__(self):
        v = self.values
        if v.ndim != 2 or v.dtype != np.float32:
            raise ContractViolation(f"diff map must be 2-D float32, got {v.dtype} {v.shape}")
        if v.size and (v.min() < 0.0 or v.max() > 1.0):
            raise ContractViolation("diff map values must lie in [0, 1]")
        if self.degenerate and v.any():
            raise ContractViolation("degenerate diff map must be all zero")


@dataclass(frozen=True)
class OtsuResult:
    epsilon: float
    objective: float
    mask: BinaryMask
    no_edit: bool


@dataclass(frozen=True)
class MaskPyramid:
    """Level 0 at latent resolution; each level OR-pools 2x2 footprints (masks.py:105-114)."""

    levels: tuple

    def level_for_shape(self, h, w) -> int:
        for i, m in enumerate(self.levels):
            if m.shape == (h, w):
                return i
        raise ContractViolation(f"no pyramid level with shape ({h}, {w})")


# ---------------------------------------------------------------------------
# device launches
# ---------------------------------------------------------------------------

def _dev():
    L.require_cuda()
    return torch.device("cuda")


def run_detect(h, w, c, t1, t2, radius, x_ref=None, y_ref=None, values_in=None):
    """fis_mask_detect; returns dict of device outputs (values, raw, mask, result, flags)."""
    dev = _dev()
    hw = h * w
    out = dict(values=torch.empty(hw, dtype=torch.float32, device=dev),
               raw=torch.empty(hw, dtype=torch.uint8, device=dev),
               mask=torch.empty(hw, dtype=torch.uint8, device=dev),
               result=torch.zeros(2, dtype=torch.float64, device=dev),
               flags=torch.zeros(2, dtype=torch.int32, device=dev))
    a = L.MaskDetectArgs()
    a.h, a.w, a.c, a.t1, a.t2, a.radius = h, w, c, t1, t2, radius
    if x_ref is not None:
        a.x, a.y = x_ref, y_ref
    a.values, a.raw_mask, a.mask = L.ptr(out["values"]), L.ptr(out["raw"]), L.ptr(out["mask"])
    a.result, a.flags = L.ptr(out["result"]), L.ptr(out["flags"])
    if values_in is not None:
        a.values_in = L.ptr(values_in)
    L.call("fis_mask_detect", a)
    return out


class DevicePlan:
    """Output of fis_mask_plan: per-level bits, active pixel lists, pixel->row maps, tile lists."""

    def __init__(self, mask_dev: torch.Tensor, h, w, levels, radius=0, tiles=True, sync=True):
        """sync=False: the plan kernel is launched but its counts are not read back yet (call
        DevicePlan.finish_all over a batch of plans: one device->host copy for all of them)."""
        dev = mask_dev.device
        self.h, self.w, self.levels = h, w, levels
        self.bits, self.rows, self.index, self.tiles = [], [], [], []
        a = L.MaskPlanArgs()
        a.h, a.w, a.levels, a.radius = h, w, levels, radius
        a.mask = L.ptr(mask_dev)
        for l in range(levels):
            hl, wl = h >> l, w >> l
            self.bits.append(torch.empty(hl * wl, dtype=torch.uint8, device=dev))
            self.rows.append(torch.empty(max(1, hl * wl), dtype=torch.int32, device=dev))
            self.index.append(torch.empty(hl * wl, dtype=torch.int32, device=dev))
            nt = ((hl + 1) // 2) * ((wl + 1) // 2)
            self.tiles.append(torch.empty(max(1, nt), dtype=torch.int32, device=dev) if tiles else None)
            a.bits[l] = L.ptr(self.bits[l])
            a.rows[l] = L.ptr(self.rows[l])
            a.index[l] = L.ptr(self.index[l])
            a.tiles[l] = L.ptr(self.tiles[l]) if tiles else None
        self.counts_dev = torch.zeros(2 * levels, dtype=torch.int32, device=dev)
        a.counts = L.ptr(self.counts_dev)
        L.call("fis_mask_plan", a)
        if sync:
            self._set_counts(self.counts_dev.cpu().tolist())  # one sync per plan: sizes the GEMM launches

    def _set_counts(self, c):
        self.n_active = c[:self.levels]
        self.n_tiles = c[self.levels:]

    @staticmethod
    def finish_all(plans):
        """Read the counts of plans built with sync=False in one device->host copy."""
        if plans:
            for dp, c in zip(plans, torch.stack([dp.counts_dev for dp in plans]).cpu().tolist()):
                dp._set_counts(c)

    def level_bits(self, l) -> np.ndarray:
        return self.bits[l].cpu().numpy().astype(bool).reshape(self.h >> l, self.w >> l)

    def origins(self, l):
        hl, wl = self.h >> l, self.w >> l
        tw = (wl + 1) // 2
        ht = getattr(self, "_host_tiles", None)
        t = ht[l] if ht is not None else self.tiles[l][: self.n_tiles[l]].cpu().numpy()
        return tuple((int(2 * (i // tw)), int(2 * (i % tw))) for i in t)

    @staticmethod
    def fetch_tiles_all(plans):
        """Host copies of every plan's tile lists in one device->host transfer (origins() then reads
        them without a device sync: the stacked edit computes its reports while its steps run)."""
        parts = [dp.tiles[l][: dp.n_tiles[l]] for dp in plans for l in range(dp.levels) if dp.tiles[l] is not None]
        if not parts:
            return
        flat = torch.cat(parts).cpu().numpy()
        i = 0
        for dp in plans:
            ht = []
            for l in range(dp.levels):
                n = dp.n_tiles[l] if dp.tiles[l] is not None else 0
                ht.append(flat[i:i + n])
                i += n
            dp._host_tiles = ht


def _mask_dev(mask: BinaryMask) -> torch.Tensor:
    return torch.from_numpy(mask.bits.astype(np.uint8).ravel()).to(_dev())


# ---------------------------------------------------------------------------
# public API (masks.py:117-243)
# ---------------------------------------------------------------------------

def _nhwc_steps(steps, t1, t2, name):
    arrs = []
    for t in range(t1 - 1, t2):
        a = require_tensor4(steps[t], f"{name}[{t}]")
        arrs.append(a)
    return arrs


def accumulate_diff(x_steps, y_steps, t1: int = 5, t2: int = 10) -> DiffMap:
    """Σ_{t1..t2} channel-mean |X_t - Y_t|, min-max normalised (masks.py:117-144), on device."""
    if not (1 <= t1 <= t2 <= 10):
        raise ContractViolation(f"window must satisfy 1 <= t1 <= t2 <= 10, got ({t1}, {t2})")
    if len(x_steps) < t2 or len(y_steps) < t2:
        raise ContractViolation(
            f"step lists must cover steps 1..{t2}, got lengths {len(x_steps)}, {len(y_steps)}")
    xs = _nhwc_steps(x_steps, t1, t2, "x_steps")
    ys = _nhwc_steps(y_steps, t1, t2, "y_steps")
    for i, (x, y) in enumerate(zip(xs, ys)):
        if x.shape != y.shape:
            raise ContractViolation(f"step {t1 + i} shape mismatch: {x.shape} vs {y.shape}")
    n, c, h, w = xs[0].shape
    dev = _dev()

    def stack(arrs):
        a = np.stack([np.ascontiguousarray(v.reshape(n * c, h * w).T.reshape(h * w, n * c)) for v in arrs])
        return torch.from_numpy(a).to(dev)

    X, Y = stack(xs), stack(ys)
    ss = X.stride(0) * 4
    xr = L.Ref(X.data_ptr(), ss, n * c, L.F32)
    yr = L.Ref(Y.data_ptr(), ss, n * c, L.F32)
    out = run_detect(h, w, n * c, 1, t2 - t1 + 1, 0, xr, yr)
    degenerate = bool(out["flags"][1].item())
    vals = out["values"].cpu().numpy().reshape(h, w)
    return DiffMap(vals, degenerate)


def otsu_threshold(diff: DiffMap) -> OtsuResult:
    """Between-class-variance threshold over 256 midpoints (masks.py:147-177), on device."""
    h, w = diff.values.shape
    if diff.degenerate:
        return OtsuResult(1.0, 0.0, BinaryMask.empty(h, w), no_edit=True)
    v = torch.from_numpy(np.ascontiguousarray(diff.values).ravel()).to(_dev())
    out = run_detect(h, w, 1, 1, 1, 0, values_in=v)
    res = out["result"].cpu().tolist()
    no_edit = bool(out["flags"][0].item())
    if no_edit:
        return OtsuResult(1.0, 0.0, BinaryMask.empty(h, w), no_edit=True)
    mask = BinaryMask(out["raw"].cpu().numpy().astype(bool).reshape(h, w))
    return OtsuResult(float(res[0]), float(res[1]), mask, no_edit=False)


def dilate(mask: BinaryMask, radius: int) -> BinaryMask:
    """Square dilation of side 2r+1, clipped at the border (masks.py:180-192), on device."""
    if radius < 0:
        raise ContractViolation(f"dilation radius must be >= 0, got {radius}")
    if radius == 0:
        return mask
    p = DevicePlan(_mask_dev(mask), mask.h, mask.w, 1, radius=radius, tiles=False)
    return BinaryMask(p.level_bits(0))


def build_pyramid(mask: BinaryMask, levels: int) -> MaskPyramid:
    """OR-pool pyramid (masks.py:195-210), on device."""
    if levels < 1:
        raise ContractViolation(f"pyramid needs at least one level, got {levels}")
    f = 2 ** (levels - 1)
    if mask.h % f or mask.w % f:
        raise ContractViolation(f"mask dims {mask.shape} not divisible by 2^(levels-1) = {f}")
    if levels > L.MAX_LEVELS:
        raise ContractViolation(f"at most {L.MAX_LEVELS} pyramid levels supported")
    p = DevicePlan(_mask_dev(mask), mask.h, mask.w, levels, tiles=False)
    return MaskPyramid(tuple(BinaryMask(p.level_bits(l)) for l in range(levels)))


def centered_square_mask(h: int, w: int, fraction: float) -> BinaryMask:
    """Benchmark mask (masks.py:213-222)."""
    if not 0.0 < fraction <= 1.0:
        raise ContractViolation(f"mask fraction must be in (0, 1], got {fraction}")
    side = max(1, min(int(round((fraction * h * w) ** 0.5)), h, w))
    top, left = (h - side) // 2, (w - side) // 2
    bits = np.zeros((h, w), dtype=bool)
    bits[top:top + side, left:left + side] = True
    return BinaryMask(bits)


def mask_to_tensor(mask: BinaryMask) -> np.ndarray:
    return mask.bits.astype(np.float32)[None, None]


def mask_from_tensor(arr: np.ndarray) -> BinaryMask:
    require_tensor4(arr, "mask tensor")
    if arr.shape[0] != 1 or arr.shape[1] != 1:
        raise ContractViolation(f"mask tensor must be 1x1xHxW, got {arr.shape}")
    return BinaryMask(arr[0, 0] >= 0.5)


def save_mask_pgm(path, mask: BinaryMask) -> None:
    with open(path, "wb") as f:
        f.write(f"P5\n{mask.w} {mask.h}\n255\n".encode("ascii"))
        f.write(np.where(mask.bits, 255, 0).astype(np.uint8).tobytes())
