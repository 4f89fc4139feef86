"""Op-level API with reference semantics, executed by libfisedit kernels.

Reference functions mirrored (same names, arguments, errors):
  conv2d / conv2d_valid            tensors.py:97-126
  group_norm / normalize_with_group_stats  tensors.py:129-180
  attention_scores / apply_attention / attention  tensors.py:183-207
  gather_blocks / sparse_conv      sparse.py:143-223
  sparse_group_norm                sparse.py:226-251
  sparse_self_attention / sparse_cross_attention  sparse.py:265-338
  dense_self_attention / dense_cross_attention    sparse.py:341-361
Inputs/outputs are float32 numpy arrays (NCHW maps, 2-D token matrices);
inside, maps are NHWC `[pixels, C]` device tensors and every op is a gather-GEMM,
softmax, group-norm or materialise launch (fp32 operands, fp32 accumulation:
the parity precision). Outside the mask, sparse ops return the cached tensor
bit-exactly (select-on-read materialisation).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib as L
from .engine import NULL, DRef, Launcher, _pad
from .errors import CacheMissError, ContractViolation
from .masks import BinaryMask, DevicePlan
from .model import require_tensor4
from .tensors import ConvWeights

_LAUNCHER = None


def _lz() -> Launcher:
    global _LAUNCHER
    if _LAUNCHER is None:
        _LAUNCHER = Launcher("fp32")
    return _LAUNCHER


def _nhwc(x: np.ndarray) -> torch.Tensor:
    n, c, h, w = x.shape
    return torch.from_numpy(np.ascontiguousarray(x[0].reshape(c, h * w).T)).to(_lz().dev)


def _nchw(t: torch.Tensor, c, h, w) -> np.ndarray:
    return t.reshape(h, w, c).permute(2, 0, 1).reshape(1, c, h, w).contiguous().cpu().numpy()


def _dev2d(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(_lz().dev)


def _finite(name, arr):
    if not np.isfinite(arr).all():
        raise ContractViolation(f"{name} produced non-finite values")
    return arr


def _full_src(t: torch.Tensor, h, w, c) -> L.Src:
    return L.Src(DRef(t).ref(), NULL, None, h, w, c, 0)


def _sel_src(fresh: torch.Tensor, index: torch.Tensor, cache: torch.Tensor, h, w, c) -> L.Src:
    return L.Src(DRef(fresh).ref(), DRef(cache).ref(), L.ptr(index), h, w, c, 0)


def _conv_b(weights: ConvWeights) -> torch.Tensor:
    w = weights.weight
    return _dev2d(w.transpose(0, 2, 3, 1).reshape(w.shape[0], -1))


def _materialize(src: L.Src, c, out: torch.Tensor):
    L.call("fis_materialize", L.MaterializeArgs(c, src, DRef(out).ref(), None))


def _active(mask: BinaryMask):
    dp = DevicePlan(torch.from_numpy(mask.bits.astype(np.uint8).ravel()).to(_lz().dev), mask.h, mask.w, 1,
                    tiles=False)
    return dp.rows[0], dp.index[0], dp.n_active[0]


# ---------------------------------------------------------------------------
# dense ops (tensors.py)
# ---------------------------------------------------------------------------

def _check_conv(x, weights, name):
    require_tensor4(x, f"{name} input")
    if x.shape[1] != weights.c_in:
        raise ContractViolation(f"{name} channel mismatch: input {x.shape} vs weight {weights.weight.shape}")
    if weights.kernel != (3, 3):
        raise ContractViolation(f"{name}: the device kernels implement 3x3 convolutions, got {weights.kernel}")


def _conv_image(img: torch.Tensor, h, w, weights: ConvWeights, rows=None, m=None) -> torch.Tensor:
    lz = _lz()
    m = h * w if m is None else m
    out = torch.empty((m, weights.c_out), dtype=torch.float32, device=lz.dev)
    lz.gemm(m, weights.c_out, 9 * weights.c_in, rows=rows, srcs=[_full_src(img, h, w, weights.c_in)],
            out_hw=(h, w), b=DRef(_conv_b(weights)), d=DRef(out), bias=_dev2d(weights.bias))
    return out


def conv2d(x: np.ndarray, weights: ConvWeights) -> np.ndarray:
    """Same-size 3x3 cross-correlation with bias (tensors.py:97-113)."""
    _check_conv(x, weights, "conv2d")
    kh, kw = weights.kernel
    if weights.padding != (kh - 1) // 2:
        raise ContractViolation(f"padding {weights.padding} does not preserve spatial size for kernel {weights.kernel}")
    n, c, h, w = x.shape
    outs = [_nchw(_conv_image(_nhwc(x[i:i + 1]), h, w, weights), weights.c_out, h, w) for i in range(n)]
    return _finite("conv2d", np.concatenate(outs, axis=0))


def conv2d_valid(blocks: np.ndarray, weights: ConvWeights) -> np.ndarray:
    """Valid 3x3 conv over stacked pre-padded blocks (tensors.py:116-126): the stack is one
    tall image; interior pixels of each block never read across block boundaries."""
    _check_conv(blocks, weights, "conv2d_valid")
    nb, c, bh, bw = blocks.shape
    if bh < 3 or bw < 3:
        raise ContractViolation(f"block {blocks.shape} smaller than kernel (3, 3)")
    img = torch.from_numpy(np.ascontiguousarray(blocks.transpose(0, 2, 3, 1).reshape(nb * bh * bw, c))).to(_lz().dev)
    oy, ox = np.meshgrid(np.arange(1, bh - 1), np.arange(1, bw - 1), indexing="ij")
    per = (oy * bw + ox).ravel()
    rows = (np.arange(nb)[:, None] * bh * bw + per[None, :]).ravel().astype(np.int32)
    out = _conv_image(img, nb * bh, bw, weights, rows=torch.from_numpy(rows).to(_lz().dev), m=rows.size)
    res = out.reshape(nb, bh - 2, bw - 2, weights.c_out).permute(0, 3, 1, 2).contiguous().cpu().numpy()
    return _finite("conv2d", res)


def _gn_stats_dev(xt, hw, c, groups):
    lz = _lz()
    mean = torch.empty(groups, dtype=torch.float32, device=lz.dev)
    var = torch.empty(groups, dtype=torch.float32, device=lz.dev)
    L.call("fis_gn_stats", L.GnStatsArgs(hw, c, groups, DRef(xt).ref(), DRef(mean[None]).ref(),
                                         DRef(var[None]).ref(), None))
    return mean, var


def _gn_apply_dev(xt, rows, n, c, mean, var, gamma, beta, eps, y_rows=None, silu=False):
    a = L.GnApplyArgs()
    out = torch.empty((n, c), dtype=torch.float32, device=_lz().dev)
    a.rows, a.c, a.groups, a.eps = n, c, mean.numel(), eps
    a.x, a.x_rows = DRef(xt).ref(), L.ptr(rows)
    a.mean, a.var = DRef(mean[None]).ref(), DRef(var[None]).ref()
    g, b = _dev2d(gamma), _dev2d(beta)
    a.gamma, a.beta = L.ptr(g), L.ptr(b)
    if silu:
        a.y_silu = DRef(out).ref()
    else:
        a.y_norm = DRef(out).ref()
    L.call("fis_gn_apply", a)
    return out


def group_norm(x, groups, gamma, beta, eps=1e-5):
    """(output, mean, var) with f32-rounded stats (tensors.py:129-146)."""
    require_tensor4(x, "group_norm input")
    n, c, h, w = x.shape
    if c % groups:
        raise ContractViolation(f"channels {c} not divisible by groups {groups}")
    ys, ms, vs = [], [], []
    for i in range(n):
        xt = _nhwc(x[i:i + 1])
        m, v = _gn_stats_dev(xt, h * w, c, groups)
        ys.append(_nchw(_gn_apply_dev(xt, None, h * w, c, m, v, gamma, beta, eps), c, h, w))
        ms.append(m.cpu().numpy())
        vs.append(v.cpu().numpy())
    return _finite("group_norm", np.concatenate(ys)), np.stack(ms), np.stack(vs)


def _check_stats(x, mean, var, gamma, beta):
    n, c, h, w = x.shape
    if mean.shape != var.shape or mean.ndim != 2 or mean.shape[0] != n:
        raise ContractViolation(f"stats shape {mean.shape} invalid for input {x.shape}")
    if c % mean.shape[1]:
        raise ContractViolation(f"channels {c} not divisible by groups {mean.shape[1]}")
    if gamma.shape != (c,) or beta.shape != (c,):
        raise ContractViolation(f"gamma/beta must have shape ({c},)")


def normalize_with_group_stats(x, mean, var, gamma, beta, eps=1e-5):
    """y = gamma*(x-mean)/sqrt(var+eps)+beta with given stats (tensors.py:149-180)."""
    require_tensor4(x, "normalize input")
    _check_stats(x, mean, var, gamma, beta)
    n, c, h, w = x.shape
    ys = []
    for i in range(n):
        m, v = _dev2d(mean[i]), _dev2d(var[i])
        ys.append(_nchw(_gn_apply_dev(_nhwc(x[i:i + 1]), None, h * w, c, m, v, gamma, beta, eps), c, h, w))
    return _finite("group_norm", np.concatenate(ys))


def _scores(qt, kt, scale, nq, nk):
    """softmax(q k^T * scale) rows on device; returns (P [nq, pad16(nk)] f32)."""
    lz = _lz()
    d = qt.shape[1]
    S = torch.empty((nq, nk), dtype=torch.float32, device=lz.dev)
    P = torch.zeros((nq, _pad(nk)), dtype=torch.float32, device=lz.dev)
    lz.gemm(nq, nk, d, a=DRef(qt), b=DRef(kt), d=DRef(S))
    lz.softmax(nq, nk, _pad(nk), DRef(S), float(scale), DRef(P))
    return P


def _apply(P, vt, nq, nk, res=None, out=None):
    lz = _lz()
    c = vt.shape[0]
    out = torch.empty((nq, c), dtype=torch.float32, device=lz.dev) if out is None else out
    lz.gemm(nq, c, _pad(nk), a=DRef(P), b=DRef(vt), d=DRef(out), res=None if res is None else DRef(res))
    return out


def _vt(v: torch.Tensor, nk):
    vt = torch.zeros((v.shape[1], _pad(nk)), dtype=torch.float32, device=v.device)
    vt[:, :nk] = v.t()
    return vt


def attention_scores(q, k, scale):
    if q.ndim != 2 or k.ndim != 2 or q.shape[1] != k.shape[1]:
        raise ContractViolation(f"attention dim mismatch: q {q.shape} vs k {k.shape}")
    P = _scores(_dev2d(q), _dev2d(k), scale, q.shape[0], k.shape[0])
    return P[:, :k.shape[0]].contiguous().cpu().numpy()


def apply_attention(weights, v):
    if weights.shape[1] != v.shape[0]:
        raise ContractViolation(f"attention apply mismatch: weights {weights.shape} vs v {v.shape}")
    nk = v.shape[0]
    P = torch.zeros((weights.shape[0], _pad(nk)), dtype=torch.float32, device=_lz().dev)
    P[:, :nk] = _dev2d(weights)
    out = _apply(P, _vt(_dev2d(v), nk), weights.shape[0], nk)
    return _finite("attention", out.cpu().numpy())


def attention(q, k, v, scale):
    if k.shape[0] != v.shape[0]:
        raise ContractViolation(f"k rows {k.shape[0]} != v rows {v.shape[0]}")
    if q.ndim != 2 or k.ndim != 2 or q.shape[1] != k.shape[1]:
        raise ContractViolation(f"attention dim mismatch: q {q.shape} vs k {k.shape}")
    P = _scores(_dev2d(q), _dev2d(k), scale, q.shape[0], k.shape[0])
    return _finite("attention", _apply(P, _vt(_dev2d(v), k.shape[0]), q.shape[0], k.shape[0]).cpu().numpy())


# ---------------------------------------------------------------------------
# sparse ops (sparse.py)
# ---------------------------------------------------------------------------

def gather_blocks(x, plan, pool=None):
    """Active tiles plus kernel halo, zero outside the image (sparse.py:143-171)."""
    require_tensor4(x, "gather input")
    n, c, h, w = x.shape
    if n != 1:
        raise ContractViolation(f"sparse path handles single-sample maps, got batch {n}")
    if (h, w) != tuple(plan.image):
        raise ContractViolation(f"plan built for {plan.image}, input is {(h, w)}")
    bh, bw = plan.block
    ph, pw = (plan.kernel[0] - 1) // 2, (plan.kernel[1] - 1) // 2
    ey = max((oy + bh for oy, _ in plan.origins), default=0)
    ex = max((ox + bw for _, ox in plan.origins), default=0)
    xt = torch.from_numpy(np.ascontiguousarray(x[0])).to(_lz().dev)
    padded = torch.nn.functional.pad(xt, (pw, pw + max(0, ex - (w + 2 * pw)), ph, ph + max(0, ey - (h + 2 * ph))))
    if not plan.origins:
        return np.zeros((0, c, bh, bw), np.float32)
    org = torch.tensor(plan.origins, device=_lz().dev)
    iy = org[:, 0, None] + torch.arange(bh, device=org.device)[None, :]
    ix = org[:, 1, None] + torch.arange(bw, device=org.device)[None, :]
    out = padded[:, iy[:, :, None], ix[:, None, :]].permute(1, 0, 2, 3)
    return out.contiguous().cpu().numpy()


def _cached(ctx, shape):
    if ctx.cached_output is None:
        raise CacheMissError(ctx.step, ctx.layer_id, "layer_output")
    co = np.asarray(ctx.cached_output)
    if co.shape != tuple(shape):
        raise ContractViolation(f"cached output shape {co.shape} != expected {tuple(shape)}")
    return co


def _finish(fresh, index, n, base: np.ndarray, c, h, w):
    """Full map = base outside the mask, fresh rows inside (select-on-read materialise)."""
    out = torch.empty((h * w, c), dtype=torch.float32, device=_lz().dev)
    if n:
        _materialize(_sel_src(fresh, index, _nhwc(base), h, w, c), c, out)
    else:
        return base.copy()
    return _nchw(out, c, h, w)


def sparse_conv(x, weights: ConvWeights, plan, ctx, mask: BinaryMask, pool=None):
    """Convolution recomputed at mask-active pixels over the cached output (sparse.py:184-223)."""
    require_tensor4(x, "sparse_conv input")
    n, _, h, w = x.shape
    if mask.shape != (h, w) or tuple(plan.image) != (h, w):
        raise ContractViolation(f"mask {mask.shape} / plan {plan.image} inconsistent with input {(h, w)}")
    shape = (n, weights.c_out, h, w)
    if not plan.origins:
        return _cached(ctx, shape).copy()
    if ctx.cached_output is not None:
        base = _cached(ctx, shape)
    elif mask.all_active():
        base = np.zeros(shape, np.float32)
    else:
        raise CacheMissError(ctx.step, ctx.layer_id, "layer_output")
    if n != 1:
        raise ContractViolation(f"sparse path handles single-sample maps, got batch {n}")
    _check_conv(x, weights, "sparse_conv")
    rows, index, na = _active(mask)
    fresh = _conv_image(_nhwc(x), h, w, weights, rows=rows, m=na)
    return _finite("conv2d", _finish(fresh, index, na, base, weights.c_out, h, w))


def sparse_group_norm(x, ctx, gamma, beta, eps, mask: BinaryMask):
    """Cached statistics inside the mask, cached output outside (sparse.py:226-251)."""
    require_tensor4(x, "sparse_group_norm input")
    if ctx.cached_mean is None or ctx.cached_var is None:
        raise CacheMissError(ctx.step, ctx.layer_id, "norm_mean/norm_var")
    if mask.shape != x.shape[2:]:
        raise ContractViolation(f"mask {mask.shape} inconsistent with input {x.shape}")
    mean, var = np.asarray(ctx.cached_mean, np.float32), np.asarray(ctx.cached_var, np.float32)
    _check_stats(x, mean, var, gamma, beta)
    n, c, h, w = x.shape
    if mask.all_active():
        return normalize_with_group_stats(x, mean, var, gamma, beta, eps)
    base = _cached(ctx, x.shape)
    rows, index, na = _active(mask)
    fresh = _gn_apply_dev(_nhwc(x), rows, na, c, _dev2d(mean[0]), _dev2d(var[0]), gamma, beta, eps)
    return _finite("group_norm", _finish(fresh, index, na, base, c, h, w))


def _check_attn(x, ctx, mask):
    if not ctx.resolution_gate:
        raise ContractViolation(f"layer {ctx.layer_id} does not pass the resolution gate; run dense attention")
    n, c, h, w = x.shape
    if mask.shape != (h, w):
        raise ContractViolation(f"mask {mask.shape} inconsistent with input {x.shape}")
    if n != 1:
        raise ContractViolation(f"sparse attention handles single-sample maps, got batch {n}")


def _proj(xt, rows, m, w_t):
    """tokens[rows] @ W on device (A_ROWS gather), W given transposed [d_out, d_in]."""
    lz = _lz()
    out = torch.empty((m, w_t.shape[0]), dtype=torch.float32, device=lz.dev)
    lz.gemm(m, w_t.shape[0], w_t.shape[1], a=DRef(xt), rows=rows, b=DRef(w_t), d=DRef(out))
    return out


def _self_attn_rows(xt, rows, m, wq, wk, wv, scale):
    q = _proj(xt, rows, m, _dev2d(wq.T))
    k = _proj(xt, rows, m, _dev2d(wk.T))
    v = _proj(xt, rows, m, _dev2d(wv.T))
    return _apply(_scores(q, k, scale, m, m), _vt(v, m), m, m)


def sparse_self_attention(x, wq, wk, wv, scale, ctx, mask: BinaryMask):
    """Attention among the gathered active tokens only (sparse.py:265-300)."""
    _check_attn(x, ctx, mask)
    require_tensor4(x, "sparse_self_attention input")
    n, c, h, w = x.shape
    rows, index, na = _active(mask)
    if na == 0:
        return _cached(ctx, x.shape).copy()
    base = np.zeros(x.shape, np.float32) if mask.all_active() else _cached(ctx, x.shape)
    out = _self_attn_rows(_nhwc(x), rows, na, wq, wk, wv, scale)
    return _finite("attention", _finish(out, index, na, base, c, h, w))


def sparse_cross_attention(x, text_k, text_v, wq, scale, ctx, mask: BinaryMask):
    """Active rows against all text tokens (sparse.py:303-338)."""
    _check_attn(x, ctx, mask)
    require_tensor4(x, "sparse_cross_attention input")
    if text_k.shape[0] != text_v.shape[0]:
        raise ContractViolation(f"text k rows {text_k.shape} != text v rows {text_v.shape}")
    n, c, h, w = x.shape
    rows, index, na = _active(mask)
    if na == 0:
        return _cached(ctx, x.shape).copy()
    base = np.zeros(x.shape, np.float32) if mask.all_active() else _cached(ctx, x.shape)
    q = _proj(_nhwc(x), rows, na, _dev2d(wq.T))
    nk = text_k.shape[0]
    out = _apply(_scores(q, _dev2d(text_k), scale, na, nk), _vt(_dev2d(text_v), nk), na, nk)
    return _finite("attention", _finish(out, index, na, base, c, h, w))


def dense_self_attention(x, wq, wk, wv, scale):
    require_tensor4(x, "dense_self_attention input")
    n, c, h, w = x.shape
    if n != 1:
        raise ContractViolation(f"sparse attention handles single-sample maps, got batch {n}")
    out = _self_attn_rows(_nhwc(x), None, h * w, wq, wk, wv, scale)
    return _finite("attention", _nchw(out, c, h, w))


def dense_cross_attention(x, text_k, text_v, wq, scale):
    require_tensor4(x, "dense_cross_attention input")
    n, c, h, w = x.shape
    if n != 1:
        raise ContractViolation(f"sparse attention handles single-sample maps, got batch {n}")
    q = _proj(_nhwc(x), None, h * w, _dev2d(wq.T))
    nk = text_k.shape[0]
    P = _scores(q, _dev2d(text_k), scale, h * w, nk)
    out = _apply(P, _vt(_dev2d(text_v), nk), h * w, nk)
    return _finite("attention", _nchw(out, c, h, w)), P[:, :nk].contiguous().cpu().numpy()
