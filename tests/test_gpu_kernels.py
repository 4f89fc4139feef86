"""Kernel-level GPU tests: the tcgen05 bf16 gather-GEMM against the SIMT fp32 kernel and a
plain torch fp32 reference, over the gather modes and fused epilogues the engine uses.

Tolerance: both paths consume the same bf16 operands and accumulate in fp32, so they differ
only by summation order: max-abs <= 2e-3 * sqrt(K/64) relative to the output scale.
"""

import os
import math

import numpy as np
import pytest
import torch

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA GPU")]


@pytest.fixture(scope="module")
def env():
    from paper_2305_17423_b200 import _lib as L
    from paper_2305_17423_b200.engine import NULL, DRef, Launcher
    return L, DRef, NULL, Launcher("bf16")


def _run(env, impl, m, n, k, **kw):
    L, DRef, NULL, lz = env
    lz.gemm_impl = impl
    lz.gemm(m, n, k, **kw)
    torch.cuda.synchronize()


def _tol(ref, k):
    return 3e-3 * max(1.0, ref.abs().max().item()) * math.sqrt(max(k, 64) / 64)


@pytest.mark.parametrize("m,n,k,ld", [(200, 320, 320, 320), (400, 77, 320, 320), (37, 640, 401, 416),
                                      (256, 1280, 2880, 2880), (1024, 256, 640, 640)])
@pytest.mark.parametrize("splits", [1, 3])
def test_rows_gemm_tc_vs_simt(env, m, n, k, ld, splits):
    L, DRef, NULL, lz = env
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n)
    A = torch.zeros((m, ld), device="cuda", dtype=torch.bfloat16)
    A[:, :k] = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn((n, ld), device="cuda", generator=g).to(torch.bfloat16) / math.sqrt(k)
    bias = torch.randn(n, device="cuda", generator=g)
    ref = A[:, :k].float() @ B[:, :k].float().t() + bias
    outs = []
    for impl in (1, 2):
        D = torch.full((m, n), float("nan"), device="cuda")
        _run(env, impl, m, n, k, a=DRef(A), b=DRef(B), d=DRef(D), bias=bias, splits=splits)
        outs.append(D)
    assert (outs[1] - ref).abs().max().item() <= _tol(ref, k)
    assert (outs[0] - ref).abs().max().item() <= _tol(ref, k)


def test_conv_gather_select_upsample_tc_vs_simt(env):
    """Implicit 3x3 conv over concat(upsample(coarse compact+cache), fine compact+cache) with
    select-on-read, GN+SiLU epilogue, as the sparse fuse/block convs use it."""
    L, DRef, NULL, lz = env
    g = torch.Generator(device="cuda").manual_seed(3)
    H = W = 32
    c_up, c_sk, n = 128, 64, 192
    bf = torch.bfloat16
    mask = torch.zeros(H * W, dtype=torch.bool, device="cuda")
    mask.view(H, W)[9:20, 5:17] = True
    mask.view(H, W)[25, 30] = True
    rows = torch.nonzero(mask).flatten().int()
    idx = torch.full((H * W,), -1, dtype=torch.int32, device="cuda")
    idx[rows.long()] = torch.arange(rows.numel(), dtype=torch.int32, device="cuda")
    cm = mask.view(H // 2, 2, W // 2, 2).any(3).any(1).flatten()
    crow = torch.nonzero(cm).flatten().int()
    cidx = torch.full(((H // 2) * (W // 2),), -1, dtype=torch.int32, device="cuda")
    cidx[crow.long()] = torch.arange(crow.numel(), dtype=torch.int32, device="cuda")
    sk_cache = torch.randn((H * W, c_sk), device="cuda", generator=g).to(bf)
    sk_fresh = torch.randn((rows.numel(), c_sk), device="cuda", generator=g).to(bf)
    up_cache = torch.randn(((H // 2) * (W // 2), c_up), device="cuda", generator=g).to(bf)
    up_fresh = torch.randn((crow.numel(), c_up), device="cuda", generator=g).to(bf)
    Wt = (torch.randn((n, 9 * (c_up + c_sk)), device="cuda", generator=g) / 40).to(bf)
    bias = torch.randn(n, device="cuda", generator=g) * 0.1
    groups = 8
    mean = torch.randn((1, groups), device="cuda", generator=g) * 0.1
    var = torch.rand((1, groups), device="cuda", generator=g) + 0.5
    gamma = torch.randn(n, device="cuda", generator=g)
    beta = torch.randn(n, device="cuda", generator=g)
    # torch reference: materialise the full input map and run conv
    skf = sk_cache.float().clone()
    skf[rows.long()] = sk_fresh.float()
    upf = up_cache.float().clone()
    upf[crow.long()] = up_fresh.float()
    upm = upf.view(H // 2, W // 2, c_up).repeat_interleave(2, 0).repeat_interleave(2, 1)
    full = torch.cat([upm, skf.view(H, W, c_sk)], dim=2).permute(2, 0, 1)[None]
    wconv = Wt.float().view(n, 3, 3, c_up + c_sk).permute(0, 3, 1, 2)
    conv = torch.nn.functional.conv2d(full, wconv, bias, padding=1)[0].permute(1, 2, 0).reshape(H * W, n)[rows.long()]
    cg = conv.view(-1, groups, n // groups)
    y = ((cg - mean[0][None, :, None]) / torch.sqrt(var[0][None, :, None] + 1e-5)).reshape(-1, n) * gamma + beta
    ref = y * torch.sigmoid(y)
    srcs = [L.Src(DRef(up_fresh).ref(), DRef(up_cache).ref(), L.ptr(cidx), H // 2, W // 2, c_up, 1),
            L.Src(DRef(sk_fresh).ref(), DRef(sk_cache).ref(), L.ptr(idx), H, W, c_sk, 0)]
    outs = []
    for impl in (1, 2):
        D = torch.full((rows.numel(), n), float("nan"), device="cuda")
        _run(env, impl, rows.numel(), n, 9 * (c_up + c_sk), rows=rows, srcs=srcs, out_hw=(H, W), b=DRef(Wt),
             d=DRef(D), bias=bias, epi=L.EPI_GN_SILU, gn=(DRef(mean), DRef(var), gamma, beta, groups), splits=2)
        outs.append(D)
    for o in outs:
        assert (o - ref).abs().max().item() <= 2e-2, (o - ref).abs().max().item()
    assert (outs[0] - outs[1]).abs().max().item() <= 2e-3


def test_transposed_store_and_residual(env):
    L, DRef, NULL, lz = env
    g = torch.Generator(device="cuda").manual_seed(9)
    m, n, k = 300, 320, 320
    A = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn((n, k), device="cuda", generator=g) / 18).to(torch.bfloat16)
    res = torch.randn((m, n), device="cuda", generator=g).to(torch.bfloat16)
    ref = A.float() @ B.float().t()
    for impl in (1, 2):
        Dt = torch.zeros((n, 304), device="cuda", dtype=torch.bfloat16)
        _run(env, impl, m, n, k, a=DRef(A), b=DRef(B), d=DRef(Dt), d_trans=True)
        assert (Dt[:, :m].float().t() - ref).abs().max().item() <= 3e-2
        D = torch.zeros((m, n), device="cuda")
        _run(env, impl, m, n, k, a=DRef(A), b=DRef(B), d=DRef(D), res=DRef(res))
        assert (D - (ref + res.float())).abs().max().item() <= 3e-2


@pytest.mark.parametrize("m,nk,d", [(400, 400, 320), (100, 100, 640), (256, 256, 1280), (64, 64, 1280),
                                    (400, 77, 320), (1024, 1024, 320), (37, 5, 64), (300, 129, 128),
                                    # d-split clusters (<= 128 keys, small grids): cs = 5, 4, 3, 2 value slices
                                    (256, 77, 1280), (64, 77, 1280), (100, 77, 640), (200, 50, 768), (130, 128, 512),
                                    # two-round d-split (129-256 keys): cs = 5, 4
                                    (200, 190, 1280), (256, 129, 1024), (64, 256, 1280),
                                    # split-KV (runs of >= 8 key blocks on small grids)
                                    (130, 1100, 320), (128, 1024, 640), (50, 1500, 256),
                                    # short-run kernel (>= 16 query tiles, <= 128 keys)
                                    (4096, 77, 320), (2100, 128, 640), (3000, 20, 1280)])
@pytest.mark.parametrize("short", ["1", "0"])  # "0": the general kernel's modes (d-split, single block, ...)
def test_fused_attention_vs_torch(env, m, nk, d, short):
    """fis_attn (tcgen05 S=QK^T, softmax, P.V, + residual) against torch fp32 on the same bf16 inputs."""
    L, DRef, NULL, lz = env
    os.environ["FIS_ATTN_SHORT"] = short
    g = torch.Generator(device="cuda").manual_seed(m + nk + d)
    bf = torch.bfloat16
    Q = torch.randn((m, d), device="cuda", generator=g).to(bf)
    K = torch.randn((nk, d), device="cuda", generator=g).to(bf)
    V = torch.randn((nk, d), device="cuda", generator=g).to(bf)
    ldv = (nk + 15) // 16 * 16
    Vt = torch.zeros((d, ldv), device="cuda", dtype=bf)
    Vt[:, :nk] = V.t()
    res = torch.randn((m, d), device="cuda", generator=g).to(bf)
    scale = 1.0 / math.sqrt(d)
    P = torch.softmax(Q.float() @ K.float().t() * scale, dim=1)
    ref = P @ V.float() + res.float()
    out = torch.full((m, d), float("nan"), device="cuda", dtype=bf)
    a = L.AttnArgs(m, nk, d, d, DRef(Q).ref(), DRef(K).ref(), DRef(Vt, ld=ldv).ref(), scale, DRef(res).ref(), NULL,
                   DRef(out).ref(), None)
    # the engine's workspace (zeroed): lets long runs on small grids take the split-KV path
    nb = int(L.lib().fis_attn_ws_bytes(m, nk, d))
    ws = torch.zeros(nb, device="cuda", dtype=torch.uint8)
    a.max_seg_k, a.ws, a.ws_bytes = nk, L.ptr(ws), nb
    L.call("fis_attn", a)
    torch.cuda.synchronize()
    os.environ.pop("FIS_ATTN_SHORT", None)
    err = (out.float() - ref).abs().max().item()
    assert err <= 3e-2 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("d,qlens,klens,kpad", [
    (320, [205, 410, 1024, 0, 37], None, 0),          # self-attention: keys = own rows
    (640, [64, 300, 129], [77, 77, 77], 80),           # cross-attention: stacked prompts padded to 80
    (1280, [256, 256, 256], None, 0),
    (640, [100, 256, 17], None, 0),
    # >= 16 query tiles with every key run <= 128: the persistent short-run kernel (fis_attn_short.cu)
    (320, [205, 410, 1024, 77, 300, 0, 515] * 3, [77, 60, 77, 1, 77, 77, 33] * 3, 80),
    (1280, [64] * 40, None, 0),
    (640, [128, 200, 17, 256] * 6, [77] * 24, 80),
    # 129-256-key runs on >= 16 query tiles: the short-run kernel's 256-key configuration
    (1280, [256] * 10, None, 0),
    (640, [200, 150, 256, 129, 0] * 5, None, 0)])
@pytest.mark.parametrize("share", [False, True])
def test_segment_attention_vs_torch(env, d, qlens, klens, kpad, share):
    """fis_attn with ragged segments (batched requests): each query run attends to its own key run only."""
    L, DRef, NULL, lz = env
    g = torch.Generator(device="cuda").manual_seed(d + len(qlens))
    bf = torch.bfloat16
    starts = [0]
    for n in qlens:  # runs padded to 16 rows like BatchedEditPlan
        starts.append(starts[-1] + (n + 15) // 16 * 16)
    m = starts[-1]
    Q = torch.randn((m, d), device="cuda", generator=g).to(bf)
    res = torch.randn((m, d), device="cuda", generator=g).to(bf)
    if klens is None:  # self
        K = torch.randn((m, d), device="cuda", generator=g).to(bf)
        V = torch.randn((m, d), device="cuda", generator=g).to(bf)
        kseg = [(starts[i], starts[i] + qlens[i]) for i in range(len(qlens))]
    else:
        nk = kpad * len(klens)
        K = torch.randn((nk, d), device="cuda", generator=g).to(bf)
        V = torch.randn((nk, d), device="cuda", generator=g).to(bf)
        kseg = [(kpad * i, kpad * i + klens[i]) for i in range(len(klens))]
    nk = K.shape[0]
    ldv = (nk + 15) // 16 * 16
    Vt = torch.zeros((d, ldv), device="cuda", dtype=bf)
    Vt[:, :nk] = V.t()
    qseg = [(starts[i], starts[i] + qlens[i]) for i in range(len(qlens))]
    qs = torch.tensor([v for p in qseg for v in p], dtype=torch.int32, device="cuda")
    ks = torch.tensor([v for p in kseg for v in p], dtype=torch.int32, device="cuda")
    scale = 1.0 / math.sqrt(d)
    out = torch.zeros((m, d), device="cuda", dtype=bf)
    a = L.AttnArgs(m, nk, d, d, DRef(Q).ref(), DRef(K).ref(), DRef(Vt, ld=ldv).ref(), scale, DRef(res).ref(), NULL,
                   DRef(out).ref(), None)
    a.nseg, a.max_seg_q, a.q_seg, a.k_seg = len(qseg), max(1, max(qlens)), L.ptr(qs), L.ptr(ks)
    max_k = max(k1 - k0 for k0, k1 in kseg)
    if share:  # value slices share one P per query tile through the scratch [m, 128 * ceil(max_k / 128)]
        ws = torch.empty(m * ((max_k + 127) // 128 * 128), device="cuda", dtype=bf)
        a.max_seg_k, a.ws, a.ws_bytes = max_k, L.ptr(ws), ws.numel() * 2
        os.environ["FIS_ATTN_SHORT"] = "0"  # the general kernel's P_OUT / P_IN sharing
    else:
        a.max_seg_k = max_k  # the short-run kernel for runs <= 256 keys
    L.call("fis_attn", a)
    torch.cuda.synchronize()
    os.environ.pop("FIS_ATTN_SHORT", None)
    for (q0, q1), (k0, k1) in zip(qseg, kseg):
        if q1 == q0:
            continue
        P = torch.softmax(Q[q0:q1].float() @ K[k0:k1].float().t() * scale, dim=1)
        ref = P @ V[k0:k1].float() + res[q0:q1].float()
        err = (out[q0:q1].float() - ref).abs().max().item()
        assert err <= 3e-2 * max(1.0, ref.abs().max().item()), (q0, q1, err)
    # padding rows between runs are not written
    for i in range(len(qlens)):
        assert (out[qseg[i][1]:starts[i + 1]] == 0).all()
