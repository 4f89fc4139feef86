"""fp32 operands on the tensor cores (precision "tf32x3": tcgen05 kind::tf32 with a 3xTF32 split,
big*big + big*small + small*big, fp32 accumulation).

Kernel level the GEMM is checked against float64 torch on the same fp32 inputs (rows mode with
K tails and split-K, the implicit 3x3 select-on-read conv with the GN+SiLU epilogue): a 3xTF32
product is exact to ~2^-21 relative per term, so the bound is fp32-GEMM-like: max-abs error
<= 2e-6 * sqrt(K) relative to the output scale (a plain TF32 GEMM misses it by ~100x); the
tensor core's fp32 accumulate truncates (~2^-24 per MMA, linear in K), so the kernel spreads the
big*big products over 7 TMEM accumulators and the small products into an 8th, summed in fp32
round-to-nearest in the epilogue (measured: at or below cuBLAS fp32's error, e.g. 1.9e-6 vs
1.2e-5 at K = 2880).
Pipeline level the mode is held to the fp32 parity bounds (tests/test_gpu_c2_parity.py
parametrises it too): C1 edit latent <= 1e-3 vs the reference golden vectors.
"""

import ast
import ctypes
import math

import numpy as np
import pytest
import torch

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA GPU")]


@pytest.fixture(scope="module")
def env():
    from paper_2305_17423_b200 import _lib as L
    from paper_2305_17423_b200.engine import DRef, Launcher
    return L, DRef, Launcher("tf32x3")


def _tol(ref, k):
    return 2e-6 * max(1.0, ref.abs().max().item()) * math.sqrt(k)


@pytest.mark.parametrize("m,n,k,ld", [(200, 320, 320, 320), (400, 77, 320, 320), (37, 640, 401, 404),
                                      (256, 1280, 2880, 2880), (64, 1280, 11520, 11520)])
@pytest.mark.parametrize("splits", [1, 0])
def test_rows_gemm_tf32x3_vs_f64(env, m, n, k, ld, splits):
    L, DRef, lz = env
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n)
    A = torch.zeros((m, ld), device="cuda")
    A[:, :k] = torch.randn((m, k), device="cuda", generator=g)
    B = torch.randn((n, ld), device="cuda", generator=g) / math.sqrt(k)
    bias = torch.randn(n, device="cuda", generator=g)
    ref = A[:, :k].double() @ B[:, :k].double().t() + bias.double()
    D = torch.full((m, n), float("nan"), device="cuda")
    lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D), bias=bias, splits=splits)
    assert L.lib().fis_gemm_kernel_kind(ctypes.byref(lz.last_gemm)) == 3  # the 3xTF32 tcgen05 kernel ran
    torch.cuda.synchronize()
    err = (D.double() - ref).abs().max().item()
    f32 = (A[:, :k] @ B[:, :k].t() + bias).double()  # torch fp32 (cuBLAS; TF32 off by default)
    print(f"3xTF32 m={m} n={n} k={k} splits={splits}: max-abs {err:.3e} (torch fp32 {(f32 - ref).abs().max().item():.3e})")
    assert err <= _tol(ref, k), (err, _tol(ref, k))


def test_conv_gather_gn_silu_tf32x3(env):
    """Implicit 3x3 conv over concat(upsample(coarse fresh+cache), fine fresh+cache) with
    select-on-read and the cached-stat GN+SiLU epilogue, fp32 operands."""
    L, DRef, lz = env
    g = torch.Generator(device="cuda").manual_seed(3)
    H = W = 32
    c_up, c_sk, n = 64, 32, 96
    mask = torch.zeros(H * W, dtype=torch.bool, device="cuda")
    mask.view(H, W)[9:20, 5:17] = True
    rows = torch.nonzero(mask).flatten().int()
    idx = torch.full((H * W,), -1, dtype=torch.int32, device="cuda")
    idx[rows.long()] = torch.arange(rows.numel(), dtype=torch.int32, device="cuda")
    cm = mask.view(H // 2, 2, W // 2, 2).any(3).any(1).flatten()
    crow = torch.nonzero(cm).flatten().int()
    cidx = torch.full(((H // 2) * (W // 2),), -1, dtype=torch.int32, device="cuda")
    cidx[crow.long()] = torch.arange(crow.numel(), dtype=torch.int32, device="cuda")
    sk_cache = torch.randn((H * W, c_sk), device="cuda", generator=g)
    sk_fresh = torch.randn((rows.numel(), c_sk), device="cuda", generator=g)
    up_cache = torch.randn(((H // 2) * (W // 2), c_up), device="cuda", generator=g)
    up_fresh = torch.randn((crow.numel(), c_up), device="cuda", generator=g)
    Wt = torch.randn((n, 9 * (c_up + c_sk)), device="cuda", generator=g) / 30
    bias = torch.randn(n, device="cuda", generator=g) * 0.1
    groups = 8
    mean = torch.randn((1, groups), device="cuda", generator=g) * 0.1
    var = torch.rand((1, groups), device="cuda", generator=g) + 0.5
    gamma = torch.randn(n, device="cuda", generator=g)
    beta = torch.randn(n, device="cuda", generator=g)
    skf = sk_cache.double().clone()
    skf[rows.long()] = sk_fresh.double()
    upf = up_cache.double().clone()
    upf[crow.long()] = up_fresh.double()
    upm = upf.view(H // 2, W // 2, c_up).repeat_interleave(2, 0).repeat_interleave(2, 1)
    full = torch.cat([upm, skf.view(H, W, c_sk)], dim=2).permute(2, 0, 1)[None]
    wconv = Wt.double().view(n, 3, 3, c_up + c_sk).permute(0, 3, 1, 2)
    conv = torch.nn.functional.conv2d(full, wconv, bias.double(), padding=1)[0].permute(1, 2, 0).reshape(H * W, n)
    conv = conv[rows.long()]
    cg = conv.view(-1, groups, n // groups)
    y = ((cg - mean.double()[0][None, :, None]) / torch.sqrt(var.double()[0][None, :, None] + 1e-5)).reshape(-1, n)
    y = y * gamma.double() + beta.double()
    ref = y * torch.sigmoid(y)
    srcs = [L.Src(DRef(up_fresh).ref(), DRef(up_cache).ref(), L.ptr(cidx), H // 2, W // 2, c_up, 1),
            L.Src(DRef(sk_fresh).ref(), DRef(sk_cache).ref(), L.ptr(idx), H, W, c_sk, 0)]
    for splits in (1, 2):
        D = torch.full((rows.numel(), n), float("nan"), device="cuda")
        lz.gemm(rows.numel(), n, 9 * (c_up + c_sk), rows=rows, srcs=srcs, out_hw=(H, W), b=DRef(Wt), d=DRef(D),
                bias=bias, epi=L.EPI_GN_SILU, gn=(DRef(mean), DRef(var), gamma, beta, groups), splits=splits)
        torch.cuda.synchronize()
        err = (D.double() - ref).abs().max().item()
        assert err <= 5e-5, (splits, err)  # K = 864, GN-amplified


def test_c1_edit_tf32x3_matches_reference(golden_dir):
    """The C1 oracle config (medium golden: 64x64, 20 steps) generated and edited in tf32x3."""
    import paper_2305_17423_b200 as P
    gd = dict(np.load(golden_dir / "medium.npz"))
    cfg = P.UNetConfig(**ast.literal_eval(str(gd["config_json"])))
    P.set_precision("tf32x3")
    try:
        store = P.CacheStore()
        final = P.generate_dense(P.PromptTokens((3, 5, 7, 11)), cfg, store, record="engine")
        assert np.abs(final - gd["final_old"]).max() <= 1e-3
        masks = [k[5:-5] for k in gd if k.startswith("edit_") and k.endswith("_mask")]
        for mname in masks:
            bits = gd[f"edit_{mname}_mask"]
            res = P.edit(P.EditSession.create((3, 5, 7, 11), (3, 5, 9, 11), cfg, store, user_mask=P.BinaryMask(bits)),
                         cfg, store)
            err = float(np.abs(res.latent - gd[f"edit_{mname}_latent"]).max())
            print(f"C1 tf32x3 edit {mname}: max-abs {err:.3e}")
            assert err <= 1e-3, (mname, err)
            if not bits.all():
                assert np.array_equal(res.latent[:, :, ~bits], final[:, :, ~bits])
    finally:
        P.set_precision("fp32")
