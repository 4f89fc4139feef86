"""GPU tests of the persistent large-M GEMM (csrc/fis_gemm_big.cu), the kernel fis_gemm picks once
the tiles fill the GPU (stacked requests). Every staging mode must give bitwise the same result
as the per-op tcgen05 kernel (FIS_BIG=0): same bf16 operands, same K order, fp32 accumulation.
  * TMA rows (contiguous A), incl. the fused QKV split with a transposed V^T output;
  * dense stacked 3x3 conv with 4-D TMA taps (zero padding at every image border);
  * select-on-read gathered conv (TMA gather4 + cp.async), 320-wide tiles (two MMAs per K block);
  * epilogues: bias, residual, GN + SiLU with cached statistics.
"""

import math
import os

import pytest
import torch

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA GPU")]


@pytest.fixture(scope="module")
def env():
    from paper_2305_17423_b200 import _lib as L
    from paper_2305_17423_b200.engine import DRef, Launcher, NULL
    return L, DRef, NULL, Launcher("bf16")


def _kind(lz):
    """Kernel fis_gemm picked for the launcher's last GEMM (2 = persistent large-M kernel)."""
    import ctypes
    from paper_2305_17423_b200 import _lib as L
    return L.lib().fis_gemm_kernel_kind(ctypes.byref(lz.last_gemm))


def _both(run, out):
    """Run with the persistent kernel, then with the per-op kernel (FIS_BIG=0); also checks that
    the first run really launched the persistent kernel (no silent fallback)."""
    from paper_2305_17423_b200 import _lib as L
    res = []
    os.environ["FIS_PAIR"] = "0"  # the single-SM persistent kernel (the CTA-pair kernel has its own tests)
    for big in ("1", "0"):
        os.environ["FIS_BIG"] = big
        out.zero_()
        n0 = L.lib().fis_gemm_big_launch_count()
        run()
        torch.cuda.synchronize()
        if big == "1":
            assert L.lib().fis_gemm_big_launch_count() > n0, "persistent GEMM fell back to the per-op kernel"
        res.append(out.clone())
    os.environ.pop("FIS_BIG", None)
    os.environ.pop("FIS_PAIR", None)
    return res


def _rnd(g, *shape, scale=1.0):
    return (torch.randn(shape, device="cuda", generator=g) * scale).to(torch.bfloat16)


def test_rows_and_qkv_split(env):
    L, DRef, NULL, lz = env
    g = torch.Generator(device="cuda").manual_seed(1)
    m, k, c = 8192, 320, 320
    A = _rnd(g, m, k)
    B = _rnd(g, 3 * c, k, scale=1 / math.sqrt(k))
    res = _rnd(g, m, c)
    bias = torch.randn(c, device="cuda", generator=g)
    D = torch.empty((m, c), device="cuda", dtype=torch.bfloat16)
    r = _both(lambda: lz.gemm(m, c, k, a=DRef(A), b=DRef(B), d=DRef(D), bias=bias, res=DRef(res)), D)
    assert _kind(lz) in (2, 6)  # persistent single-SM or CTA-pair kernel for this shape
    assert torch.equal(r[0], r[1])
    ref = (A.float() @ B[:c].float().t() + bias + res.float())
    assert (r[0].float() - ref).abs().max().item() <= 5e-2
    qk = torch.empty((m, 2 * c), device="cuda", dtype=torch.bfloat16)
    vt = torch.zeros((c, m), device="cuda", dtype=torch.bfloat16)
    outs = []
    for big in ("1", "0"):
        os.environ["FIS_BIG"] = big
        qk.zero_()
        vt.zero_()
        lz.gemm(m, 3 * c, k, a=DRef(A), b=DRef(B), d=DRef(qk), n_split=2 * c, d2=DRef(vt, ld=m), d2_trans=True)
        torch.cuda.synchronize()
        outs.append((qk.clone(), vt.clone()))
    os.environ.pop("FIS_BIG", None)
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("R,h,w,cin,cout", [(32, 16, 16, 128, 256), (160, 8, 8, 128, 256), (4, 64, 64, 64, 320),
                                             (16, 16, 16, 128, 1280)])  # last: 320-wide tiles (1 wave)
def test_dense_stacked_conv(env, R, h, w, cin, cout):
    L, DRef, NULL, lz = env
    g = torch.Generator(device="cuda").manual_seed(R + h)
    hw = h * w
    x = _rnd(g, R * hw, cin)
    W = _rnd(g, cout, 9 * cin, scale=1 / math.sqrt(9 * cin))
    out = torch.empty((R * hw, cout), device="cuda", dtype=torch.bfloat16)
    src = L.Src(DRef(x).ref(), NULL, None, h, w, cin, 0)
    r = _both(lambda: lz.gemm(R * hw, cout, 9 * cin, srcs=[src], out_hw=(h, w), b=DRef(W), d=DRef(out)), out)
    assert _kind(lz) in (2, 6)  # persistent single-SM or CTA-pair kernel for this shape
    assert torch.equal(r[0], r[1])
    xi = x.float().reshape(R, h, w, cin).permute(0, 3, 1, 2)
    Wk = W.float().reshape(cout, 3, 3, cin).permute(0, 3, 1, 2)
    ref = torch.nn.functional.conv2d(xi, Wk, padding=1).permute(0, 2, 3, 1).reshape(R * hw, cout)
    assert (r[0].float() - ref).abs().max().item() <= 5e-2


def test_gathered_conv_with_gn_silu(env):
    L, DRef, NULL, lz = env
    g = torch.Generator(device="cuda").manual_seed(7)
    R, h, w, cin, cout, groups = 48, 32, 32, 128, 320, 32
    hw = h * w
    act = torch.zeros((R, h, w), dtype=torch.bool, device="cuda")
    for r in range(R):
        y0, x0 = (5 * r) % 16, (3 * r) % 16
        act[r, y0:y0 + 14, x0:x0 + 12] = True
    act = act.flatten()
    rows = act.nonzero().flatten().to(torch.int32)
    n = rows.numel()
    index = torch.full((R * hw,), -1, dtype=torch.int32, device="cuda")
    index[rows.long()] = torch.arange(n, dtype=torch.int32, device="cuda")
    cache = _rnd(g, R * hw, cin)
    fresh = _rnd(g, n, cin)
    W = _rnd(g, cout, 9 * cin, scale=1 / math.sqrt(9 * cin))
    bias = torch.randn(cout, device="cuda", generator=g)
    mean = torch.randn((1, groups), device="cuda", generator=g) * 0.1
    var = torch.rand((1, groups), device="cuda", generator=g) + 0.5
    gamma = torch.randn(cout, device="cuda", generator=g)
    beta = torch.randn(cout, device="cuda", generator=g)
    out = torch.empty((n, cout), device="cuda", dtype=torch.bfloat16)
    src = L.Src(DRef(fresh).ref(), DRef(cache).ref(), L.ptr(index), h, w, cin, 0)
    run = lambda: lz.gemm(n, cout, 9 * cin, rows=rows, srcs=[src], out_hw=(h, w), b=DRef(W), d=DRef(out), bias=bias,
                          epi=L.EPI_GN_SILU, gn=(DRef(mean), DRef(var), gamma, beta, groups))
    r = _both(run, out)
    assert _kind(lz) in (2, 6)  # persistent single-SM or CTA-pair kernel for this shape
    assert torch.equal(r[0], r[1])
    # reference: select-on-read map, conv, cached-stat GN, SiLU (fp32 on the same bf16 values)
    full = cache.float().clone()
    full[rows.long()] = fresh.float()
    xi = full.reshape(R, h, w, cin).permute(0, 3, 1, 2)
    Wk = W.float().reshape(cout, 3, 3, cin).permute(0, 3, 1, 2)
    y = torch.nn.functional.conv2d(xi, Wk, bias, padding=1).permute(0, 2, 3, 1).reshape(R * hw, cout)[rows.long()]
    cpg = cout // groups
    mu = mean.repeat_interleave(cpg, dim=1)
    rs = torch.rsqrt(var + 1e-5).repeat_interleave(cpg, dim=1)
    yn = (y - mu) * rs * gamma + beta
    ref = yn * torch.sigmoid(yn)
    assert (r[0].float() - ref).abs().max().item() <= 8e-2


@pytest.mark.parametrize("R,h,w,cout,sparse", [(1, 64, 64, 320, True), (64, 64, 64, 320, True), (2, 16, 16, 64, False)])
def test_small_cin_stem_conv(env, R, h, w, cout, sparse):
    """The latent stem conv (C_in = 4, K = 36, csrc/fis_conv_small.cu): fp32 latent rows with
    select-on-read (fresh active rows / cached latent), bias + per-step time bias, bf16 output,
    against torch fp32 conv2d on the same values."""
    L, DRef, NULL, lz = env
    g = torch.Generator(device="cuda").manual_seed(R + cout)
    cin, hw = 4, h * w
    if sparse:
        act = torch.zeros((R, h, w), dtype=torch.bool, device="cuda")
        for r in range(R):
            y0, x0 = (7 * r) % (h // 2), (5 * r) % (w // 2)
            act[r, y0:y0 + h // 3, x0:x0 + w // 4] = True
        act = act.flatten()
        rows = act.nonzero().flatten().to(torch.int32)
    else:
        rows = None
    n = rows.numel() if sparse else R * hw
    cache = torch.randn((R * hw, cin), device="cuda", generator=g)
    fresh = torch.randn((n, cin), device="cuda", generator=g) if sparse else cache
    W = _rnd(g, cout, 9 * cin, scale=1 / math.sqrt(9 * cin))
    bias = torch.randn(cout, device="cuda", generator=g)
    tbias = torch.randn(cout, device="cuda", generator=g)
    out = torch.empty((n, cout), device="cuda", dtype=torch.bfloat16)
    if sparse:
        index = torch.full((R * hw,), -1, dtype=torch.int32, device="cuda")
        index[rows.long()] = torch.arange(n, dtype=torch.int32, device="cuda")
        src = L.Src(DRef(fresh).ref(), DRef(cache).ref(), L.ptr(index), h, w, cin, 0)
    else:
        src = L.Src(DRef(fresh).ref(), NULL, None, h, w, cin, 0)
    lz.gemm(n, cout, 9 * cin, rows=rows, srcs=[src], out_hw=(h, w), b=DRef(W), d=DRef(out), bias=bias,
            bias2=DRef(tbias))
    torch.cuda.synchronize()
    assert _kind(lz) == 5  # the FMA-pipe stem kernel ran (no SIMT fallback)
    full = cache.clone()
    if sparse:
        full[rows.long()] = fresh
    xi = full.reshape(R, h, w, cin).permute(0, 3, 1, 2)
    Wk = W.float().reshape(cout, 3, 3, cin).permute(0, 3, 1, 2)
    y = torch.nn.functional.conv2d(xi, Wk, bias + tbias, padding=1).permute(0, 2, 3, 1).reshape(R * hw, cout)
    if sparse:
        y = y[rows.long()]
    assert (out.float() - y).abs().max().item() <= 3e-2 * max(1.0, y.abs().max().item())


@pytest.mark.parametrize("R,h,w,cin,cout,two", [(32, 16, 16, 128, 512, False), (8, 32, 32, 128, 256, True),
                                                 (48, 8, 8, 64, 768, False)])
def test_pair_kernel_dense_conv(env, R, h, w, cin, cout, two):
    """The 2-SM CTA-pair GEMM (csrc/fis_gemm_pair.cu, tcgen05 cta_group::2, M = 256): dense stacked
    3x3 conv (one or two concatenated sources, 4-D TMA taps) against the single-SM persistent kernel
    and torch; the pair kernel must really run (launch counter)."""
    import ctypes
    L, DRef, NULL, lz = env
    g = torch.Generator(device="cuda").manual_seed(R + cout)
    hw = h * w
    x = _rnd(g, R * hw, cin)
    x2 = _rnd(g, R * hw, cin) if two else None
    ct = cin * (2 if two else 1)
    W = _rnd(g, cout, 9 * ct, scale=1 / math.sqrt(9 * ct))
    bias = torch.randn(cout, device="cuda", generator=g)
    out = torch.empty((R * hw, cout), device="cuda", dtype=torch.bfloat16)
    srcs = [L.Src(DRef(x).ref(), NULL, None, h, w, cin, 0)]
    if two:
        srcs.append(L.Src(DRef(x2).ref(), NULL, None, h, w, cin, 0))
    res = []
    for mode in ("2", "0"):
        os.environ["FIS_PAIR"] = mode
        out.zero_()
        n0 = L.lib().fis_gemm_pair_launch_count()
        lz.gemm(R * hw, cout, 9 * ct, srcs=srcs, out_hw=(h, w), b=DRef(W), d=DRef(out), bias=bias)
        torch.cuda.synchronize()
        ran = L.lib().fis_gemm_pair_launch_count() > n0
        assert ran == (mode == "2"), "pair kernel launch state"
        if mode == "2":
            assert L.lib().fis_gemm_kernel_kind(ctypes.byref(lz.last_gemm)) == 6
        res.append(out.clone())
    os.environ.pop("FIS_PAIR", None)
    xi = x.float().reshape(R, h, w, cin)
    if two:
        xi = torch.cat([xi, x2.float().reshape(R, h, w, cin)], dim=3)
    Wk = W.float().reshape(cout, 3, 3, ct).permute(0, 3, 1, 2)
    ref = torch.nn.functional.conv2d(xi.permute(0, 3, 1, 2), Wk, bias, padding=1).permute(0, 2, 3, 1).reshape(R * hw, cout)
    assert (res[0].float() - ref).abs().max().item() <= 5e-2
    assert (res[0].float() - res[1].float()).abs().max().item() <= 2e-2  # vs the single-SM kernel


def test_pair_kernel_rows(env):
    L, DRef, NULL, lz = env
    g = torch.Generator(device="cuda").manual_seed(11)
    m, k, n = 5000, 640, 1280  # ragged last pair tile
    A = _rnd(g, m, k)
    B = _rnd(g, n, k, scale=1 / math.sqrt(k))
    res = _rnd(g, m, n)
    D = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    os.environ["FIS_PAIR"] = "2"
    n0 = L.lib().fis_gemm_pair_launch_count()
    lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D), res=DRef(res))
    torch.cuda.synchronize()
    os.environ.pop("FIS_PAIR", None)
    assert L.lib().fis_gemm_pair_launch_count() > n0
    ref = A.float() @ B.float().t() + res.float()
    assert (D.float() - ref).abs().max().item() <= 5e-2


@pytest.mark.parametrize("m,k,c", [(4000, 640, 640), (3001, 320, 320)])  # (the L0 split falls mid-tile)
def test_pair_kernel_qkv_split(env, m, k, c):
    """Fused QKV on the CTA-pair kernel: Q' row-major (TMA-stored boxes at small K), V^T transposed
    into d2 (direct per-column stores)."""
    L, DRef, NULL, lz = env
    g = torch.Generator(device="cuda").manual_seed(12)
    A = _rnd(g, m, k)
    B = _rnd(g, 2 * c, k, scale=1 / math.sqrt(k))
    bias = torch.randn(2 * c, device="cuda", generator=g)
    outs = []
    for mode in ("2", "0"):
        os.environ["FIS_PAIR"] = mode
        qk = torch.zeros((m, c), device="cuda", dtype=torch.bfloat16)
        vt = torch.zeros((c, 4096), device="cuda", dtype=torch.bfloat16)
        n0 = L.lib().fis_gemm_pair_launch_count()
        lz.gemm(m, 2 * c, k, a=DRef(A), b=DRef(B), d=DRef(qk), bias=bias, n_split=c, d2=DRef(vt, ld=4096),
                d2_trans=True)
        torch.cuda.synchronize()
        assert (L.lib().fis_gemm_pair_launch_count() > n0) == (mode == "2")
        outs.append((qk.clone(), vt.clone()))
    os.environ.pop("FIS_PAIR", None)
    ref = A.float() @ B.float().t() + bias
    assert (outs[0][0].float() - ref[:, :c]).abs().max().item() <= 5e-2
    assert (outs[0][1][:, :m].float().t() - ref[:, c:]).abs().max().item() <= 5e-2
    assert (outs[0][0].float() - outs[1][0].float()).abs().max().item() <= 2e-2
    assert (outs[0][1].float() - outs[1][1].float()).abs().max().item() <= 2e-2
