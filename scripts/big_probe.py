"""Persistent large-M GEMM (csrc/fis_gemm_big.cu) vs the per-op tcgen05 kernel: bitwise check and
timing on stacked-request shapes (dense conv over R images, gathered conv rows, plain rows)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_17423_b200 import _lib as L  # noqa: E402
from paper_2305_17423_b200.engine import DRef, Launcher, NULL  # noqa: E402

lz = Launcher("bf16")
g = torch.Generator(device="cuda").manual_seed(0)
dev = "cuda"


def rnd(*shape, scale=1.0):
    return (torch.randn(shape, device=dev, generator=g) * scale).to(torch.bfloat16)


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def both(name, m, n, k, run, out):
    res = {}
    for big in ("1", "0"):
        os.environ["FIS_BIG"] = big
        out.zero_()
        run()
        torch.cuda.synchronize()
        res[big] = (out.clone(), timeit(run))
    os.environ.pop("FIS_BIG", None)
    d = (res["1"][0].float() - res["0"][0].float()).abs().max().item()
    fl = 2.0 * m * n * k
    print(f"{name:28s} m={m:6d} n={n:5d} k={k:6d}  big {res['1'][1]:8.1f} us {fl / res['1'][1] / 1e6:7.1f} TF/s | "
          f"per-op {res['0'][1]:8.1f} us {fl / res['0'][1] / 1e6:7.1f} TF/s | maxdiff {d:.3g}", flush=True)
    return d


def conv_dense(R, h, w, cin, cout):
    x = rnd(R * h * w, cin)
    W = rnd(cout, 9 * cin, scale=1 / math.sqrt(9 * cin))
    bias = torch.randn(cout, device=dev, generator=g)
    out = torch.empty((R * h * w, cout), device=dev, dtype=torch.bfloat16)
    src = L.Src(DRef(x).ref(), NULL, None, h, w, cin, 0)
    m = R * h * w
    run = lambda: lz.gemm(m, cout, 9 * cin, srcs=[src], out_hw=(h, w), b=DRef(W), d=DRef(out), bias=bias)
    return both(f"conv dense R={R} {h}x{w}", m, cout, 9 * cin, run, out)


def conv_gather(R, h, w, cin, cout, frac):
    hw = h * w
    cache = rnd(R * hw, cin)
    # one square per image (the bench's user masks), at an image-dependent offset
    act = torch.zeros((R, h, w), dtype=torch.bool, device=dev)
    side = max(1, int(round((frac * hw) ** 0.5)))
    for r in range(R):
        y0, x0 = (7 * r) % (h - side + 1), (13 * r) % (w - side + 1)
        act[r, y0:y0 + side, x0:x0 + side] = True
    act = act.flatten()
    rows = act.nonzero().flatten().to(torch.int32)
    n = rows.numel()
    index = torch.full((R * hw,), -1, dtype=torch.int32, device=dev)
    index[rows.long()] = torch.arange(n, dtype=torch.int32, device=dev)
    fresh = rnd(n, cin)
    W = rnd(cout, 9 * cin, scale=1 / math.sqrt(9 * cin))
    out = torch.empty((n, cout), device=dev, dtype=torch.bfloat16)
    src = L.Src(DRef(fresh).ref(), DRef(cache).ref(), L.ptr(index), h, w, cin, 0)
    run = lambda: lz.gemm(n, cout, 9 * cin, rows=rows, srcs=[src], out_hw=(h, w), b=DRef(W), d=DRef(out))
    return both(f"conv gather R={R} {frac:.2f}", n, cout, 9 * cin, run, out)


def rows_gemm(m, n, k):
    A = rnd(m, k)
    B = rnd(n, k, scale=1 / math.sqrt(k))
    out = torch.empty((m, n), device=dev, dtype=torch.bfloat16)
    run = lambda: lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(out))
    d = both("rows", m, n, k, run, out)
    ref = (A.float() @ B.float().t())
    e = (out.float() - ref).abs().max().item()
    t = timeit(lambda: torch.matmul(A, B.t()))
    print(f"{'':28s} vs fp32 matmul maxdiff {e:.3g}; cuBLAS bf16 {t:.1f} us {2.0 * m * n * k / t / 1e6:.1f} TF/s")
    return d


if len(sys.argv) > 1 and sys.argv[1] == "medium":
    for (m, n, k) in [(256, 256, 512), (256, 256, 1024), (1024, 1024, 1024), (4096, 3840, 1280)]:
        rows_gemm(m, n, k)
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "small":
    rows_gemm(256, 256, 128)
    conv_dense(2, 16, 16, 64, 128)
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    rows_gemm(4096, 3840, 1280)
    conv_dense(32, 16, 16, 1280, 1280)
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "gtrace":
    import ctypes
    conv_gather(32, 64, 64, 320, 320, 0.12)
    buf = (ctypes.c_ulonglong * 768)()
    L.lib().fis_big_trace_read(buf)
    t = list(buf)
    t0 = min(x for x in t if x)
    for i in range(0, 60):
        print(i, [(t[r * 256 + i] - t0) if t[r * 256 + i] else None for r in range(3)])
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "trace":
    import ctypes
    os.environ["FIS_BIG"] = "1"
    A, B = rnd(8192, 1280), rnd(1280, 1280, scale=1 / 36)
    out = torch.empty((8192, 1280), device=dev, dtype=torch.bfloat16)
    for _ in range(2):
        lz.gemm(8192, 1280, 1280, a=DRef(A), b=DRef(B), d=DRef(out))
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 768)()
    L.lib().fis_big_trace_read(buf)
    t = list(buf)
    t0 = min(x for x in t if x)
    for i in range(0, 60):
        print(i, [(t[r * 256 + i] - t0) if t[r * 256 + i] else None for r in range(3)])
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "one":  # one big-kernel launch of each kind (ncu)
    os.environ["FIS_BIG"] = "1"
    A, B = rnd(4096, 1280), rnd(3840, 1280, scale=1 / 36)
    out = torch.empty((4096, 3840), device=dev, dtype=torch.bfloat16)
    lz.gemm(4096, 3840, 1280, a=DRef(A), b=DRef(B), d=DRef(out))
    torch.cuda.synchronize()
    sys.exit(0)
worst = 0.0
worst = max(worst, rows_gemm(4096, 3840, 1280))
worst = max(worst, rows_gemm(8192, 1280, 1280))
worst = max(worst, rows_gemm(3872, 960, 320))
for R in (8, 32):
    worst = max(worst, conv_dense(R, 16, 16, 1280, 1280))
    worst = max(worst, conv_dense(R, 8, 8, 1280, 1280))
    worst = max(worst, conv_gather(R, 64, 64, 320, 320, 0.12))
    worst = max(worst, conv_gather(R, 32, 32, 640, 640, 0.15))
worst = max(worst, conv_dense(8, 64, 64, 320, 320))
print("WORST", worst)
