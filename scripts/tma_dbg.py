import os, sys, torch, math
sys.path.insert(0, "/root/repo")
os.environ["FIS_BIG_MIN_TILES"] = "1"
from paper_2305_17423_b200 import _lib as L
from paper_2305_17423_b200.engine import DRef, Launcher, NULL
lz = Launcher("bf16")
R, h, w, cin, cout = 2, 16, 16, 64, 128
hw = h * w
x = torch.zeros((R * hw, cin), device="cuda")
for p in range(R * hw):
    x[p, 0] = p % 64
    x[p, 1] = p // 64
x = x.to(torch.bfloat16)
out = torch.zeros((R * hw, cout), device="cuda", dtype=torch.bfloat16)
src = L.Src(DRef(x).ref(), NULL, None, h, w, cin, 0)
for tap in range(9):
    W = torch.zeros((cout, 9 * cin), device="cuda")
    W[0, tap * cin + 0] = 1
    W[1, tap * cin + 1] = 1
    W = W.to(torch.bfloat16)
    out.zero_()
    lz.gemm(R * hw, cout, 9 * cin, srcs=[src], out_hw=(h, w), b=DRef(W), d=DRef(out))
    torch.cuda.synchronize()
    got = out[:, 0].float() + 64 * out[:, 1].float()
    bad = []
    for p in range(R * hw):
        img, lp = divmod(p, hw)
        oy, ox = divmod(lp, w)
        y, xx = oy + tap // 3 - 1, ox + tap % 3 - 1
        exp = -1 if not (0 <= y < h and 0 <= xx < w) else img * hw + y * w + xx
        g = int(got[p].item()) if exp >= 0 or got[p].item() != 0 else -1
        if g != exp:
            bad.append((p, exp, g))
    print("tap", tap, "bad", len(bad), bad[:6])

# random data, all taps, against torch conv2d (fp32 on the same bf16 values)
g = torch.Generator(device="cuda").manual_seed(0)
for (R, h, w, cin, cout) in [(2, 16, 16, 64, 128), (2, 16, 16, 128, 256), (4, 8, 8, 64, 128), (1, 64, 64, 64, 128)]:
    hw = h * w
    x = torch.randn((R * hw, cin), device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn((cout, 9 * cin), device="cuda", generator=g) / math.sqrt(9 * cin)).to(torch.bfloat16)
    bias = torch.randn(cout, device="cuda", generator=g)
    out = torch.zeros((R * hw, cout), device="cuda", dtype=torch.bfloat16)
    src = L.Src(DRef(x).ref(), NULL, None, h, w, cin, 0)
    lz.gemm(R * hw, cout, 9 * cin, srcs=[src], out_hw=(h, w), b=DRef(W), d=DRef(out), bias=bias)
    torch.cuda.synchronize()
    xi = x.float().reshape(R, h, w, cin).permute(0, 3, 1, 2)
    Wk = W.float().reshape(cout, 3, 3, cin).permute(0, 3, 1, 2)
    ref = torch.nn.functional.conv2d(xi, Wk, bias, padding=1).permute(0, 2, 3, 1).reshape(R * hw, cout)
    err = (out.float() - ref).abs()
    rows_bad = (err.max(dim=1).values > 0.05).nonzero().flatten()
    print((R, h, w, cin, cout), "maxerr", err.max().item(), "bad rows", rows_bad.numel(), rows_bad[:10].tolist())
