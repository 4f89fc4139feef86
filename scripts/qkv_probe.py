import math, os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2305_17423_b200.engine import DRef, Launcher
lz = Launcher("bf16")
g = torch.Generator(device="cuda").manual_seed(0)
m, k, c = 34480, 320, 320
A = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
B = (torch.randn((3 * c, k), device="cuda", generator=g) / 18).to(torch.bfloat16)
qk = torch.empty((m, 2 * c), device="cuda", dtype=torch.bfloat16)
vt = torch.zeros((c, m + 16), device="cuda", dtype=torch.bfloat16)
v = torch.empty((m, c), device="cuda", dtype=torch.bfloat16)
full = torch.empty((m, 3 * c), device="cuda", dtype=torch.bfloat16)
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
print("qkv split V^T  %.1f us" % t(lambda: lz.gemm(m, 3 * c, k, a=DRef(A), b=DRef(B), d=DRef(qk), n_split=2 * c, d2=DRef(vt, ld=m + 16), d2_trans=True)))
print("qkv split V    %.1f us" % t(lambda: lz.gemm(m, 3 * c, k, a=DRef(A), b=DRef(B), d=DRef(qk), n_split=2 * c, d2=DRef(v))))
print("qkv one output %.1f us" % t(lambda: lz.gemm(m, 3 * c, k, a=DRef(A), b=DRef(B), d=DRef(full))))
