"""One VM program with a single 256x1280x11520 GEMM (TMA A/B), run a few times (for ncu)."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_17423_b200.engine import DRef, Launcher, VmProgram  # noqa: E402
lz = Launcher("bf16")
g = torch.Generator(device="cuda").manual_seed(0)
m, n, k = 256, 1280, 11520
A = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
B = (torch.randn((n, k), device="cuda", generator=g) / math.sqrt(k)).to(torch.bfloat16)
D = torch.zeros((m, n), device="cuda", dtype=torch.bfloat16)
lz.capture = []
lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D), b_static=True)
calls, lz.capture = lz.capture, None
vm = VmProgram(lz, calls)
for _ in range(3):
    vm.run()
torch.cuda.synchronize()
print("ok")
