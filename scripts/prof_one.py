"""Launch one GEMM shape a few times (for ncu --set full source-level capture)."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_17423_b200.engine import DRef, Launcher
lz = Launcher("bf16")
m, n, k = (int(v) for v in sys.argv[1:4])
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
B = (torch.randn((n, k), device="cuda", generator=g) / math.sqrt(k)).to(torch.bfloat16)
D = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
for _ in range(4):
    lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D))
torch.cuda.synchronize()
