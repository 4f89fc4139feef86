"""Launch representative gather-GEMM shapes of the C2 sparse step (for ncu / timing)."""
import math
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_17423_b200 import _lib as L
from paper_2305_17423_b200.engine import DRef, Launcher

lz = Launcher("bf16")
impl = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = torch.Generator(device="cuda").manual_seed(0)
shapes = [(400, 320, 2880, 8), (400, 77, 320, 1), (256, 1280, 11520, 7), (100, 640, 5760, 14)]
for m, n, k, s in shapes:
    A = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn((n, k), device="cuda", generator=g) / math.sqrt(k)).to(torch.bfloat16)
    D = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    lz.gemm_impl = impl
    for _ in range(2):
        lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D), splits=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D), splits=s)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(f"m={m} n={n} k={k} splits={s} impl={impl}: {us:.1f} us  {2*m*n*k/us/1e6:.1f} TFLOP/s  "
          f"weights {n*k*2/us/1e3:.0f} GB/s", flush=True)
