"""Per-phase timestamps of one tcgen05 GEMM CTA (fis_trace) for representative sparse-step shapes."""
import ctypes as C
import math
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_17423_b200 import _lib as L
from paper_2305_17423_b200.engine import DRef, Launcher

lib = L.lib()
lz = Launcher("bf16")
g = torch.Generator(device="cuda").manual_seed(0)
names = ["entry", "tmem+sync", "pdl_wait", "stage0 issued", "mma: full[0]", "mma: last full", "epi: done", "exit"]
for m, n, k, s in [(400, 77, 320, 1), (400, 320, 2880, 0), (256, 1280, 11520, 0), (100, 640, 5760, 0)]:
    A = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn((n, k), device="cuda", generator=g) / math.sqrt(k)).to(torch.bfloat16)
    D = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D), splits=s or None)
    torch.cuda.synchronize()
    lib.fis_trace(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D), splits=s or None)
    e1.record()
    torch.cuda.synchronize()
    lib.fis_trace(0)
    buf = (C.c_ulonglong * 16)()
    lib.fis_trace_read(buf)
    t0 = buf[0]
    print(f"m={m} n={n} k={k}: event {e0.elapsed_time(e1)*1e3:.1f} us; " +
          ", ".join(f"{nm} +{(buf[i]-t0)/1e3:.2f}" for i, nm in enumerate(names) if buf[i] >= t0), flush=True)
