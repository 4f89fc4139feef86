"""Per-phase timestamps of one tcgen05 GEMM CTA (fis_trace) + graph-replayed kernel time for
representative sparse-step shapes (graph replay removes host launch overhead)."""
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
names = {0: "entry", 1: "tmem+sync", 2: "pdl_wait", 3: "stage0 issued", 4: "mma:full0", 5: "mma:lastfull",
         10: "epi:params", 6: "epi:done", 8: "epi:end", 9: "sync", 7: "dealloc"}
shapes = [(400, 77, 320, 80), (400, 320, 2880, 320), (256, 1280, 11520, 1280), (100, 640, 5760, 640),
          (400, 960, 320, 960), (1024, 1280, 320, 1280)]
for m, n, k, ldd in shapes:
    A = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn((n, k), device="cuda", generator=g) / math.sqrt(k)).to(torch.bfloat16)
    D = torch.empty((m, ldd), device="cuda", dtype=torch.bfloat16)
    run = lambda: lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D, ld=ldd))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr, stream=s):
            for _ in range(20):
                run()
    torch.cuda.synchronize()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    lib.fis_trace(1)
    run()
    torch.cuda.synchronize()
    lib.fis_trace(0)
    buf = (C.c_ulonglong * 16)()
    lib.fis_trace_read(buf)
    t0 = buf[0]
    ph = ", ".join(f"{nm} +{(buf[i]-t0)/1e3:.2f}" for i, nm in names.items() if buf[i] >= t0)
    print(f"m={m} n={n} k={k}: graph {us:.1f} us/launch ({2*m*n*k/us/1e6:.0f} TFLOP/s, "
          f"B {n*k*2/us/1e3:.0f} GB/s) | {ph}", flush=True)

# per-CTA timelines of a split-K (cluster) launch
print("--- per-CTA (z, y, x): entry / mma-done / cluster-sync / exit, us from first entry")
for m, n, k in [(400, 320, 2880), (100, 640, 5760)]:
    A = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn((n, k), device="cuda", generator=g) / math.sqrt(k)).to(torch.bfloat16)
    D = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D))
    torch.cuda.synchronize()
    big = (C.c_ulonglong * 2048)()
    lib.fis_trace_read_ctas(big)  # clear snapshot
    lib.fis_trace(1)
    lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D))
    torch.cuda.synchronize()
    lib.fis_trace(0)
    lib.fis_trace_read_ctas(big)
    rows = [(i, big[4 * i:4 * i + 4]) for i in range(512) if big[4 * i] > 0]
    t0 = min(r[1][0] for r in rows)
    print(f"m={m} n={n} k={k}: {len(rows)} CTAs")
    for i, r in rows[:48]:
        print(f"  cta {i:3d}: " + " ".join(f"{(x - t0)/1e3:6.2f}" if x >= t0 else "   -  " for x in r))
