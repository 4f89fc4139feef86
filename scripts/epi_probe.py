"""Launch-trace phases of isolated per-op GEMMs (graph of repeated launches)."""
import math, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2305_17423_b200 import _lib as L
from paper_2305_17423_b200.engine import DRef, Launcher
lz = Launcher("bf16")
import pynvml as N
N.nvmlInit()
_h = N.nvmlDeviceGetHandleByIndex(0)
def warm(ms=300):
    x = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    import time
    t0 = time.time()
    while time.time() - t0 < ms / 1e3:
        x = x @ x.T * 0.001
    torch.cuda.synchronize()
    return N.nvmlDeviceGetClockInfo(_h, N.NVML_CLOCK_SM)
lz.static_meta = True
g = torch.Generator(device="cuda").manual_seed(0)
for m, n, k, splits in [(400, 320, 320, 1), (400, 320, 320, 0), (256, 1280, 1280, 1), (256, 1280, 1280, 0),
                        (400, 320, 2880, 0), (400, 320, 2880, 1), (128, 128, 320, 1)]:
    A = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn((n, k), device="cuda", generator=g) / math.sqrt(k)).to(torch.bfloat16)
    D = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    run = lambda: lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D), splits=splits)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr, stream=s):
            for _ in range(10):
                run()
    torch.cuda.synchronize()
    gr.replay(); torch.cuda.synchronize()
    buf = torch.zeros(16 + 16 * 4096, dtype=torch.int64, device="cuda")
    clk = warm()
    L.lib().fis_trace_launches(buf.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); gr.replay(); e1.record()
    torch.cuda.synchronize()
    L.lib().fis_trace_launches(None)
    tr = buf[16:16 + 160].view(10, 16).cpu().numpy()
    print(f"m={m} n={n} k={k} splits={splits}: {e0.elapsed_time(e1)*100:.2f} us/launch, kind {tr[0,15]}, sm clock {clk} MHz")
    for i in (4, 5):
        r = tr[i]
        print("   " + " ".join(f"{(r[p]-r[0])/1e3:6.2f}" for p in range(12)))
