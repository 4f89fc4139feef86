"""Time fis_attn on the stacked (R = 64) step's shapes in isolation, per kernel launch (CUPTI).

usage: python scripts/attn_micro.py [cross|self|all] [levels, e.g. 02]   (env FIS_ATTN_* toggles apply)
Prints per-shape: launches, per-launch median us, total us, and the HBM floor (q + res + out bytes).
"""
import math
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_17423_b200 import _lib as L  # noqa: E402
from paper_2305_17423_b200.engine import NULL, DRef  # noqa: E402

R = 64


def lens_l0():
    # 5 / 10 / 25 % squares of a 64x64 latent, dilated: ~205 / 410 / 1024 active rows
    return [(205, 410, 1024)[i % 3] for i in range(R)]


def shape(kind, level):
    if level == 0:
        d, q = 320, lens_l0()
    elif level == 1:
        d, q = 640, [max(16, n // 4 + 40) for n in lens_l0()]
    elif level == 2:
        d, q = 1280, [256] * R
    else:
        d, q = 1280, [64] * R
    return d, q


def run(kind, level, reps=20):
    d, qlens = shape(kind, level)
    bf = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(level)
    starts = [0]
    for n in qlens:
        starts.append(starts[-1] + (n + 15) // 16 * 16)
    m = starts[-1]
    Q = torch.randn((m, d), device="cuda", generator=g).to(bf)
    res = torch.randn((m, d), device="cuda", generator=g).to(bf)
    out = torch.zeros((m, d), device="cuda", dtype=bf)
    if kind == "self":
        K = torch.randn((m, d), device="cuda", generator=g).to(bf)
        kseg = [(starts[i], starts[i] + qlens[i]) for i in range(R)]
    else:
        K = torch.randn((80 * R, d), device="cuda", generator=g).to(bf)
        kseg = [(80 * i, 80 * i + 77) for i in range(R)]
    nk = K.shape[0]
    ldv = (nk + 15) // 16 * 16
    Vt = torch.randn((d, ldv), device="cuda", generator=g).to(bf)
    qseg = [(starts[i], starts[i] + qlens[i]) for i in range(R)]
    qs = torch.tensor([v for p in qseg for v in p], dtype=torch.int32, device="cuda")
    ks = torch.tensor([v for p in kseg for v in p], dtype=torch.int32, device="cuda")
    a = L.AttnArgs(m, nk, d, d, DRef(Q).ref(), DRef(K).ref(), DRef(Vt, ld=ldv).ref(), 1.0 / math.sqrt(d),
                   DRef(res).ref(), NULL, DRef(out).ref(), None)
    maxk = max(k1 - k0 for k0, k1 in kseg)
    a.nseg, a.max_seg_q, a.q_seg, a.k_seg = R, max(qlens), L.ptr(qs), L.ptr(ks)
    nb = int(L.lib().fis_attn_ws_bytes(m, maxk, d))
    ws = torch.zeros(nb, device="cuda", dtype=torch.uint8)
    a.max_seg_k, a.ws, a.ws_bytes = maxk, L.ptr(ws), nb
    flush = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
    for _ in range(3):
        L.call("fis_attn", a)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            flush.zero_()
            L.call("fis_attn", a)
        torch.cuda.synchronize()
    ks_ = [e for e in prof.events() if e.device_type.name == "CUDA" and "attn" in e.name]
    nl = len(ks_) // reps
    per = [statistics.median(ks_[i * nl + j].device_time for i in range(reps)) for j in range(nl)]
    if os.environ.get("TRACE"):  # FIS_LIB=libfisedit_trace.so: CTA 0's phase stamps of one launch
        buf = torch.zeros(16 + 16 * 4096, dtype=torch.int64, device="cuda")
        L.lib().fis_trace_launches(buf.data_ptr())
        flush.zero_()
        L.call("fis_attn", a)
        torch.cuda.synchronize()
        L.lib().fis_trace_launches(None)
        n = int(buf[0].item())
        for i in range(n):
            row = buf[16 + 16 * i:32 + 16 * i].tolist()
            t0 = row[0]
            print(f"  trace kind {row[15]}: " + " ".join(f"{p}:{(row[p] - t0) / 1e3:.2f}" for p in range(1, 15)
                                                        if row[p] > 0), flush=True)
    rows = sum(qlens)
    floor_b = rows * d * 2 * 3 + nk * d * 2 * 2
    print(f"{kind} L{level}: m={m} rows={rows} d={d} keys/seg={maxk} launches={nl} per-launch us="
          f"{[round(p, 1) for p in per]} total={sum(per):.1f} us  hbm floor {floor_b / 7.4e6:.1f} us "
          f"({floor_b / 1e6:.1f} MB)", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    for kind in ("cross", "self"):
        if which not in ("all", kind):
            continue
        for lv in (0, 1, 2, 3):
            if len(sys.argv) > 2 and str(lv) not in sys.argv[2]:
                continue
            run(kind, lv, reps=int(os.environ.get("REPS", "20")))
