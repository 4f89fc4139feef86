"""Per-kernel phase timeline of one graph-replayed C2 sparse step (batch 1): CTA (0,0,0)'s
globaltimer stamps (fis_trace_launches) joined with CUPTI kernel start/end.

    python scripts/launch_trace.py [--mask 0.1] [--dense] [--out gpurun_out/launch_trace.txt]
Columns (us, relative to the previous kernel's CUPTI end): start, pre-wait, post-wait, first MMA
stage / first S, last stage / o_done, epilogue, exit(CTA0), end(CUPTI)."""
import argparse
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import bench as B
import paper_2305_17423_b200 as P
from paper_2305_17423_b200 import _lib as L
from paper_2305_17423_b200 import unet as U

KIND = {1: "tc", 2: "attn", 3: "simt", 4: "big", 5: "gn", 6: "pool", 7: "gn_apply", 8: "softmax", 9: "mat",
        10: "up2", 11: "gn_stats", 12: "xattn"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mask", type=float, default=0.10)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--out", default="gpurun_out/launch_trace.txt")
    args = ap.parse_args()
    P.set_precision("bf16")
    cfg = P.UNetConfig(**B.C2)
    eng = U.get_engine(cfg)
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens(B.OLD_IDS), cfg, store, record="engine")
    kv = eng.text_kv(P.embed_tokens(P.PromptTokens(B.NEW_IDS), cfg))
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    if args.dense:
        lat = torch.empty((cfg.steps + 1, eng.hw(0), 4), dtype=torch.float32, device=eng.dev)
        lat[0].copy_(lat0)
        plan = U.StepPlan(eng, kv, lat, None)
    else:
        plan = U.EditPlan(eng, store.arena, P.centered_square_mask(64, 64, args.mask), kv, lat0).plan
    ops = B._op_log(eng, plan)
    run = U._Runner(eng, plan, True)
    ms = B._time_runner(run, cfg.steps, 20, 3)
    table = B.replay_kernels(run, ops, cfg.steps)
    # CUPTI raw start/end of the last replay
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run.step(3)
        torch.cuda.synchronize()
    ks = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                if e.device_type == torch.autograd.DeviceType.CUDA and "fis::" in e.name)
    buf = torch.zeros(16 + 16 * 4096, dtype=torch.int64, device=eng.dev)
    L.lib().fis_trace_launches(buf.data_ptr())
    run.step(4)
    torch.cuda.synchronize()
    L.lib().fis_trace_launches(None)
    n = int(buf[0].item())
    tr = buf[16:16 + 16 * n].view(n, 16).cpu().numpy()
    f = open(args.out, "w")
    print(f"step {ms * 1e3:.1f} us (events); {len(ks)} CUPTI kernels, {n} traced launches", file=f)
    t0 = tr[0, 0]
    # align the two clocks on the first kernel's start
    c0 = ks[0][0] if ks else 0.0
    prev_end = None
    for i in range(min(n, len(ks))):
        st, en, nm = ks[i]
        st, en = st - c0, en - c0
        row = tr[i]
        kind = KIND.get(int(row[15]) % 16, "?")
        ph = [(row[p] - t0) / 1e3 if row[p] > 0 else float("nan") for p in range(12)]
        ref = prev_end if prev_end is not None else 0.0
        o = ops[i] if i < len(ops) else {}
        desc = {k: v for k, v in o.items() if k not in ("kernels",)}
        cells = " ".join(f"{x - ref:7.2f}" for x in ph)
        print(f"{i:3d} {kind:5s} crit {en - ref:6.2f} | start {st - ref:7.2f} | phases {cells} | {desc}", file=f)
        prev_end = en if prev_end is None else max(prev_end, en)
    f.close()
    print(open(args.out).read())


if __name__ == "__main__":
    main()
