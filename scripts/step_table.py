"""Per-op CUPTI table (graph replay, critical-path us) of the C2 batch-1 sparse step, the dense
step and (optional) the R-request stacked step.

    python scripts/step_table.py [--R 64] [--out profiles/r02/step_table.txt]
"""
import argparse
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import bench as B
import paper_2305_17423_b200 as P
from paper_2305_17423_b200 import unet as U


def show(title, table, f):
    tot = sum(us for _, us, _ in table)
    print(f"== {title}: {len(table)} ops, {tot:.1f} us", file=f)
    for i, (o, us, name) in enumerate(table):
        d = {k: v for k, v in o.items() if k not in ("op", "kernels")}
        print(f"{i:3d} {us:8.2f} us  {o['op']:<14s} x{o['kernels']} {d}", file=f)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--R", type=int, default=0)
    ap.add_argument("--out", default="gpurun_out/step_table.txt")
    ap.add_argument("--only-R", action="store_true", help="skip the batch-1 / dense tables")
    ap.add_argument("--trace-kind", type=int, default=0,
                    help="with FIS_LIB=libfisedit_trace.so: CTA 0 phase stamps of this kernel kind in one "
                         "stacked-step replay (e.g. 13 = short-run attention)")
    args = ap.parse_args()
    P.set_precision("bf16")
    cfg = P.UNetConfig(**B.C2)
    eng = U.get_engine(cfg)
    f = open(args.out, "w")
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens(B.OLD_IDS), cfg, store, record="engine")
    kv = eng.text_kv(P.embed_tokens(P.PromptTokens(B.NEW_IDS), cfg))
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    for frac in (() if args.only_R else (0.10,)):
        mask = P.centered_square_mask(64, 64, frac)
        ep = U.EditPlan(eng, store.arena, mask, kv, lat0)
        ops = B._op_log(eng, ep.plan)
        run = U._Runner(eng, ep.plan, True)
        ms = B._time_runner(run, cfg.steps, 20, 3)
        t = B.replay_kernels(run, ops, cfg.steps)
        show(f"sparse {frac:.0%} step ({ms * 1e3:.1f} us events)", t, f)
    if not args.only_R:
        lat = torch.empty((cfg.steps + 1, eng.hw(0), 4), dtype=torch.float32, device=eng.dev)
        lat[0].copy_(lat0)
        plan = U.StepPlan(eng, kv, lat, None)
        ops = B._op_log(eng, plan)
        run = U._Runner(eng, plan, True)
        ms = B._time_runner(run, cfg.steps, 10, 3)
        t = B.replay_kernels(run, ops, cfg.steps)
        if t is None:
            print("dense: kernel count mismatch", sum(o["kernels"] for o in ops), file=f)
        else:
            show(f"dense step ({ms * 1e3:.1f} us events)", t, f)
    if args.R:
        store.close()
        reqs = [B._request(r, cfg) for r in range(args.R)]
        stores = [P.CacheStore() for _ in reqs]
        U.generate_dense_batch([P.PromptTokens(o) for o, _, _ in reqs], cfg, stores)
        kvs = [eng.text_kv(P.embed_tokens(P.PromptTokens(n), cfg)) for _, n, _ in reqs]
        bp = U.BatchedEditPlan(eng, stores[0].arena.stacked, [P.BinaryMask(b) for _, _, b in reqs], kvs,
                               [lat0] * args.R)
        ops = B._op_log(eng, bp.plan)
        run = U._Runner(eng, bp.plan, True)
        ms = B._time_runner(run, cfg.steps, 5, 3)
        t = B.replay_kernels(run, ops, cfg.steps)
        show(f"stacked R={args.R} step ({ms * 1e3:.1f} us events)", t, f)
        if args.trace_kind:
            from paper_2305_17423_b200 import _lib as L
            buf = torch.zeros(16 + 16 * 4096, dtype=torch.int64, device=eng.dev)
            L.lib().fis_trace_launches(buf.data_ptr())
            run.step(4)
            torch.cuda.synchronize()
            L.lib().fis_trace_launches(None)
            n = int(buf[0].item())
            tr = buf[16:16 + 16 * n].view(n, 16).cpu().tolist()
            for i, row in enumerate(tr):
                if row[15] % 16 != args.trace_kind % 16 or row[15] != args.trace_kind:
                    continue
                print(f"trace {i:3d} kind {row[15]}: " + " ".join(
                    f"{p}:{(row[p] - row[0]) / 1e3:.2f}" for p in range(1, 15) if row[p] > 0), file=f)
    f.close()
    print(open(args.out).read())


if __name__ == "__main__":
    main()
