"""Probe the step VM on a B200: per-GEMM equivalence vs the per-op kernel, and a per-op
timeline of the C2 sparse step (globaltimer stamps recorded by the VM).

    python scripts/vm_probe.py [gemm] [trace] [dense]
"""
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_17423_b200 import _lib as L  # noqa: E402
from paper_2305_17423_b200.engine import DRef, Launcher, VmProgram  # noqa: E402

KIND = {1: "gemm", 2: "softmax", 3: "gn_stats", 4: "gn_apply", 5: "pool", 6: "materialize", 7: "attn", 8: "gn"}


def gemm_equivalence():
    lz = Launcher("bf16")
    g = torch.Generator(device="cuda").manual_seed(0)
    for (m, n, k) in [(400, 320, 2880), (100, 640, 5760), (256, 1280, 11520), (400, 960, 320), (64, 1280, 1280),
                      (400, 400, 320), (400, 77, 320), (100, 4, 2880)]:
        A = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
        B = (torch.randn((n, k), device="cuda", generator=g) / math.sqrt(k)).to(torch.bfloat16)
        bias = torch.randn((n,), device="cuda", generator=g)
        D0 = torch.zeros((m, n), device="cuda", dtype=torch.bfloat16)
        D1 = torch.zeros((m, n), device="cuda", dtype=torch.bfloat16)
        lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D0), bias=bias)
        lz.capture = []
        lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D1), bias=bias)
        calls, lz.capture = lz.capture, None
        vm = VmProgram(lz, calls)
        vm.run()
        torch.cuda.synchronize()
        ref = (A.float() @ B.float().T + bias)
        e0 = (D0.float() - ref).abs().max().item()
        e1 = (D1.float() - ref).abs().max().item()
        it = vm.items()[0]
        print(f"gemm {m}x{n}x{k}: per-op err {e0:.3e}  vm err {e1:.3e}  vm items {it[1]} splits {it[2]}", flush=True)


def step_trace(dense=False):
    import paper_2305_17423_b200 as P
    from paper_2305_17423_b200 import unet as U
    P.set_precision("bf16")
    C2 = dict(latent_h=64, latent_w=64, latent_channels=4, channels=(320, 640, 1280, 1280), blocks_per_level=2,
              groups=32, steps=50, t1=5, t2=10, gate_fraction=0.25, dilation_radius=1, text_dim=768,
              vocab_size=49408, seed=0)
    cfg = P.UNetConfig(**C2)
    eng = U.get_engine(cfg)
    old = tuple(range(1, 78))
    new = tuple(99 if i == 3 else v for i, v in enumerate(old))
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens(old), cfg, store, record="engine")
    kv = eng.text_kv(P.embed_tokens(P.PromptTokens(new), cfg))
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    if dense:
        lat = torch.empty((cfg.steps + 1, eng.hw(0), 4), dtype=torch.float32, device=eng.dev)
        lat[0].copy_(lat0)
        plan = U.StepPlan(eng, kv, lat, None)
    else:
        mask = P.centered_square_mask(64, 64, 0.1)
        ep = U.EditPlan(eng, store.arena, mask, kv, lat0)
        plan = ep.plan
    vm = eng.record_step(plan)
    vm.enable_trace()
    for it in range(6):
        eng.step_dev.fill_(1 + it)
        vm.reset_trace()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        vm.run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    rows = vm.read_trace()
    print(f"{'dense' if dense else 'sparse'} step: {ms * 1e3:.1f} us (events), {len(rows)} ops, span "
          f"{max(r[4] for r in rows) / 1e3:.1f} us", flush=True)
    prev_end = 0.0
    tot = {}
    for i, (k, n, s, st, en) in enumerate(rows):
        c = vm.calls[i][1]
        desc = ""
        if k == 1:
            desc = f"m={c.m} n={c.n} k={c.k} mode={c.a_mode}"
        elif k == 7:
            desc = f"m={c.m} keys={c.n_keys} d={c.d}"
        print(f"{i:3d} {KIND[k]:9s} items={n:4d} S={s:2d} wait={(st - prev_end) / 1e3:6.2f} dur={(en - st) / 1e3:6.2f} "
              f"end={en / 1e3:7.1f}  {desc}")
        tot[KIND[k]] = tot.get(KIND[k], 0.0) + (en - prev_end) / 1e3
        prev_end = en
    print("time by kind (incl. wait):", {k: round(v, 1) for k, v in tot.items()})
    for j in [int(x) for x in os.environ.get("TRACE_OPS", "0,1,4,9").split(",")]:
        vm.trace_op(j)
        eng.step_dev.fill_(3)
        vm.reset_trace()
        vm.run()
        torch.cuda.synchronize()
        st = vm.items_trace.cpu().numpy().astype(np.float64)
        prev_end = rows[j - 1][4] if j > 0 else 0.0
        tr = vm.trace.cpu().numpy().view(np.uint64).astype(np.float64)
        t_dep = tr[j - 1, 1] if j > 0 else tr[:, 0].min()
        print(f"op {j} ({KIND[rows[j][0]]}, {rows[j][1]} items) phase stamps (us after dep op end; "
              "0 start,1 B issued,2 dep ok,3 A issued,4 tables,5 mma done,6 epi done,7 signaled,8 A0 issued,"
              "9 tmem staged,10 staged+bar,11 split met):")
        for i in range(min(st.shape[0], 4)):
            vals = ["   -  " if v == 0 else f"{(v - t_dep) / 1e3:6.2f}" for v in st[i][:14]]
            if st[i][15] and st[i][14] and st[i][7] and st[i][2]:
                vals.append(f"clk {(st[i][15] - st[i][14]) / (st[i][7] - st[i][2]) * 1e3:5.0f} MHz")
            print(f"   item {i:3d}: " + " ".join(vals))
        vm.args.trace_op, vm.args.trace_items = -1, None


if __name__ == "__main__":
    what = sys.argv[1:] or ["gemm", "trace"]
    if "gemm" in what:
        gemm_equivalence()
    if "trace" in what:
        step_trace(False)
    if "dense" in what:
        step_trace(True)


def single_op():
    """One GEMM (400x320x80 + residual, the cross-attention P.V shape) as a one-op VM program."""
    lz = Launcher("bf16")
    g = torch.Generator(device="cuda").manual_seed(0)
    for (m, n, k, res) in [(400, 320, 80, True), (256, 1280, 11520, False), (256, 1280, 1280, False)]:
        A = torch.randn((m, k), device="cuda", generator=g).to(torch.bfloat16)
        B = (torch.randn((n, k), device="cuda", generator=g) / math.sqrt(k)).to(torch.bfloat16)
        R = torch.randn((m, n), device="cuda", generator=g).to(torch.bfloat16)
        D = torch.zeros((m, n), device="cuda", dtype=torch.bfloat16)
        lz.capture = []
        lz.gemm(m, n, k, a=DRef(A), b=DRef(B), d=DRef(D), res=DRef(R) if res else None, b_static=True)
        calls, lz.capture = lz.capture, None
        vm = VmProgram(lz, calls)
        vm.enable_trace()
        vm.trace_op(0)
        for _ in range(3):
            vm.reset_trace()
            vm.items_trace.zero_()
            vm.run()
        torch.cuda.synchronize()
        st = vm.items_trace.cpu().numpy().astype(np.float64)
        t0 = st[:, 2].min()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            vm.run()
        e1.record()
        torch.cuda.synchronize()
        print(f"single op {m}x{n}x{k} res={res}: items {vm.items()[0][1]} splits {vm.items()[0][2]} "
              f"tma a/b {vm.ops_host[0].tmap_a}/{vm.ops_host[0].tmap_b}: {e0.elapsed_time(e1) * 100:.1f} us/launch")
        for i in range(min(st.shape[0], 6)):
            print("   " + " ".join("   -  " if v == 0 else f"{(v - t0) / 1e3:6.2f}" for v in st[i][:15]))


if __name__ == "__main__" and "single" in sys.argv:
    single_op()


def checks():
    """VM (TMA paths) vs per-op kernels / torch on single ops at SD shapes."""
    from paper_2305_17423_b200.engine import NULL
    lz = Launcher("bf16")
    g = torch.Generator(device="cuda").manual_seed(0)
    # dense 3x3 conv on a 16x16x1280 map (TMA per-tap boxes) and with a 2-segment concat
    for (h, w, c0, c1, n) in [(16, 16, 1280, 0, 1280), (8, 8, 1280, 0, 1280), (16, 16, 1280, 1280, 1280)]:
        x0 = torch.randn((h * w, c0), device="cuda", generator=g).to(torch.bfloat16)
        x1 = torch.randn((h * w, max(c1, 8)), device="cuda", generator=g).to(torch.bfloat16)
        k = 9 * (c0 + c1)
        B = (torch.randn((n, k), device="cuda", generator=g) / math.sqrt(k)).to(torch.bfloat16)
        srcs = [L.Src(DRef(x0).ref(), NULL, None, h, w, c0, 0)]
        if c1:
            srcs.append(L.Src(DRef(x1).ref(), NULL, None, h, w, c1, 0))
        outs = []
        for vm in (False, True):
            D = torch.zeros((h * w, n), device="cuda", dtype=torch.bfloat16)
            if vm:
                lz.capture = []
            lz.gemm(h * w, n, k, srcs=srcs, out_hw=(h, w), b=DRef(B), d=DRef(D), b_static=True)
            if vm:
                calls, lz.capture = lz.capture, None
                prog = VmProgram(lz, calls)
                prog.run()
                print(f"  conv tmaps a/a2/b = {prog.ops_host[0].tmap_a}/{prog.ops_host[0].tmap_a2}/{prog.ops_host[0].tmap_b}")
            torch.cuda.synchronize()
            outs.append(D.float())
        print(f"conv {h}x{w} cin {c0}+{c1} -> {n}: vm vs per-op max diff {(outs[0] - outs[1]).abs().max().item():.3e} "
              f"(|ref| max {outs[0].abs().max().item():.2f})", flush=True)
    # attention: out = res + softmax(q k^T s) v
    for (m, nk, d) in [(400, 400, 320), (256, 256, 1280), (100, 100, 640), (400, 77, 320)]:
        q = torch.randn((m, d), device="cuda", generator=g).to(torch.bfloat16)
        kk = torch.randn((nk, d), device="cuda", generator=g).to(torch.bfloat16)
        v = torch.randn((nk, d), device="cuda", generator=g).to(torch.bfloat16)
        mp = (nk + 15) // 16 * 16
        vt = torch.zeros((d, mp), device="cuda", dtype=torch.bfloat16)
        vt[:, :nk] = v.T
        res = torch.randn((m, d), device="cuda", generator=g).to(torch.bfloat16)
        out = torch.zeros((m, d), device="cuda", dtype=torch.bfloat16)
        sc = 1.0 / math.sqrt(d)
        lz.capture = []
        a = L.AttnArgs(m, nk, d, d, DRef(q).ref(), DRef(kk).ref(), DRef(vt).ref(), sc, DRef(res).ref(), NULL,
                       DRef(out).ref(), L.ptr(lz.step_dev))
        lz._call("fis_attn", a)
        calls, lz.capture = lz.capture, None
        prog = VmProgram(lz, calls)
        prog.run()
        torch.cuda.synchronize()
        ref = res.float() + torch.softmax(q.float() @ kk.float().T * sc, -1) @ v.float()
        print(f"attn m={m} keys={nk} d={d}: vm vs torch max diff {(out.float() - ref).abs().max().item():.3e} "
              f"tmaps {prog.ops_host[0].tmap_a}/{prog.ops_host[0].tmap_b}/{prog.ops_host[0].tmap_a2}", flush=True)


if __name__ == "__main__" and "checks" in sys.argv:
    checks()


def chain_check(c=1280, fuse=False, swap=False, splits=None):
    """Conv whose input is produced by the previous op of the same VM program (TMA after the dep)."""
    from paper_2305_17423_b200.engine import NULL
    lz = Launcher("bf16")
    g = torch.Generator(device="cuda").manual_seed(1)
    h = w = 16
    X = torch.randn((h * w, c), device="cuda", generator=g).to(torch.bfloat16)
    W0 = (torch.randn((c, c), device="cuda", generator=g) / math.sqrt(c)).to(torch.bfloat16)
    cu = 1280 if fuse else 0
    U = torch.randn((64, max(cu, 8)), device="cuda", generator=g).to(torch.bfloat16)  # 8x8 coarse map
    B = (torch.randn((c, 9 * (c + cu)), device="cuda", generator=g) / math.sqrt(9 * c)).to(torch.bfloat16)
    outs = []
    for vm in (False, True):
        Y = torch.zeros((h * w, c), device="cuda", dtype=torch.bfloat16)
        D = torch.zeros((h * w, c), device="cuda", dtype=torch.bfloat16)
        if vm:
            lz.capture = []
        lz.gemm(h * w, c, c, a=DRef(X), b=DRef(W0), d=DRef(Y), b_static=True)
        srcs = [L.Src(DRef(Y).ref(), NULL, None, h, w, c, 0)]
        if fuse:
            up = L.Src(DRef(U).ref(), NULL, None, 8, 8, cu, 1)
            srcs = srcs + [up] if swap else [up] + srcs
        lz.gemm(h * w, c, 9 * (c + cu), srcs=srcs, out_hw=(h, w), b=DRef(B), d=DRef(D), b_static=True, splits=splits)
        if vm:
            calls, lz.capture = lz.capture, None
            prog = VmProgram(lz, calls)
            for _ in range(3):
                Y.zero_(); D.zero_()
                prog.run()
        torch.cuda.synchronize()
        outs.append((Y.float(), D.float()))
    print(f"chain c={c} fuse={fuse} swap={swap} splits={splits}: Y diff {(outs[0][0] - outs[1][0]).abs().max().item():.3e}, conv diff "
          f"{(outs[0][1] - outs[1][1]).abs().max().item():.3e}", flush=True)


if __name__ == "__main__" and "chain" in sys.argv:
    chain_check(1280, True)
    chain_check(1280, True, swap=True)
    chain_check(1280, True, splits=1)
    chain_check(1280, True, splits=2)
