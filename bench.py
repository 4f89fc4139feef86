"""Benchmark of the sparse edit step (BASELINE.json metric: edit-steps/sec at SD-1.5 512^2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mask 0.10]

Workload (BASELINE configs[1]): SD-1.5-shape toy UNet (channels
320/640/1280/1280, 2 blocks/level, 32 groups, 64x64x4 latent, 77-token text of
width 768), 50-step schedule, one cached dense generation in HBM, user-mask
edit with centered_square_mask(64, 64, 0.10). A "step" is one sparse UNet
forward + step update (unet.py:874-883) replayed from one captured CUDA graph;
each rank edits its own request (weak scaling, no collective in the step).

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize, CUDA
events on the launching stream, max over ranks. Inputs larger than L2: each
step streams 444 MB (bf16) of weights plus that step's cache slab, so no L2
flush is needed. Clocks: NVML polled every ~1 ms on a thread during the timed
region.

Per-kernel numbers (roofline, kernel shares) come from CUPTI kernel records
(torch.profiler) of graph replays of the SAME captured step: each kernel's
critical-path time is end_i - end_{i-1} (kernels overlap their prologue with the
previous kernel through programmatic dependent launch), so the per-kernel times
of one replay sum to the step.

Sections of the JSON line beyond the base contract:
  roofline       gated-conv gather-GEMMs of the timed step (algorithmic FLOPs / CUPTI time)
  kernels        per-op-class share of the step (CUPTI, graph replay)
  sweep          C3: sparse step vs mask ratio 1..100% + random-dilated 10%, vs the dense step
  fp32_parity    the same step with fp32 operands on the tensor cores (3xTF32; *_simt: SIMT FFMA)
  c4             SD-2 shape (96x96, 1024-wide text): sparse step + multi-round edit() e2e
  batched        C5: 64 requests over the N GPUs, each GPU's share stepped as one stacked batch
  cpu_baseline   the reference package's own CPU path (baseline/_ref) on a bounded sample
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2 = dict(latent_h=64, latent_w=64, latent_channels=4, channels=(320, 640, 1280, 1280), blocks_per_level=2,
          groups=32, steps=50, t1=5, t2=10, gate_fraction=0.25, dilation_radius=1, text_dim=768,
          vocab_size=49408, seed=0)
C4 = dict(C2, latent_h=96, latent_w=96, text_dim=1024)
OLD_IDS = tuple(range(1, 78))
NEW_IDS = tuple(99 if i == 3 else v for i, v in enumerate(OLD_IDS))
METRIC = "edit-steps/sec at SD-1.5 512^2 vs mask ratio; sparse-conv % of TC peak"
WEIGHT_BYTES_BF16 = 2 * 221_700_000  # 221.7 M params of the SD-1.5-shape toy UNet
E2E_CALLS = 5


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["hbm_gbs"], d["bf16_tflops"], "measured (MEASURED_PEAKS.json, burst)"
    except Exception:
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """NVML sampler of SM clock and throttle reasons on a thread (~1 ms period) during the timed
    region (nvidia-smi's 100 ms minimum period cannot resolve a ~30 ms region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, idx):
        self.idx, self.samples, self.max_mhz, self.reasons = idx, [], None, set()
        self._stop = threading.Event()
        self._h = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self._N = N
            self._h = N.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._h = None
        return self

    def _sample(self):
        N = self._N
        self.samples.append(float(N.nvmlDeviceGetClockInfo(self._h, N.NVML_CLOCK_SM)))
        r = N.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        for name, bit in self.REASONS.items():
            if r & bit:
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.001)

    def __exit__(self, *a):
        if self._h is not None:
            self._stop.set()
            self._t.join()
            if not self.samples:
                try:
                    self._sample()
                except Exception:
                    pass

    def summary(self):
        s = self.samples
        return {"sm_mhz": float(np.median(s)) if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s), "source": "NVML, ~1 ms period"}


def dist_init():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def reduce_max(x):
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ----------------------------------------------------------------------------- CPU arms
def _ref_package():
    """The unmodified reference package installed in baseline/_ref (pip --target), or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "sparsedit")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import sparsedit
        return sparsedit
    except Exception:
        return None


def ref_sample(cfg_d, frac, steps, warmup):
    """The reference package's own CPU path (sparsedit 0.1.0 from baseline/_ref): UNet(config),
    one dense caching step t=1 recorded into its CacheStore (DenseMode recorder, unet.py:680-696),
    then `warmup + steps` sparse steps at t=1 through SparseMode over that cache with the 10%
    centered-square plan (unet.py:868-883). Returns (edit-steps/s, s/step, setup s)."""
    sd = _ref_package()
    from sparsedit import unet as RU
    t0 = time.perf_counter()
    cfg = RU.UNetConfig(**dict(cfg_d, channels=tuple(cfg_d["channels"])))
    net = RU.UNet(cfg)
    store = sd.CacheStore()
    text_old = RU.embed_tokens(RU.PromptTokens(OLD_IDS), cfg)
    text_new = RU.embed_tokens(RU.PromptTokens(NEW_IDS), cfg)
    lat = RU.initial_latent(cfg)
    rec = lambda lid, role, payload: store.put((1, lid, role), payload)
    net.forward(lat, 1, text_old, RU.DenseMode(cfg.groups, recorder=rec))
    mask = sd.centered_square_mask(cfg.latent_h, cfg.latent_w, frac)
    pyr = sd.build_pyramid(mask, cfg.levels)
    plans = {lv: sd.select_gather_plan(pyr.levels[lv], (3, 3)) for lv in RU._gated_levels(net)}
    setup = time.perf_counter() - t0
    times = []
    for i in range(warmup + steps):
        t1 = time.perf_counter()
        ctx = RU._sparse_contexts(net, store, 1)
        net.forward(lat, 1, text_new, RU.SparseMode(cfg, pyr, plans, ctx, pool=store.buffer_pool))
        times.append(time.perf_counter() - t1)
    per = float(np.mean(times[warmup:]))
    return 1.0 / per, per, setup


def port_sample(cfg_d, frac, steps, warmup):
    """Oracle port (numpy f64 restatement of the reference) on the same bounded sample."""
    from oracle import sparsedit_oracle as O
    cfg = O.cfg_of(dict(cfg_d))
    net = O.build_net(cfg)
    text_old, text_new = O.embed(OLD_IDS, cfg), O.embed(NEW_IDS, cfg)
    lat = O.init_latent(cfg)
    cache = {}
    rec = lambda lid, role, v: cache.__setitem__((1, lid, role), v)
    O.forward(net, lat, 1, text_old, O.DenseOps(net, rec))
    mask = O.centered_square(cfg["latent_h"], cfg["latent_w"], frac)
    pyr = O.pyramid(mask, len(cfg["channels"]))
    plans = {lv: O.gather_plan(pyr[lv]) for lv in range(len(cfg["channels"]))}
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        O.forward(net, lat, 1, text_new, O.SparseOps(net, pyr, plans, cache, 1))
        times.append(time.perf_counter() - t0)
    per = float(np.mean(times[warmup:]))
    return 1.0 / per, per


def cpu_baseline(frac, steps, warmup):
    threads = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    if _ref_package() is not None:
        v, per, setup = ref_sample(C2, frac, steps, warmup)
        return {"value": v, "unit": "edit-steps/s", "cores": threads, "kind": "reference",
                "ms_per_step": per * 1e3,
                "sample": f"reference package sparsedit 0.1.0 (baseline/_ref, unmodified): UNet + one dense caching "
                          f"step t=1 into its CacheStore ({setup:.1f} s setup, not timed), then {warmup}+{steps} "
                          f"SparseMode steps at t=1 (10% centered square), numpy/OpenBLAS on {threads} threads"}
    v, per = port_sample(C2, frac, steps, warmup)
    return {"value": v, "unit": "edit-steps/s", "cores": threads, "kind": "port", "ms_per_step": per * 1e3,
            "sample": f"oracle port (numpy f64 restatement), {warmup}+{steps} sparse steps at t=1 after one dense "
                      "caching step"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # bounded sample: the reference's sparse C2 step takes ~9 s on 8 cores, so at most 6 timed
    # steps after at most 1 warm-up (the line reports the counts actually timed)
    n_steps, n_warm = max(1, min(args.steps, 6)), min(args.warmup, 1)
    cb = cpu_baseline(args.mask, n_steps, n_warm)
    v = cb["value"]
    line = {"metric": METRIC, "value": v, "unit": "edit-steps/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": n_steps, "warmup": n_warm, "steps_requested": args.steps, "warmup_requested": args.warmup,
            "ms_per_step": cb["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64-accumulate/f32", "data": "synthetic",
            "config": {"workload": f"C2 SD-1.5-shape sparse edit step, {int(args.mask * 100)}% centered-square user mask",
                       "model": "sparsedit toy UNet @ SD-1.5 widths (320/640/1280/1280), 2 blocks/level",
                       "latent": "1x4x64x64", "text": "77x768", "mask_fraction": args.mask},
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "edit-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ----------------------------------------------------------------------------- kernel timing
def _op_log(eng, plan):
    """Ops (and kernel counts) of one step, in launch order (one eager step with the op log on)."""
    import torch
    eng.op_log = []
    try:
        eng.step_dev.fill_(1)
        eng.run_step(plan)
        torch.cuda.synchronize()
        return eng.op_log
    finally:
        eng.op_log = None


def replay_kernels(runner, ops, T, reps=9):
    """CUPTI kernel records of `reps` graph replays of the runner's captured step, mapped to ops.

    Returns [(op dict, critical-path us, kernel name)]: per op the MEDIAN over the replays after
    the first (L2/TLB warm) of its critical-path time, or None when the profiler's kernel records
    do not match the op log."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    n_k = sum(o["kernels"] for o in ops)
    runner.step(2)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(reps):
            runner.step(2 + i % (T - 1))
        torch.cuda.synchronize()
    ks = []
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA:
            continue
        nm = e.name
        if "fis::" not in nm:  # torch's step-counter fill, memcpy/memset records
            continue
        ks.append((e.time_range.start, e.time_range.end, nm))
    ks.sort()
    want = {"fis_gemm": "gemm", "fis_attn": "attn", "fis_gn": "gn_", "fis_gn_apply": "gn_apply",
            "fis_gn_stats": "gn_stats", "fis_pool2": "pool2", "fis_up2": "up2", "fis_softmax": "softmax",
            "fis_materialize": "materialize"}

    def one(rep):  # per-op critical-path us of one replay's kernel records, or None on a mismatch
        if len(rep) != n_k:
            return None
        pos = 0
        for o in ops:
            for _ in range(o["kernels"]):
                if want.get(o["op"], "fis") not in rep[pos][2]:
                    return None
                pos += 1
        out, i, prev_end = [], 0, None
        for o in ops:
            seg = rep[i:i + o["kernels"]]
            i += o["kernels"]
            end = max(x[1] for x in seg)
            start = min(x[0] for x in seg)
            out.append(max(0.0, end - (max(prev_end, start) if prev_end is not None else start)))
            prev_end = end if prev_end is None else max(prev_end, end)
        return out

    # replays from the end (CUPTI may miss a kernel at the very start of the profiled window)
    nrep = min(reps - 1, len(ks) // n_k) if n_k else 0
    per = [one(ks[len(ks) - (q + 1) * n_k:len(ks) - q * n_k]) for q in range(nrep)]
    per = [p for p in per if p is not None]
    if not per or per[0] is None or one(ks[-n_k:]) is None:
        from collections import Counter
        print(f"replay_kernels: {len(ks)} CUPTI kernels for {reps} x {n_k} expected, the last replay does not "
              f"match the op log; {Counter(k[2][:40] for k in ks).most_common(8)}", file=sys.stderr)
        return None
    import statistics
    last = ks[-n_k:]
    out, i = [], 0
    for j, o in enumerate(ops):
        out.append((o, statistics.median(p[j] for p in per), last[i][2]))
        i += o["kernels"]
    return out


def kernel_summary(table, step_us):
    agg = {}
    for o, us, name in table:
        if o["op"] == "fis_gemm":
            cls = "gathered conv" if o.get("gathered") else ("dense conv" if o.get("conv") else "projection GEMM")
        elif o["op"] == "fis_attn":
            cls = "attention"
        else:
            cls = o["op"]
        a = agg.setdefault(cls, [0, 0.0])
        a[0] += o["kernels"]
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    return {k: {"kernels": v[0], "us": round(v[1], 2), "share": round(v[1] / tot, 4) if tot else None}
            for k, v in sorted(agg.items(), key=lambda x: -x[1][1])} | {"sum_us": round(tot, 2),
                                                                     "step_us_events": round(step_us, 2)}


def gated_conv_flops(o, active):
    """Algorithmic FLOPs of a gathered conv launch: 2 * active rows * N * K (plan.cost pixels at
    batch 1; padding rows of stacked requests excluded)."""
    return 2.0 * active * o["n"] * o["k"]


# ----------------------------------------------------------------------------- GPU arm
def _time_runner(runner, T, steps, warmup):
    import torch
    runner.step(1)
    for i in range(warmup):
        runner.step(1 + (i + 1) % T)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        runner.step(1 + i % T)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / max(1, steps)


def run_ours(args):
    import torch
    ws, rank, local = dist_init()
    torch.cuda.set_device(local)
    import paper_2305_17423_b200 as P
    from paper_2305_17423_b200 import unet as U
    P.set_precision(args.precision)
    cfg = P.UNetConfig(**C2)
    eng = U.get_engine(cfg)
    hbm, tf_peak, peak_src = peaks()
    # --- cached generation of this rank's request (not timed: per-request setup)
    store = P.CacheStore()
    t0 = time.perf_counter()
    P.generate_dense(P.PromptTokens(OLD_IDS), cfg, store, record="engine")
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    arena = store.arena
    mask = P.centered_square_mask(cfg.latent_h, cfg.latent_w, args.mask)
    kv = eng.text_kv(P.embed_tokens(P.PromptTokens(NEW_IDS), cfg))
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    ep = U.EditPlan(eng, arena, mask, kv, lat0)
    ops = _op_log(eng, ep.plan)
    runner = U._Runner(eng, ep.plan, True)
    T = cfg.steps
    runner.step(1)  # warms + captures the step graph
    per_step_launches = runner.launches_per_step
    for i in range(args.warmup):
        runner.step(1 + (i + 1) % T)
    torch.cuda.synchronize()
    barrier()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()  # ncu --profile-from-start off captures only the timed steps
        e0.record(st)
        for i in range(args.steps):
            runner.step(1 + i % T)
        e1.record(st)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    ms = e0.elapsed_time(e1)
    barrier()
    ms = reduce_max(ms)
    per_ms = ms / max(1, args.steps)
    value = ws * args.steps / (ms / 1e3)

    # --- per-kernel times of the same captured step (CUPTI, graph replay)
    table = replay_kernels(runner, ops, T)
    unet = U.UNet(cfg)
    cost = {l: 4 * ep.dp.n_tiles[l] for l in range(cfg.levels)}
    conv_fl = sum(2 * unet.layer_macs(i, cost[i.level], 77) for i in unet.layers if i.kind == "conv" and i.gated)
    roof = {"bound": "tensor", "achieved": None, "peak": tf_peak, "unit": "TFLOP/s", "frac": None, "traffic": None}
    kern = None
    if table is not None:
        conv_us = sum(us for o, us, _ in table if o["op"] == "fis_gemm" and o.get("gathered"))
        n_conv = sum(1 for o, _, _ in table if o["op"] == "fis_gemm" and o.get("gathered"))
        ach = conv_fl / (conv_us * 1e-6) / 1e12 if conv_us else None
        roof.update(achieved=ach, frac=ach / tf_peak if ach else None,
                    traffic=conv_traffic(), kernel=f"fis_gemm gated-conv gather-GEMMs ({n_conv}/step)",
                    note=f"algorithmic {conv_fl / 1e9:.2f} GFLOP/step (2 x plan.cost x c_out x 9 c_in, reference "
                         f"SparseMode accounting) over {conv_us:.1f} us/step of gated-conv critical-path time "
                         f"(CUPTI kernel records of graph replays of the timed step, end_i - end_(i-1)); peak "
                         f"{peak_src}; traffic = ncu dram bytes per launch of the L0 gated conv "
                         f"(profiles/r02/ncu_gated_conv.json); batch 1 is latency / weight-stream bound "
                         f"(SURVEY §7 H1), the batched section carries the tensor-bound roofline")
        kern = kernel_summary(table, per_ms * 1e3)
    # --- end-to-end through the public API (host mask in, host latent out, all T steps)
    e2e_masks = [P.BinaryMask(np.roll(mask.bits, (2 * i, -2 * i), axis=(0, 1))) for i in range(E2E_CALLS)]
    sessions = [P.EditSession.create(OLD_IDS, NEW_IDS, cfg, store, user_mask=m) for m in e2e_masks]
    P.edit(P.EditSession.create(OLD_IDS, NEW_IDS, cfg, store, user_mask=mask), cfg, store)  # untimed warm-up
    import gc
    gc.collect()
    call_s = []
    for s_ in sessions:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.edit(s_, cfg, store)
        torch.cuda.synchronize()
        call_s.append(time.perf_counter() - t0)
    e2e_s = reduce_max(float(np.median(call_s)))
    # --- dense UNet step on the same GPU (what edit() runs for a full mask)
    dense_ms, dense_kern = dense_step(eng, U, P, cfg, kv, args)
    sweep = mask_sweep(eng, U, P, cfg, arena, kv, lat0, args, dense_ms) if not args.no_sweep else None
    line = {
        "metric": METRIC, "value": value, "unit": "edit-steps/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16" if args.precision == "bf16" else "f32", "data": "synthetic",
        "config": {"workload": f"C2 SD-1.5-shape sparse edit step, {int(args.mask * 100)}% centered-square user mask",
                   "model": "sparsedit toy UNet @ SD-1.5 widths (320/640/1280/1280), 2 blocks/level",
                   "latent": "1x4x64x64", "text": "77x768", "schedule_steps": T, "mask_fraction": args.mask,
                   "active_px_L0_L1": ep.dp.n_active[:2], "requests_per_gpu": 1, "parallelism": f"replicas x{ws}",
                   "l2": "inputs larger than L2 (weights + cache slab streamed per step > 126 MB); no flush",
                   "precision": args.precision, "generation_s": gen_s},
        "roofline": roof,
        "kernels": kern,
        "step_hbm": {"bytes_per_step": WEIGHT_BYTES_BF16, "achieved_gbs": WEIGHT_BYTES_BF16 / (per_ms / 1e3) / 1e9,
                     "peak_gbs": hbm, "frac": WEIGHT_BYTES_BF16 / (per_ms / 1e3) / 1e9 / hbm,
                     "note": "whole step vs the weight-streaming floor (221.7 M bf16 params read once per step)"},
        "dense_baseline": {"ms_per_step": dense_ms, "steps_per_s": 1e3 / dense_ms, "sparse_speedup": dense_ms / per_ms,
                           "tflops": 310.0 / dense_ms, "frac_of_peak": 310.0 / dense_ms / tf_peak,
                           "kernels": dense_kern,
                           "note": "dense C2 step (310.0 GFLOP algorithmic) on the same GPU, one graph replay each"},
        "gpu_launches": per_step_launches * args.steps,
        "clocks": clk.summary(),
        "e2e": {"value": T / e2e_s, "unit": "edit-steps/s", "h2d_bytes_per_step": (cfg.latent_h * cfg.latent_w * 17) // T,
                "d2h_bytes_per_step": (4 * cfg.latent_h * cfg.latent_w * cfg.latent_channels + 64) // T,
                "note": f"median of {E2E_CALLS} consecutive P.edit() calls after one untimed warm-up call (each: "
                        "T steps, planning, text K/V, H2D mask/latent, D2H result; step graphs reused when the launch "
                        "shapes match, inputs copied in)",
                "call_seconds": [round(x, 5) for x in call_s]},
    }
    if sweep is not None:
        line["sweep"] = sweep
    del runner, ep
    # --- the same step in the fp32 parity precision (SIMT fp32; the numerics of tensors.py:76-94)
    if args.precision == "bf16" and not args.no_fp32:
        line["fp32_parity"] = fp32_parity_step(U, P, cfg, args, mask, "tf32x3")
        line["fp32_parity_simt"] = fp32_parity_step(U, P, cfg, args, mask, "fp32")
    # --- C4: SD-2 shape, multi-round edits against one HBM generation
    if not args.no_c4:
        line["c4"] = c4_section(U, P, args)
    # --- C5: 64 requests over the box, each GPU's share as one stacked batch
    R = args.requests if args.requests > 0 else max(1, 64 // ws)
    if R > 1 and args.precision == "bf16":
        from paper_2305_17423_b200 import dist as D
        store.close()
        del store, arena
        # the fp32 / tf32x3 / C4 engines of the sections above are not used again: release their
        # weights and workspaces so the 64-request arena and its step graph allocate without churn
        for k in [k for k, e in U._ENGINES.items() if e is not eng]:
            del U._ENGINES[k]
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        costs = [D.request_cost(_request(i, cfg)[2]) for i in range(R * ws)]
        ids = D.shard_requests(costs, ws)[rank]
        batched = stacked_requests(eng, U, P, cfg, args, tf_peak, ids=ids)
        batched["edit_steps_per_s_all_ranks"] = ws * len(ids) * 1e3 / reduce_max(batched["ms_per_batched_step"])
        line["batched"] = batched
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.mask, 1, 0)
    if rank == 0:
        print(json.dumps(line))
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


def conv_traffic():
    """DRAM bytes per launch of the profiled gated-conv GEMM (committed ncu --set full capture)."""
    for r in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", r, "ncu_gated_conv.json")) as f:
                return json.load(f)["traffic_bytes_per_launch"]
        except Exception:
            continue
    return None


def dense_step(eng, U, P, cfg, kv, args):
    """Dense forward + step update of the same UNet (no recording), one graph replay per step."""
    import torch
    lat = torch.empty((cfg.steps + 1, eng.hw(0), cfg.latent_channels), dtype=torch.float32, device=eng.dev)
    lat[0].copy_(U._to_nhwc(P.initial_latent(cfg), eng.dev))
    plan = U.StepPlan(eng, kv, lat, None)
    ops = _op_log(eng, plan)
    runner = U._Runner(eng, plan, True)
    ms = _time_runner(runner, cfg.steps, max(5, args.steps // 2), 3)
    table = replay_kernels(runner, ops, cfg.steps)
    return ms, (kernel_summary(table, ms * 1e3) if table is not None else None)


def random_dilated(P, cfg, seed, frac=0.10):
    """SURVEY §8 C1/C3 random-dilated mask: dilate(PCG64(s).random((H, W)) < f / 9, 1)."""
    g = np.random.Generator(np.random.PCG64(seed))
    return P.dilate(P.BinaryMask(g.random((cfg.latent_h, cfg.latent_w)) < frac / 9), 1)


def mask_sweep(eng, U, P, cfg, arena, kv, lat0, args, dense_ms):
    """C3 (cli.py:304-365): sparse step vs mask ratio on the same cache and GPU; 100% is the dense
    step edit() runs for a full mask (unet.py:877-878)."""
    unet = U.UNet(cfg)
    out = []
    cases = [(f, f"centered square {f:.0%}", P.centered_square_mask(cfg.latent_h, cfg.latent_w, f))
             for f in (0.01, 0.05, 0.10, 0.25, 0.50, 1.0)]
    cases.append((0.10, "random dilated 10% (seed 0)", random_dilated(P, cfg, 0)))
    dense_gfl = 2 * sum(unet.dense_step_macs(77).values()) / 1e9
    for f, name, mask in cases:
        if mask.all_active():
            ms, act, gfl = dense_ms, cfg.latent_h * cfg.latent_w, dense_gfl
        else:
            ep = U.EditPlan(eng, arena, mask, kv, lat0)
            ms = _time_runner(U._Runner(eng, ep.plan, True), cfg.steps, max(5, args.steps // 2), 3)
            cost = {l: 4 * ep.dp.n_tiles[l] for l in range(cfg.levels)}
            gfl = 2 * sum(unet.sparse_step_macs(77, ep.dp.n_active, cost).values()) / 1e9
            act = ep.dp.n_active[0]
        out.append({"mask": name, "mask_fraction": round(act / (cfg.latent_h * cfg.latent_w), 4),
                    "active_px_L0": act, "ms_per_step": ms, "edit_steps_per_s": 1e3 / ms,
                    "algorithmic_gflop_per_step": gfl, "speedup_vs_dense": dense_ms / ms,
                    "mac_ratio_vs_dense": dense_gfl / gfl})
    return out


def fp32_parity_step(U, P, cfg, args, mask, precision="fp32"):
    """The C2 sparse step with fp32 operands: "fp32" (SIMT FFMA, the reference numerics) or
    "tf32x3" (tcgen05 kind::tf32, 3xTF32 split, fp32 accumulate)."""
    import torch
    eng = U.get_engine(cfg, precision)
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens(OLD_IDS), cfg, store, record="engine", precision=precision)
    kv = eng.text_kv(P.embed_tokens(P.PromptTokens(NEW_IDS), cfg))
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    ep = U.EditPlan(eng, store.arena, mask, kv, lat0)
    ms = _time_runner(U._Runner(eng, ep.plan, True), cfg.steps, max(5, args.steps // 2), 3)
    store.close()
    del ep, store
    torch.cuda.empty_cache()
    note = {"fp32": "set_precision('fp32'): fp32 operands / accumulation on SIMT FFMA GEMMs",
            "tf32x3": "set_precision('tf32x3'): fp32 operands on the tcgen05 tensor cores as 3xTF32 (big*big + "
                      "big*small + small*big, kind::tf32, fp32 accumulate)"}[precision]
    return {"ms_per_step": ms, "edit_steps_per_s": 1e3 / ms, "dtype": "f32", "precision": precision,
            "note": f"same C2 10% step, {note}; pinned to the oracle at <= 1e-4 latent max-abs per sampled step "
                    "(tests/test_gpu_c2_parity.py)"}


def c4_section(U, P, args):
    """BASELINE configs[3]: SD-2 shape (96x96 latent, 1024-wide text), bf16. Device-timed sparse
    step at 10% and end-to-end edit() rounds (new prompt + mask each) on ONE HBM generation."""
    import torch
    cfg = P.UNetConfig(**C4)
    eng = U.get_engine(cfg, "bf16")
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens(OLD_IDS), cfg, store, record="engine", precision="bf16")
    kv = eng.text_kv(P.embed_tokens(P.PromptTokens(NEW_IDS), cfg))
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    mask = P.centered_square_mask(96, 96, 0.10)
    ep = U.EditPlan(eng, store.arena, mask, kv, lat0)
    ms = _time_runner(U._Runner(eng, ep.plan, True), cfg.steps, max(5, args.steps // 2), 3)
    dense_ms, _ = dense_step(eng, U, P, cfg, kv, args)
    rounds = []
    for k, f in enumerate((0.10, 0.05, 0.25)):
        new = tuple(200 + k if i == 3 + k else v for i, v in enumerate(OLD_IDS))
        m = P.BinaryMask(np.roll(P.centered_square_mask(96, 96, f).bits, (6 * k, -4 * k), axis=(0, 1)))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.edit(P.EditSession.create(OLD_IDS, new, cfg, store, user_mask=m), cfg, store)
        torch.cuda.synchronize()
        rounds.append({"mask_fraction": f, "seconds": time.perf_counter() - t0})
    store.close()
    del ep, store
    torch.cuda.empty_cache()
    return {"ms_per_step": ms, "edit_steps_per_s": 1e3 / ms, "dense_ms_per_step": dense_ms,
            "sparse_speedup": dense_ms / ms, "rounds_e2e": rounds,
            "e2e_edit_steps_per_s": [cfg.steps / r["seconds"] for r in rounds],
            "note": "96x96x4 latent, 77x1024 text, 10% centered square; rounds = successive edit() calls (new "
                    "prompt and mask each, incl. planning and graph capture) against one recorded generation"}


def _request(r, cfg):
    """Request r of the C5 mix: own prompt pair and a 5/10/25% square mask at its own offset."""
    fracs = (0.05, 0.10, 0.25)
    old = tuple((i * 7 + r) % 49000 + 1 for i in range(77))
    new = tuple(99 + r if i == 3 else v for i, v in enumerate(old))
    side = int(round((fracs[r % 3] * cfg.latent_h * cfg.latent_w) ** 0.5))
    y0, x0 = (7 * r) % (cfg.latent_h - side), (13 * r) % (cfg.latent_w - side)
    bits = np.zeros((cfg.latent_h, cfg.latent_w), dtype=bool)
    bits[y0:y0 + side, x0:x0 + side] = True
    return old, new, bits


def stacked_requests(eng, U, P, cfg, args, peak_tf, ids):
    """C5 throughput on one GPU: this rank's requests stepped as ONE stacked batch
    (BatchedEditPlan: concatenated rows, every weight read once per step for all of them;
    block-diagonal segment attention). Device-timed edit-steps/s, the gated-conv gather-GEMMs'
    tensor-core rate inside graph replays of that step (CUPTI), and one end-to-end edit_batch()
    call (host masks / prompts in, host latents out)."""
    import torch
    t0 = time.perf_counter()
    ids = list(ids)
    R = len(ids)
    reqs = [_request(r, cfg) for r in ids]
    stores = [P.CacheStore() for _ in reqs]
    eng.ns = 0
    U.generate_dense_batch([P.PromptTokens(o) for o, _, _ in reqs], cfg, stores)
    stacked = stores[0].arena.stacked
    setup_s = time.perf_counter() - t0
    kvs = [eng.text_kv(P.embed_tokens(P.PromptTokens(n), cfg)) for _, n, _ in reqs]
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    bp = U.BatchedEditPlan(eng, stacked, [P.BinaryMask(b) for _, _, b in reqs], kvs, [lat0] * R)
    ops = _op_log(eng, bp.plan)
    run = U._Runner(eng, bp.plan, True, ns=0)
    ms = _time_runner(run, cfg.steps, max(5, args.steps // 2), 3)
    # end to end through the public API: R sessions (host masks, prompts) in, R host latents out;
    # one untimed call first (its graph capture and allocations), then the median of five calls
    mk = lambda: [P.EditSession.create(o, n, cfg, st_, user_mask=P.BinaryMask(b)) for (o, n, b), st_ in zip(reqs, stores)]
    P.edit_batch(mk(), cfg)
    import gc
    e2e_calls = []
    for _ in range(5):
        sessions = mk()
        gc.collect()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        results = P.edit_batch(sessions, cfg)
        torch.cuda.synchronize()
        e2e_calls.append(time.perf_counter() - t1)
    e2e_s = float(np.median(e2e_calls))
    eng.ns = 0
    table = replay_kernels(run, ops, cfg.steps)
    active = {l: sum(dp.n_active[l] for dp in bp.dps) for l in range(cfg.levels)}
    padded = {l: bp.lists[l][2] for l in bp.lists}
    gc_ = None
    kern = None
    if table is not None:
        conv_us, conv_fl = 0.0, 0.0
        per = []
        for o, us, name in table:
            if o["op"] == "fis_gemm" and o.get("gathered"):
                lvl = o.get("level")
                if lvl is None:
                    lvl = next(l for l in padded if padded[l] == o["m"])
                conv_us += us
                fl = gated_conv_flops(o, active[lvl])
                conv_fl += fl
                per.append({"m_rows": o["m"], "n": o["n"], "k": o["k"], "us": round(us, 2), "halo": o.get("halo"),
                            "tflops": round(fl / (us * 1e-6) / 1e12, 1) if us else None})
        tf = conv_fl / (conv_us * 1e-6) / 1e12 if conv_us else 0.0
        gc_ = {"bound": "tensor", "achieved": tf, "peak": peak_tf, "unit": "TFLOP/s",
               "frac": tf / peak_tf if peak_tf else None, "gflop_per_step": conv_fl / 1e9,
               "us_per_step": conv_us, "per_launch": per,
               "note": "gathered (select-on-read) 3x3 conv GEMMs of the stacked step; algorithmic FLOPs = 2 x active "
                       "rows x N x K (16-row request padding excluded); CUPTI critical-path time in graph replay"}
        kern = kernel_summary(table, ms * 1e3)
    from paper_2305_17423_b200 import dist as D
    t2 = time.perf_counter()
    gathered = D.gather_results({i: r.latent for i, r in zip(ids, results)}, D.dist.get_world_size()
                                if D.is_dist() else 1, device=eng.dev)
    gather_s = time.perf_counter() - t2
    return {"requests_per_gpu": R, "edit_steps_per_s": R * 1e3 / ms, "ms_per_batched_step": ms,
            "rows_L0_L1": [padded[0], padded.get(1)], "active_L0_L1": [active[0], active[1]],
            "gated_conv": gc_, "kernels": kern,
            "e2e": {"edit_steps_per_s": R * cfg.steps / e2e_s, "seconds": e2e_s,
                    "call_seconds": [round(x, 4) for x in e2e_calls],
                    "note": "median of 5 edit_batch() calls after an untimed one: R sessions (host masks, prompts) -> "
                            "R host latents, all T steps incl. planning and graph capture"},
            "result_gather": {"requests_on_rank0": len(gathered), "seconds": gather_s},
            "setup_generation_s": setup_s,
            "masks": "5/10/25% squares at distinct offsets, distinct prompts, own cached generations",
            "note": "C5: 64 requests sharded by estimated cost over the GPUs (LPT), each GPU's ~64/N stepped as ONE "
                    "stacked batch; no collective in the step, one final gather of the edited latents to rank 0"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mask", type=float, default=0.10)
    ap.add_argument("--precision", default="bf16", choices=["fp32", "tf32x3", "bf16"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-fp32", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--requests", type=int, default=0,
                    help="requests per GPU of the C5 batched measurement (0: 64 / n_gpus; 1 disables)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
