"""Host-side phase times of one warm P.edit() call at C2 (batch 1): where the end-to-end time
beyond the 50 device steps goes. python scripts/edit_phases.py"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import bench as B
import paper_2305_17423_b200 as P
from paper_2305_17423_b200 import unet as U

P.set_precision("bf16")
cfg = P.UNetConfig(**B.C2)
store = P.CacheStore()
P.generate_dense(P.PromptTokens(B.OLD_IDS), cfg, store, record="engine")
mask = P.centered_square_mask(64, 64, 0.10)
sess = lambda: P.EditSession.create(B.OLD_IDS, B.NEW_IDS, cfg, store, user_mask=mask)
for _ in range(2):
    P.edit(sess(), cfg, store)
torch.cuda.synchronize()

T = {}
def tick(name, t0):
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    T[name] = T.get(name, 0.0) + (t1 - t0) * 1e3
    return t1

for rep in range(5):
    t = time.perf_counter()
    s = sess(); t = tick("session", t)
    unet = U.UNet(cfg); t = tick("UNet()", t)
    outcome = U.detect_mask(s, cfg, store); t = tick("detect_mask", t)
    arena = U._arena_of(store, cfg, 1); t = tick("arena_of", t)
    eng = U.get_engine(cfg, arena.eng.precision); t = tick("get_engine", t)
    emb = P.embed_tokens(s.new_tokens, cfg); t = tick("embed_tokens", t)
    kv = eng.text_kv(emb); t = tick("text_kv", t)
    lat0 = U._to_nhwc(U.initial_latent_np(cfg), eng.dev); t = tick("initial_latent", t)
    ep = U.EditPlan(eng, arena, outcome.mask, kv, lat0); t = tick("EditPlan", t)
    run = U._cached_runner(eng, store, 1, ep, kv); t = tick("cached_runner", t)
    run.run(1, cfg.steps); t = tick("50 steps", t)
    final = ep.final_latent(eng, arena); t = tick("final_latent", t)
    lat = U._to_nchw(final, cfg.latent_channels, cfg.latent_h, cfg.latent_w); t = tick("to_nchw(D2H)", t)
    ph2 = U._MacsCounter()
    U._add_sparse_macs(ph2, unet, len(s.new_tokens.ids), ep.dp, cfg.steps); t = tick("macs", t)
    U._build_report(unet, len(s.new_tokens.ids), cfg, [outcome.phase1_macs, ph2]); t = tick("report", t)
    U._gather_plans(unet, ep.dp); t = tick("gather_plans", t)
    store.stats(); t = tick("stats", t)
tot = sum(T.values()) / 5
for k, v in T.items():
    print(f"{k:16s} {v / 5:8.3f} ms")
print(f"{'total':16s} {tot:8.3f} ms")
