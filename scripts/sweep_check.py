import os, sys
sys.path.insert(0, os.getcwd())
import torch
import bench as B
import paper_2305_17423_b200 as P
from paper_2305_17423_b200 import unet as U
P.set_precision("bf16")
cfg = P.UNetConfig(**B.C2)
eng = U.get_engine(cfg)
store = P.CacheStore()
P.generate_dense(P.PromptTokens(B.OLD_IDS), cfg, store, record="engine")
kv = eng.text_kv(P.embed_tokens(P.PromptTokens(B.NEW_IDS), cfg))
lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
for frac in (0.05, 0.10, 0.05, 0.10):
    ep = U.EditPlan(eng, store.arena, P.centered_square_mask(64, 64, frac), kv, lat0)
    run = U._Runner(eng, ep.plan, True)
    ms = B._time_runner(run, cfg.steps, 20, 3)
    print(frac, round(ms, 4), flush=True)
