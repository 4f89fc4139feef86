"""One graph replay of the C2 batch-1 sparse step between cudaProfilerStart/Stop (for ncu
--profile-from-start off): python scripts/prof_step.py [--dense]"""
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
if "--dense" in sys.argv:
    lat = torch.empty((cfg.steps + 1, eng.hw(0), 4), dtype=torch.float32, device=eng.dev)
    lat[0].copy_(lat0)
    plan = U.StepPlan(eng, kv, lat, None)
else:
    plan = U.EditPlan(eng, store.arena, P.centered_square_mask(64, 64, 0.10), kv, lat0).plan
run = U._Runner(eng, plan, True)
for t in range(1, 6):
    run.step(t)
torch.cuda.synchronize()
torch.cuda.profiler.start()
run.step(7)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
