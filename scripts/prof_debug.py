import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import bench as B
import paper_2305_17423_b200 as P
from paper_2305_17423_b200 import unet as U
P.set_precision("bf16")
cfg = P.UNetConfig(**B.C2)
eng = U.get_engine(cfg)
store = P.CacheStore()
P.generate_dense(P.PromptTokens(B.OLD_IDS), cfg, store, record="engine")
mask = P.centered_square_mask(64, 64, 0.1)
kv = eng.text_kv(P.embed_tokens(P.PromptTokens(B.NEW_IDS), cfg))
lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
ep = U.EditPlan(eng, store.arena, mask, kv, lat0)
ops = B._op_log(eng, ep.plan)
run = U._Runner(eng, ep.plan, True)
run.step(1)
print("ops", len(ops), "kernels", sum(o["kernels"] for o in ops), "launches_per_step", run.launches_per_step)
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(3):
        run.step(2 + i)
    torch.cuda.synchronize()
ev = prof.events()
from collections import Counter
c = Counter((str(e.device_type), e.name[:60]) for e in ev)
for k, v in c.most_common(40):
    print(v, k)
ks = [e for e in ev if e.device_type == torch.autograd.DeviceType.CUDA]
print("cuda events", len(ks))
ks.sort(key=lambda e: e.time_range.start)
for e in ks[:10]:
    print(e.name[:80], e.time_range.start, e.time_range.end)
