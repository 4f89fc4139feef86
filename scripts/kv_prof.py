import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench as B
import paper_2305_17423_b200 as P
from paper_2305_17423_b200 import unet as U
P.set_precision("bf16")
cfg = P.UNetConfig(**B.C2)
eng = U.get_engine(cfg)
emb = P.embed_tokens(P.PromptTokens(B.NEW_IDS), cfg)
for _ in range(3): eng.text_kv(emb)
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(10): eng.text_kv(emb)
torch.cuda.synchronize(); print("text_kv", (time.perf_counter()-t)/10*1e3, "ms")
g, eb, outs = list(eng._kv_graphs.values())[0]
t=time.perf_counter()
for _ in range(10): g.replay()
torch.cuda.synchronize(); print("replay only", (time.perf_counter()-t)/10*1e3, "ms")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g.replay(); torch.cuda.synchronize()
ks=sorted((e.time_range.start,e.time_range.end,e.name) for e in prof.events() if e.device_type==torch.autograd.DeviceType.CUDA)
print(len(ks), "kernels; span", (ks[-1][1]-ks[0][0]), "us")
from collections import Counter
c=Counter(); d=Counter()
for s,e,n in ks: c[n[:50]]+=1; d[n[:50]]+=e-s
for n in c: print(f"{c[n]:3d} {d[n]:8.1f} us  {n}")
