"""One graph replay of the R-request stacked C2 step between cudaProfilerStart/Stop (ncu)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import bench as B
import paper_2305_17423_b200 as P
from paper_2305_17423_b200 import unet as U
R = int(sys.argv[1]) if len(sys.argv) > 1 else 64
P.set_precision("bf16")
cfg = P.UNetConfig(**B.C2)
eng = U.get_engine(cfg)
reqs = [B._request(r, cfg) for r in range(R)]
stores = [P.CacheStore() for _ in reqs]
U.generate_dense_batch([P.PromptTokens(o) for o, _, _ in reqs], cfg, stores)
kvs = [eng.text_kv(P.embed_tokens(P.PromptTokens(n), cfg)) for _, n, _ in reqs]
lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
bp = U.BatchedEditPlan(eng, stores[0].arena.stacked, [P.BinaryMask(b) for _, _, b in reqs], kvs, [lat0] * R)
run = U._Runner(eng, bp.plan, True)
for t in range(1, 4):
    run.step(t)
torch.cuda.synchronize()
torch.cuda.profiler.start()
run.step(5)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
