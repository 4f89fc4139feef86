"""cProfile of one edit_batch() call (R stacked requests, C2) after a warm-up call."""
import cProfile, os, pstats, sys, time
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
mk = lambda: [P.EditSession.create(o, n, cfg, st, user_mask=P.BinaryMask(b)) for (o, n, b), st in zip(reqs, stores)]
P.edit_batch(mk(), cfg)
torch.cuda.synchronize()
for i in range(2):
    s = mk()
    t0 = time.perf_counter()
    P.edit_batch(s, cfg)
    torch.cuda.synchronize()
    print("edit_batch seconds", time.perf_counter() - t0)
s = mk()
pr = cProfile.Profile()
pr.enable()
P.edit_batch(s, cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
