"""Wall times of consecutive edit_batch() calls (64 stacked C2 requests) with a cProfile of the
slowest: python scripts/edit_batch_times.py [R]"""
import cProfile, gc, io, os, pstats, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import bench as B
import paper_2305_17423_b200 as P
R = int(sys.argv[1]) if len(sys.argv) > 1 else 64
P.set_precision("bf16")
cfg = P.UNetConfig(**B.C2)
reqs = [B._request(r, cfg) for r in range(R)]
stores = [P.CacheStore() for _ in reqs]
P.generate_dense_batch([P.PromptTokens(o) for o, _, _ in reqs], cfg, stores)
mk = lambda: [P.EditSession.create(o, n, cfg, st, user_mask=P.BinaryMask(b)) for (o, n, b), st in zip(reqs, stores)]
P.edit_batch(mk(), cfg)
times, profs = [], []
for i in range(6):
    s = mk()
    gc.collect()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t = time.perf_counter()
    pr.enable()
    P.edit_batch(s, cfg)
    torch.cuda.synchronize()
    pr.disable()
    times.append(time.perf_counter() - t)
    profs.append(pr)
    print(f"call {i}: {times[-1]:.3f} s  allocated {torch.cuda.memory_allocated() / 1e9:.1f} GB  reserved "
          f"{torch.cuda.memory_reserved() / 1e9:.1f} GB  free {torch.cuda.mem_get_info()[0] / 1e9:.1f} GB", flush=True)
print("calls (s):", [round(x, 3) for x in times])
k = int(np.argmax(times))
out = io.StringIO()
pstats.Stats(profs[k], stream=out).sort_stats(os.environ.get("SORT", "cumulative")).print_stats(40)
print(out.getvalue()[:6000])
