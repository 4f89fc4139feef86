"""One eager C2 sparse step inside cudaProfilerStart/Stop (ncu --profile-from-start off): the first
tcgen05 GEMM launch of the step is the first gated 3x3 conv (L0 enc block, M=400 N=320 K=2880)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_17423_b200 as P  # noqa: E402
from paper_2305_17423_b200 import unet as U  # noqa: E402
P.set_precision("bf16")
cfg = P.UNetConfig(latent_h=64, latent_w=64, latent_channels=4, channels=(320, 640, 1280, 1280), blocks_per_level=2,
                   groups=32, steps=2, t1=1, t2=1, text_dim=768, vocab_size=49408, seed=0)
eng = U.get_engine(cfg)
old = tuple(range(1, 78))
new = tuple(99 if i == 3 else v for i, v in enumerate(old))
store = P.CacheStore()
P.generate_dense(P.PromptTokens(old), cfg, store, record="engine")
kv = eng.text_kv(P.embed_tokens(P.PromptTokens(new), cfg))
ep = U.EditPlan(eng, store.arena, P.centered_square_mask(64, 64, 0.1), kv, U._to_nhwc(P.initial_latent(cfg), eng.dev))
eng.step_dev.fill_(1)
eng.run_step(ep.plan)
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.run_step(ep.plan)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
