"""Run the C2 sparse step through the step VM a few times (for ncu --kernel-name vm_kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_17423_b200 as P  # noqa: E402
from paper_2305_17423_b200 import unet as U  # noqa: E402

P.set_precision("bf16")
C2 = dict(latent_h=64, latent_w=64, latent_channels=4, channels=(320, 640, 1280, 1280), blocks_per_level=2,
          groups=32, steps=50, t1=5, t2=10, gate_fraction=0.25, dilation_radius=1, text_dim=768, vocab_size=49408,
          seed=0)
cfg = P.UNetConfig(**{**C2, "steps": 2, "t1": 1, "t2": 1})
eng = U.get_engine(cfg)
old = tuple(range(1, 78))
new = tuple(99 if i == 3 else v for i, v in enumerate(old))
store = P.CacheStore()
eng.use_vm = False  # generation through the per-op path: the profiled launches are the edit's VM steps
P.generate_dense(P.PromptTokens(old), cfg, store, record="engine")
eng.use_vm = True
kv = eng.text_kv(P.embed_tokens(P.PromptTokens(new), cfg))
lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
ep = U.EditPlan(eng, store.arena, P.centered_square_mask(64, 64, float(os.environ.get("MASK", "0.1"))), kv, lat0)
vm = eng.record_step(ep.plan)
for i in range(int(os.environ.get("N", "3"))):
    eng.step_dev.fill_(1 + i % 2)
    vm.run()
torch.cuda.synchronize()
print("ok")
