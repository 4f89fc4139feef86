"""One eager single-request sparse step (C2, 10% mask; bench.py's main workload) between
cudaProfilerStart/Stop, printing the launch sequence (for ncu launch lists)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch
    import paper_2305_17423_b200 as P
    from paper_2305_17423_b200 import _lib as L
    from paper_2305_17423_b200 import unet as U
    P.set_precision("bf16")
    cfg = P.UNetConfig(**bench.C2)
    eng = U.get_engine(cfg)
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens(bench.OLD_IDS), cfg, store, record="engine")
    mask = P.centered_square_mask(cfg.latent_h, cfg.latent_w, 0.10)
    kv = eng.text_kv(P.embed_tokens(P.PromptTokens(bench.NEW_IDS), cfg))
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    ep = U.EditPlan(eng, store.arena, mask, kv, lat0)
    eng.step_dev.fill_(1)
    eng.run_step(ep.plan)
    torch.cuda.synchronize()
    seq, orig = [], L.call

    def rec(name, args):
        d = {"op": name}
        for f in ("m", "n", "k", "rows", "n_keys", "hw"):
            v = getattr(args, f, None)
            if isinstance(v, int):
                d[f] = v
        seq.append(d)
        return orig(name, args)

    L.call = rec
    torch.cuda.profiler.start()
    eng.run_step(ep.plan)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    L.call = orig
    for i, d in enumerate(seq):
        print(i, json.dumps(d))


if __name__ == "__main__":
    main()
