"""One eager batched step (R requests, C2 shapes) between cudaProfilerStart/Stop, for an ncu launch
list; prints the launch sequence (entry point, m, n, k) so the list can be matched op by op."""
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
    R = int(os.environ.get("R", "8"))
    P.set_precision("bf16")
    cfg = P.UNetConfig(**bench.C2)
    eng = U.get_engine(cfg)
    reqs = [bench._request(r, cfg) for r in range(R)]
    stores = [P.CacheStore() for _ in reqs]
    U.generate_dense_batch([P.PromptTokens(o) for o, _, _ in reqs], cfg, stores)
    kvs = [eng.text_kv(P.embed_tokens(P.PromptTokens(n), cfg)) for _, n, _ in reqs]
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    bp = U.BatchedEditPlan(eng, stores[0].arena.stacked, [P.BinaryMask(b) for _, _, b in reqs], kvs, [lat0] * R)
    eng.step_dev.fill_(1)
    eng.run_step(bp.plan)
    torch.cuda.synchronize()
    seq = []
    orig = L.call

    def rec(name, args):
        d = {"op": name}
        for f in ("m", "n", "k", "rows", "n_keys", "nseg", "max_seg_q", "hw", "n_img"):
            v = getattr(args, f, None)
            if isinstance(v, int):
                d[f] = v
        seq.append(d)
        return orig(name, args)

    L.call = rec
    torch.cuda.profiler.start()
    eng.run_step(bp.plan)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    L.call = orig
    for i, d in enumerate(seq):
        print(i, json.dumps(d))


if __name__ == "__main__":
    main()
