"""cProfile of one warm edit_batch() call with R stacked requests (host overhead of the C5 e2e)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch
    import paper_2305_17423_b200 as P
    from paper_2305_17423_b200 import unet as U
    R = int(os.environ.get("R", "64"))
    P.set_precision("bf16")
    cfg = P.UNetConfig(**bench.C2)
    reqs = [bench._request(r, cfg) for r in range(R)]
    stores = [P.CacheStore() for _ in reqs]
    U.generate_dense_batch([P.PromptTokens(o) for o, _, _ in reqs], cfg, stores)

    def call():
        ss = [P.EditSession.create(o, n, cfg, st, user_mask=P.BinaryMask(b)) for (o, n, b), st in zip(reqs, stores)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.edit_batch(ss, cfg)
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    print("cold", call())
    pr = cProfile.Profile()
    pr.enable()
    t = call()
    pr.disable()
    print("warm", t)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
