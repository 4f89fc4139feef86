"""cProfile of one warm single-request edit() call at C2 (host overhead of bench.py's e2e)."""
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
    P.set_precision("bf16")
    cfg = P.UNetConfig(**bench.C2)
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens(bench.OLD_IDS), cfg, store, record="engine")
    mask = P.centered_square_mask(64, 64, 0.10)

    def call():
        s = P.EditSession.create(bench.OLD_IDS, bench.NEW_IDS, cfg, store, user_mask=mask)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.edit(s, cfg, store)
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    print("cold", call())
    pr = cProfile.Profile()
    pr.enable()
    t = call()
    pr.disable()
    print("warm", t)
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
