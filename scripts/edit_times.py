"""Wall time of consecutive single-request edit() calls at C2 (e2e variance diagnosis)."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import numpy as np
    import torch
    import paper_2305_17423_b200 as P
    P.set_precision("bf16")
    cfg = P.UNetConfig(**bench.C2)
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens(bench.OLD_IDS), cfg, store, record="engine")
    mask = P.centered_square_mask(64, 64, 0.10)
    for i in range(12):
        b = np.roll(mask.bits, (2 * (i % 3), -2 * (i % 3)), axis=(0, 1))
        s = P.EditSession.create(bench.OLD_IDS, bench.NEW_IDS, cfg, store, user_mask=P.BinaryMask(b))
        gc.collect()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.edit(s, cfg, store)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(i, round((t1 - t0) * 1e3, 1), "ms", flush=True)


if __name__ == "__main__":
    main()
