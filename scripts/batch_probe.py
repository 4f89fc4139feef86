"""Stacked-batch throughput vs R at C2 shapes (bench.py's stacked_requests)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--R", default="1,2,4,8,16")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--streams", action="store_true")
    args = ap.parse_args()
    import paper_2305_17423_b200 as P
    from paper_2305_17423_b200 import unet as U
    P.set_precision("bf16")
    cfg = P.UNetConfig(**bench.C2)
    eng = U.get_engine(cfg)
    for R in [int(x) for x in args.R.split(",")]:
        d = bench.stacked_requests(eng, U, P, cfg, R, args, 1633.8)
        out = {"R": R, "stacked_steps_per_s": d["edit_steps_per_s"], "ms_per_batched_step": d["ms_per_batched_step"],
               "gated_conv_tflops": d["gated_conv"]["achieved_tflops"], "e2e": d["e2e"]["edit_steps_per_s"]}
        if args.streams and R > 1:
            bv, bms = bench.batched_requests(eng, U, P, cfg, R, args)
            out.update(streams_steps_per_s=bv, streams_ms_per_round=bms)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
