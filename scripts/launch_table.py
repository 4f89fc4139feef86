"""Join an ncu launch list (gpu__time_duration CSV) with prof_batch.py's launch sequence.

    python scripts/launch_table.py gpurun_out/batch_launches.csv gpurun_out/batch_seq.txt
"""
import csv
import json
import re
import sys
from collections import defaultdict


def main(csv_path, seq_path, top=30):
    rows = list(csv.reader(open(csv_path)))
    hdr, ks = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                ks.append((d["Kernel Name"], float(d["Metric Value"].replace(",", ""))))
    seq = [json.loads(l.split(" ", 1)[1]) for l in open(seq_path) if re.match(r"^\d+ \{", l)]
    agg, cnt = defaultdict(float), defaultdict(int)
    i = 0
    for s in seq:  # a fis_attn op launches one kernel, or two (P_OUT + P_IN) when P is shared
        key = s["op"] + (f" n={s['n']} k={s['k']}" if s["op"] == "fis_gemm" else "") + f" m={s.get('m', s.get('rows'))}"
        t = ks[i][1]
        i += 1
        nxt = seq[seq.index(s) + 1]["op"] if s is not seq[-1] else None
        if s["op"] == "fis_attn" and i < len(ks) and "attn" in ks[i][0] and nxt != "fis_attn":
            t += ks[i][1]
            i += 1
        agg[key] += t
        cnt[key] += 1
    tot = sum(t for _, t in ks)
    print(f"{len(ks)} launches, {len(seq)} ops, total {tot / 1e3:.1f} us")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{v / 1e3:8.1f} us  {100 * v / tot:5.1f}%  x{cnt[k]:<3d} {k}")


if __name__ == "__main__":
    main(*sys.argv[1:3])
