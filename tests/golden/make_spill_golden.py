"""Golden spill file written by the REAL reference package (run in the build container).

    python tests/golden/make_spill_golden.py [/root/reference/pkg/src]

Writes tests/golden/ref_spill_small.bin: the reference's generate_dense of a 2-step tiny
config into a CacheStore with a spill path, flushed and closed (reference cache.py:216-276,
580-600, 649-673), plus ref_spill_small.npz with what the reference's own open_spill reads
back for every entry. tests/test_spill_format.py checks this package's reader against both.
"""

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")

import sparsedit as sd  # noqa: E402
from sparsedit import unet as un  # noqa: E402

CFG = dict(latent_h=32, latent_w=32, channels=(8, 16), blocks_per_level=1, groups=4, steps=2, t1=1, t2=2,
           text_dim=8, seed=7)

if __name__ == "__main__":
    path = HERE / "ref_spill_small.bin"
    cfg = un.UNetConfig(**CFG)
    with sd.CacheStore(spill_path=path, async_transfer=False) as st:
        un.generate_dense(un.PromptTokens((3, 5, 7, 11)), cfg, st)
        st.flush_all()
    out = {}
    with sd.CacheStore.open_spill(path, async_transfer=False) as st:
        for k in sorted(st.keys()):
            out[f"{k.step}_{k.layer_id}_{int(k.role)}"] = np.asarray(sd.cache.materialize_payload(st.get(k)))
    np.savez_compressed(HERE / "ref_spill_small.npz", **out)
    print(path, path.stat().st_size, len(out), "entries")
