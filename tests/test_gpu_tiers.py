"""Cache tiers beyond HBM and persistence on the device engine.

  * spill: generate -> flush_all (cache.bin in the reference layout + engine sidecar) -> close ->
    CacheStore.open_spill -> edit equals the edit on the in-memory generation bit for bit, and
    `get` of reference roles from the file equals `get` from HBM;
  * tiers: with a hot_budget below two generations, binding the second moves the least recently
    used one to pinned host memory; an edit on it promotes it back (a blocking load), `prefetch`
    promotes it ahead (a prefetch hit); results bit-identical to never-tiered edits;
  * CLI: generate / edit / sweep end to end with the reference's files and reports.
"""

import json

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA GPU")]

CFG = dict(latent_h=32, latent_w=32, channels=(64, 128), blocks_per_level=1, groups=4, steps=4, t1=1, t2=2,
           text_dim=64, seed=5)
OLD, NEW = (3, 5, 7, 11), (3, 5, 9, 11)


@pytest.fixture(scope="module")
def P():
    import paper_2305_17423_b200 as P
    P.set_precision("bf16")
    yield P
    P.set_precision("fp32")


def _mask(P, y0, x0, side):
    b = np.zeros((32, 32), bool)
    b[y0:y0 + side, x0:x0 + side] = True
    return P.BinaryMask(b)


def test_spill_roundtrip_edit_bitwise(P, tmp_path):
    cfg = P.UNetConfig(**CFG)
    path = tmp_path / "cache.bin"
    store = P.CacheStore(spill_path=path)
    final = P.generate_dense(P.PromptTokens(OLD), cfg, store, record="full")
    m = _mask(P, 4, 6, 10)
    want = P.edit(P.EditSession.create(OLD, NEW, cfg, store, user_mask=m), cfg, store)
    ref_keys = [k for k in store.keys()][:40]
    ref_vals = {k: store.get(k) for k in ref_keys}
    store.flush_all()
    store.close()
    back = P.CacheStore.open_spill(path)
    for k in ref_keys:  # served from the file (reference record layout)
        assert np.array_equal(back.get(k), ref_vals[k]), k
    got = P.edit(P.EditSession.create(OLD, NEW, cfg, back, user_mask=m), cfg, back)
    assert np.array_equal(got.latent, want.latent)
    assert np.array_equal(got.latent[:, :, ~m.bits], final[:, :, ~m.bits])
    st = back.stats()
    assert st.blocking_loads == 1 and st.transfer_count >= 1
    back.close()


def test_hbm_budget_tiers_to_host_and_back(P):
    cfg = P.UNetConfig(**CFG)
    m = _mask(P, 8, 8, 12)
    # reference results on untiered stores
    want = {}
    for old in (OLD, (2, 4, 6)):
        s = P.CacheStore()
        P.generate_dense(P.PromptTokens(old), cfg, s, record="engine")
        want[old] = P.edit(P.EditSession.create(old, NEW, cfg, s, user_mask=m), cfg, s).latent
        s.close()
    a, b = P.CacheStore(hot_budget=1), P.CacheStore(hot_budget=1)  # budget below one generation
    P.generate_dense(P.PromptTokens(OLD), cfg, a, record="engine")
    P.generate_dense(P.PromptTokens((2, 4, 6)), cfg, b, record="engine")
    assert a._state == "cold" and b._state == "hot"  # LRU `a` went to pinned host memory
    assert a.stats().cold_bytes > 0 and a.stats().hot_bytes == 0
    ra = P.edit(P.EditSession.create(OLD, NEW, cfg, a, user_mask=m), cfg, a)  # promotes `a`, evicts `b`
    assert a.stats().blocking_loads == 1 and b._state == "cold"
    assert a.stats().evict_warnings >= 1  # a generation alone above the budget stays hot (warned)
    b.prefetch(1)  # copy engine starts promoting `b` before its edit
    rb = P.edit(P.EditSession.create((2, 4, 6), NEW, cfg, b, user_mask=m), cfg, b)
    assert b.stats().prefetch_hits == 1 and b.stats().blocking_loads == 0
    assert np.array_equal(ra.latent, want[OLD]) and np.array_equal(rb.latent, want[(2, 4, 6)])
    a.close()
    b.close()


def test_cli_generate_edit_sweep(P, tmp_path):
    from paper_2305_17423_b200 import cli
    from paper_2305_17423_b200.tensors import load_tensor, save_tensor
    cfg = P.UNetConfig(**CFG)
    (tmp_path / "cfg.json").write_text(json.dumps(cfg.to_json()))
    gen = tmp_path / "gen"
    assert cli.main(["--precision", "bf16", "generate", "--config", str(tmp_path / "cfg.json"), "--prompt",
                     *map(str, OLD), "--out", str(gen)]) == 0
    man = json.loads((gen / "manifest.json").read_text())
    assert man["prompt"] == list(OLD) and (gen / "cache.bin").is_file() and (gen / "final.ft4").is_file()
    m = _mask(P, 4, 6, 10)
    save_tensor(tmp_path / "mask.ft4", P.mask_to_tensor(m))
    sess = {"config": cfg.to_json(), "old_tokens": list(OLD), "new_tokens": list(NEW), "prior_dir": "gen",
            "user_mask": "mask.ft4"}
    (tmp_path / "session.json").write_text(json.dumps(sess))
    assert cli.main(["--precision", "bf16", "edit", "--session", str(tmp_path / "session.json"), "--out",
                     str(tmp_path / "ed")]) == 0
    rep = json.loads((tmp_path / "ed" / "report.json").read_text())
    cli.BenchReport.from_json(rep)
    # the CLI's edit equals the API edit on an in-memory generation
    s = P.CacheStore()
    P.generate_dense(P.PromptTokens(OLD), cfg, s)
    api = P.edit(P.EditSession.create(OLD, NEW, cfg, s, user_mask=m), cfg, s)
    assert np.array_equal(load_tensor(tmp_path / "ed" / "edited.ft4"), api.latent)
    assert rep["runs"][0]["sparse_macs"] == api.macs.sparse_total
    assert cli.main(["--precision", "bf16", "sweep", "--session", str(tmp_path / "session.json"), "--sizes", "0.05",
                     "0.25", "--out", str(tmp_path / "sw.csv"), "--repeats", "1", "--warmup", "0"]) == 0
    sw = cli.BenchReport.from_json(json.loads((tmp_path / "sw.json").read_text()))
    assert [r.edit_size for r in sw.runs] == [0.05, 0.25] and all(r.macs_ratio > 1 for r in sw.runs)
    # session / manifest mismatch is a usage error (exit 2)
    (tmp_path / "bad.json").write_text(json.dumps(dict(sess, old_tokens=[1, 2])))
    assert cli.main(["edit", "--session", str(tmp_path / "bad.json"), "--out", str(tmp_path / "x")]) == 2
