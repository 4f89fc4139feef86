"""GPU tests of the persistent step VM (csrc/fis_vm.cu) in bf16 mode.

The VM executes a recorded step (gather-GEMMs on tcgen05 / SIMT, softmax, GN, pool) in one
cooperative launch. Checks:
  * bf16 generation and user-mask edits agree with the CPU oracle within the bf16 bound
    (final latent max-abs <= 5e-2) at configs whose channels take the
    tcgen05 path (multiples of 64);
  * VM and per-op CUDA-graph paths agree (same bf16 operands, different split-K order:
    <= 2e-2 on the final latent);
  * outside the mask the edit returns the device's cached generation bit-exactly;
  * VM results are bitwise reproducible run to run (split-K sums in fixed split order).
"""

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA GPU")]

OLD, NEW = (3, 5, 7, 11), (3, 5, 9, 11)
BF16_FINAL_TOL = 5e-2


@pytest.fixture(scope="module")
def P():
    import paper_2305_17423_b200 as P
    P.set_precision("bf16")
    yield P
    P.set_precision("fp32")


def _cfg(P, **kw):
    d = dict(latent_h=32, latent_w=32, channels=(64, 128), blocks_per_level=1, groups=4, steps=4, t1=1, t2=2,
             text_dim=64, seed=5)
    d.update(kw)
    return P.UNetConfig(**d)


def _engine(P, cfg):
    from paper_2305_17423_b200 import unet as U
    return U.get_engine(cfg, "bf16")


def _run(P, cfg, mask, use_vm):
    eng = _engine(P, cfg)
    prev = eng.use_vm
    eng.use_vm = use_vm
    try:
        store = P.CacheStore()
        final = P.generate_dense(P.PromptTokens(OLD), cfg, store, record="engine")
        res = P.edit(P.EditSession.create(OLD, NEW, cfg, store, user_mask=mask), cfg, store)
    finally:
        eng.use_vm = prev
    return final, res


@pytest.mark.parametrize("kw", [dict(), dict(channels=(64, 128, 128), latent_h=64, latent_w=64, blocks_per_level=2)])
def test_vm_bf16_matches_oracle_and_graph_path(P, kw):
    from oracle import sparsedit_oracle as O
    cfg = _cfg(P, **kw)
    mask = P.centered_square_mask(cfg.latent_h, cfg.latent_w, 0.1)
    final_vm, res_vm = _run(P, cfg, mask, True)
    final_g, res_g = _run(P, cfg, mask, False)
    net = O.build_net(cfg)
    ref_final, cache = O.generate(cfg, OLD, net)
    ref = O.edit(cfg, cache, OLD, NEW, user_mask=mask.bits, net=net)
    err = {"gen_vm": np.abs(final_vm - ref_final).max(), "gen_graph": np.abs(final_g - ref_final).max(),
           "edit_vm": np.abs(res_vm.latent - ref["latent"]).max(),
           "edit_graph": np.abs(res_g.latent - ref["latent"]).max(),
           "gen_vm_vs_graph": np.abs(final_vm - final_g).max(),
           "edit_vm_vs_graph": np.abs(res_vm.latent - res_g.latent).max()}
    assert err["gen_vm"] <= BF16_FINAL_TOL and err["edit_vm"] <= BF16_FINAL_TOL, err
    assert err["gen_vm_vs_graph"] <= 2e-2 and err["edit_vm_vs_graph"] <= 2e-2, err
    bits = mask.bits
    assert np.array_equal(res_vm.latent[:, :, ~bits], final_vm[:, :, ~bits])


def test_vm_bitwise_reproducible(P):
    cfg = _cfg(P)
    mask = P.centered_square_mask(32, 32, 0.25)
    f1, r1 = _run(P, cfg, mask, True)
    f2, r2 = _run(P, cfg, mask, True)
    assert np.array_equal(f1, f2) and np.array_equal(r1.latent, r2.latent)


def test_vm_sd_shape_step_matches_graph_path(P):
    """One sparse step at SD-1.5 widths (C2 shapes, 2-step schedule): VM vs per-op graph path."""
    import torch
    from paper_2305_17423_b200 import unet as U
    cfg = P.UNetConfig(latent_h=64, latent_w=64, latent_channels=4, channels=(320, 640, 1280, 1280),
                       blocks_per_level=2, groups=32, steps=2, t1=1, t2=1, text_dim=768, vocab_size=49408, seed=0)
    eng = U.get_engine(cfg, "bf16")
    store = P.CacheStore()
    old = tuple(range(1, 78))
    new = tuple(99 if i == 3 else v for i, v in enumerate(old))
    P.generate_dense(P.PromptTokens(old), cfg, store, record="engine")
    mask = P.centered_square_mask(64, 64, 0.1)
    kv = eng.text_kv(P.embed_tokens(P.PromptTokens(new), cfg))
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    outs = []
    for use_vm in (True, False):
        eng.use_vm = use_vm
        ep = U.EditPlan(eng, store.arena, mask, kv, lat0)
        r = U._Runner(eng, ep.plan, True)
        r.step(1)
        r.step(2)
        torch.cuda.synchronize()
        outs.append(ep.plan.lat_rows.clone())
    eng.use_vm = False
    assert torch.isfinite(outs[0]).all()
    assert (outs[0] - outs[1]).abs().max().item() <= 5e-2


def test_concurrent_requests_match_sequential(P):
    """Two edit requests stepped concurrently (own namespace + CUDA stream each, bench C5 shard) give
    bitwise the same latents as stepping them one after the other."""
    import torch
    from paper_2305_17423_b200 import unet as U
    cfg = _cfg(P)
    eng = _engine(P, cfg)
    masks = [P.centered_square_mask(32, 32, 0.1), P.centered_square_mask(32, 32, 0.3)]
    plans = []
    for r, mask in enumerate(masks):
        store = P.CacheStore()
        eng.ns = 0
        P.generate_dense(P.PromptTokens(OLD), cfg, store, record="engine")
        kv = eng.text_kv(P.embed_tokens(P.PromptTokens(NEW), cfg))
        lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
        plans.append((store, kv, lat0, mask))

    def run(concurrent):
        runners, eps = [], []
        for r, (store, kv, lat0, mask) in enumerate(plans):
            ep = U.EditPlan(eng, store.arena, mask, kv, lat0)
            runners.append(U._Runner(eng, ep.plan, True, ns=10 + r + (2 if concurrent else 0)))
            eps.append(ep)
        streams = [torch.cuda.Stream() for _ in runners]
        for t in range(1, cfg.steps + 1):
            for run_, st in zip(runners, streams):
                if concurrent:
                    with torch.cuda.stream(st):
                        run_.step(t)
                else:
                    run_.step(t)
                    torch.cuda.synchronize()
        torch.cuda.synchronize()
        eng.ns = 0
        return [ep.plan.lat_rows.clone() for ep in eps]

    seq, conc = run(False), run(True)
    for a, b in zip(seq, conc):
        assert torch.equal(a, b)


def test_edit_graph_reuse_matches_fresh_capture(P):
    """A second edit on the same cached generation with the same active-row counts per level reuses
    the first edit's captured step graph (new lists / latent rows / text K/V copied in); it must
    give bitwise the same latent as a freshly captured graph."""
    from paper_2305_17423_b200 import unet as U
    cfg = _cfg(P)
    eng = _engine(P, cfg)
    vm = eng.use_vm
    eng.use_vm = False  # graph reuse is a property of the per-op CUDA-graph path
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens(OLD), cfg, store, record="engine")
    b1 = np.zeros((32, 32), bool)
    b1[4:12, 6:14] = True
    b2 = np.zeros((32, 32), bool)
    b2[16:24, 18:26] = True  # same 8x8 size -> same counts per level
    graphs = store.graph_cache()  # captured edit graphs are owned by the store of the generation
    graphs.clear()
    P.edit(P.EditSession.create(OLD, NEW, cfg, store, user_mask=P.BinaryMask(b1)), cfg, store)
    reused = P.edit(P.EditSession.create(OLD, (3, 5, 13, 11), cfg, store, user_mask=P.BinaryMask(b2)), cfg, store)
    assert len(graphs) == 1  # the second edit hit the first one's graph
    graphs.clear()
    fresh = P.edit(P.EditSession.create(OLD, (3, 5, 13, 11), cfg, store, user_mask=P.BinaryMask(b2)), cfg, store)
    eng.use_vm = vm
    assert np.array_equal(reused.latent, fresh.latent)
