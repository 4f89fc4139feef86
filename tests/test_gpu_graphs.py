"""GPU tests of the captured step graphs (bf16 mode): concurrent requests on their own namespaces
and streams, and the reuse of an edit's captured step graph by a later edit with the same launch
shapes (bitwise equal to a fresh capture)."""

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA GPU")]

OLD, NEW = (3, 5, 7, 11), (3, 5, 9, 11)


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
    assert np.array_equal(reused.latent, fresh.latent)
