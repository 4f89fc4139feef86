"""GPU tests of batched requests: R edits stepped as ONE stacked batch (SURVEY §8 C5 shard).

`generate_dense_batch` records R generations into one stacked arena; `edit_batch` steps their
edits together (concatenated rows per level, block-diagonal segment attention, per-image
GroupNorm). Each request's result must equal its own `edit()` within the bf16 bound and the
CPU oracle within the bf16 bound, and keep the cached generation bit-exactly
outside its mask.
"""

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA GPU")]

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


def _square(h, w, y0, x0, side):
    b = np.zeros((h, w), dtype=bool)
    b[y0:y0 + side, x0:x0 + side] = True
    return b


REQS = [((3, 5, 7, 11), (3, 5, 9, 11), (4, 4, 9)),
        ((2, 4, 6), (2, 8, 6), (10, 3, 13)),
        ((1, 2, 3, 4, 5), (1, 2, 7, 4, 5), (0, 17, 6)),
        ((9, 8), (9, 12), (20, 20, 12))]


@pytest.mark.parametrize("kw", [dict(), dict(channels=(64, 128, 128), latent_h=64, latent_w=64, blocks_per_level=2)])
def test_batched_edits_match_individual_edits_and_oracle(P, kw):
    from oracle import sparsedit_oracle as O
    cfg = _cfg(P, **kw)
    H, W = cfg.latent_h, cfg.latent_w
    reqs = [(old, new, P.BinaryMask(_square(H, W, *[v * H // 32 for v in sq]))) for old, new, sq in REQS]
    stores = [P.CacheStore() for _ in reqs]
    finals = P.generate_dense_batch([P.PromptTokens(o) for o, _, _ in reqs], cfg, stores)
    sessions = [P.EditSession.create(o, n, cfg, st, user_mask=m) for (o, n, m), st in zip(reqs, stores)]
    # results come back in session order whatever order they are passed in
    res = P.edit_batch(sessions[::-1], cfg)[::-1]
    net = O.build_net(cfg)
    for (old, new, mask), final, r in zip(reqs, finals, res):
        store = P.CacheStore()
        final1 = P.generate_dense(P.PromptTokens(old), cfg, store, record="engine")
        one = P.edit(P.EditSession.create(old, new, cfg, store, user_mask=mask), cfg, store)
        ref_final, cache = O.generate(cfg, old, net)
        ref = O.edit(cfg, cache, old, new, user_mask=mask.bits, net=net)
        err = {"gen_batch_vs_one": np.abs(final - final1).max(), "gen_vs_oracle": np.abs(final - ref_final).max(),
               "edit_batch_vs_one": np.abs(r.latent - one.latent).max(),
               "edit_vs_oracle": np.abs(r.latent - ref["latent"]).max()}
        assert np.array_equal(final, final1), err  # same generation kernels into a view of the stacked arena
        assert err["edit_batch_vs_one"] <= BF16_FINAL_TOL and err["edit_vs_oracle"] <= BF16_FINAL_TOL, err
        assert np.array_equal(r.latent[:, :, ~mask.bits], final[:, :, ~mask.bits])


def test_batched_detected_masks(P):
    """Detection (controlled steps + Otsu mask) per request, then one batched sparse phase."""
    cfg = _cfg(P)
    pairs = [((3, 5, 7, 11), (3, 5, 9, 11)), ((2, 4, 6), (2, 8, 6))]
    stores = [P.CacheStore() for _ in pairs]
    P.generate_dense_batch([P.PromptTokens(o) for o, _ in pairs], cfg, stores)
    sessions = [P.EditSession.create(o, n, cfg, st) for (o, n), st in zip(pairs, stores)]
    res = P.edit_batch(sessions, cfg)
    for (old, new), r in zip(pairs, res):
        store = P.CacheStore()
        P.generate_dense(P.PromptTokens(old), cfg, store, record="engine")
        one = P.edit(P.EditSession.create(old, new, cfg, store), cfg, store)
        assert (r.mask is None) == (one.mask is None)
        if r.mask is not None:
            assert np.array_equal(r.mask.bits, one.mask.bits)
        assert np.abs(r.latent - one.latent).max() <= BF16_FINAL_TOL


def test_batched_odd_latent_and_repeat_rounds(P):
    """96x96 latent (SD-2 shape, C4; levels 96/48/24: dense-level boxes that TMA cannot tile since
    128 % 48 != 0) and two edit rounds on the same stores (the HBM cache is never compacted)."""
    cfg = _cfg(P, latent_h=96, latent_w=96, channels=(64, 128, 128))
    reqs = [((3, 5, 7, 11), (3, 5, 9, 11), (5, 6, 20)), ((2, 4, 6), (2, 8, 6), (40, 55, 24))]
    stores = [P.CacheStore() for _ in reqs]
    finals = P.generate_dense_batch([P.PromptTokens(o) for o, _, _ in reqs], cfg, stores)
    masks = [P.BinaryMask(_square(96, 96, *sq)) for _, _, sq in reqs]
    for _ in range(2):
        res = P.edit_batch([P.EditSession.create(o, n, cfg, st, user_mask=m)
                            for (o, n, _), st, m in zip(reqs, stores, masks)], cfg)
        for (old, new, _), m, final, r in zip(reqs, masks, finals, res):
            store = P.CacheStore()
            P.generate_dense(P.PromptTokens(old), cfg, store, record="engine")
            one = P.edit(P.EditSession.create(old, new, cfg, store, user_mask=m), cfg, store)
            assert np.abs(r.latent - one.latent).max() <= BF16_FINAL_TOL
            assert np.array_equal(r.latent[:, :, ~m.bits], final[:, :, ~m.bits])


def test_batched_no_edit_request_rides_along(P):
    """A request whose detection finds nothing to edit (same prompt) rides along in the batch with
    an empty mask: its latent is the cached generation's, bit-exactly; the other request equals
    its own edit()."""
    cfg = _cfg(P)
    pairs = [((3, 5, 7, 11), (3, 5, 7, 11)), ((2, 4, 6), (2, 8, 6))]
    stores = [P.CacheStore() for _ in pairs]
    finals = P.generate_dense_batch([P.PromptTokens(o) for o, _ in pairs], cfg, stores)
    res = P.edit_batch([P.EditSession.create(o, n, cfg, st) for (o, n), st in zip(pairs, stores)], cfg)
    assert res[0].no_edit and res[0].mask is None
    assert np.array_equal(res[0].latent, finals[0])
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens(pairs[1][0]), cfg, store, record="engine")
    one = P.edit(P.EditSession.create(pairs[1][0], pairs[1][1], cfg, store), cfg, store)
    assert np.abs(res[1].latent - one.latent).max() <= BF16_FINAL_TOL


def test_edit_batch_rejects_foreign_stores(P):
    cfg = _cfg(P)
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens((3, 5, 7, 11)), cfg, store, record="engine")
    with pytest.raises(P.ContractViolation):
        P.edit_batch([P.EditSession.create((3, 5, 7, 11), (3, 5, 9, 11), cfg, store,
                                           user_mask=P.centered_square_mask(32, 32, 0.1))], cfg)


def test_edit_batch_subset_in_any_order(P):
    """Any subset of one generate_dense_batch, sessions in any order: the missing generations ride
    along with empty masks, each returned result equals its own edit() (bf16 bound) and keeps its
    own generation outside the mask bit-exactly; detected masks read their own generation."""
    cfg = _cfg(P)
    stores = [P.CacheStore() for _ in REQS]
    finals = P.generate_dense_batch([P.PromptTokens(o) for o, _, _ in REQS], cfg, stores)
    pick = [3, 1]  # a subset, out of order
    sessions = []
    for i in pick:
        old, new, (y0, x0, side) = REQS[i]
        sessions.append(P.EditSession.create(old, new, cfg, stores[i], user_mask=P.BinaryMask(_square(32, 32, y0, x0, side))))
    res = P.edit_batch(sessions, cfg)
    assert len(res) == len(pick)
    for r, i in zip(res, pick):
        old, new, (y0, x0, side) = REQS[i]
        m = P.BinaryMask(_square(32, 32, y0, x0, side))
        assert np.array_equal(r.latent[:, :, ~m.bits], finals[i][:, :, ~m.bits])
        store = P.CacheStore()
        P.generate_dense(P.PromptTokens(old), cfg, store, record="engine")
        one = P.edit(P.EditSession.create(old, new, cfg, store, user_mask=m), cfg, store)
        assert np.abs(r.latent - one.latent).max() <= BF16_FINAL_TOL
    # detected masks (no user mask), order reversed
    det = [P.EditSession.create(REQS[i][0], REQS[i][1], cfg, stores[i]) for i in (2, 0)]
    res = P.edit_batch(det, cfg)
    for r, i in zip(res, (2, 0)):
        store = P.CacheStore()
        P.generate_dense(P.PromptTokens(REQS[i][0]), cfg, store, record="engine")
        one = P.edit(P.EditSession.create(REQS[i][0], REQS[i][1], cfg, store), cfg, store)
        assert np.array_equal(r.mask.bits, one.mask.bits)
        assert np.abs(r.latent - one.latent).max() <= BF16_FINAL_TOL
