"""The reference's per-layer execution-mode protocol on the GPU (test_unet.py:138-225 strategy):
UNet.forward with DenseMode / ControlledMode / SparseMode over the HBM store."""

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA GPU")]

OLD, NEW = (3, 5, 7, 11), (3, 5, 9, 11)


@pytest.fixture(scope="module")
def setup():
    import paper_2305_17423_b200 as P
    from paper_2305_17423_b200 import unet as U
    P.set_precision("fp32")
    cfg = P.UNetConfig(latent_h=32, latent_w=32, channels=(8, 16), blocks_per_level=1, groups=4, steps=6,
                       t1=2, t2=3, text_dim=8, seed=7)
    store = P.CacheStore()
    final = P.generate_dense(P.PromptTokens(OLD), cfg, store)
    return P, U, cfg, store, final


def _sparse_mode(P, U, cfg, store, t, mask, macs=None):
    unet = P.UNet(cfg)
    pyr = P.build_pyramid(mask, cfg.levels)
    plans = {lv: P.select_gather_plan(pyr.levels[lv], (3, 3)) for lv in sorted({i.level for i in unet.layers if i.gated})}
    return unet, U.SparseMode(cfg, pyr, plans, U._sparse_contexts(unet, store, t), macs=macs)


def test_dense_forward_matches_engine_step(setup):
    P, U, cfg, store, final = setup
    t = cfg.steps
    prev = store.get((t - 1, 0, P.Role.STEP_LATENT))
    text = P.embed_tokens(P.PromptTokens(OLD), cfg)
    unet = P.UNet(cfg)
    delta = unet.forward(prev, t, text, U.DenseMode(cfg.groups))
    stepped = prev - U._step_scale(cfg) * delta
    assert np.abs(stepped - store.get((t, 0, P.Role.STEP_LATENT))).max() <= 1e-5
    assert np.abs(delta - store.get((t, unet.topo["out"], P.Role.LAYER_OUTPUT))).max() <= 1e-4


def test_sparse_full_mask_matches_dense(setup):
    P, U, cfg, store, final = setup
    t = cfg.steps
    prev = store.get((t - 1, 0, P.Role.STEP_LATENT))
    text = P.embed_tokens(P.PromptTokens(OLD), cfg)
    unet, mode = _sparse_mode(P, U, cfg, store, t, P.BinaryMask.full(32, 32))
    sparse = unet.forward(prev, t, text, mode)
    dense = unet.forward(prev, t, text, U.DenseMode(cfg.groups))
    assert np.abs(sparse - dense).max() <= 1e-4


def test_sparse_empty_mask_replays_cached_step(setup):
    P, U, cfg, store, final = setup
    t = cfg.steps
    prev = store.get((t - 1, 0, P.Role.STEP_LATENT))
    text = P.embed_tokens(P.PromptTokens(OLD), cfg)
    unet, mode = _sparse_mode(P, U, cfg, store, t, P.BinaryMask.empty(32, 32))
    stepped = prev - U._step_scale(cfg) * unet.forward(prev, t, text, mode)
    assert np.abs(stepped - store.get((t, 0, P.Role.STEP_LATENT))).max() <= 1e-6


def test_sparse_macs_smaller_than_dense(setup):
    P, U, cfg, store, final = setup
    t = cfg.steps
    prev = store.get((t - 1, 0, P.Role.STEP_LATENT))
    text = P.embed_tokens(P.PromptTokens(NEW), cfg)
    macs = U._ModeMacsCounter()
    unet, mode = _sparse_mode(P, U, cfg, store, t, P.centered_square_mask(32, 32, 0.05), macs=macs)
    unet.forward(prev, t, text, mode)
    assert 0 < macs.total < sum(unet.dense_step_macs(len(NEW)).values()) / 4


def test_controlled_identical_prompts_replay(setup):
    P, U, cfg, store, final = setup
    unet = P.UNet(cfg)
    text = P.embed_tokens(P.PromptTokens(OLD), cfg)
    shared = P.SharedTokenMap.from_ids(OLD, OLD)
    lat = P.initial_latent(cfg)
    for t in range(1, cfg.steps + 1):
        maps = {lid: store.get((t, lid, P.Role.CROSS_ATTN_MAP)) for lid in unet.cross_layers}
        lat = lat - U._step_scale(cfg) * unet.forward(lat, t, text, U.ControlledMode(cfg, maps, shared, len(OLD)))
        assert np.abs(lat - store.get((t, 0, P.Role.STEP_LATENT))).max() <= 1e-5


def test_controlled_changed_prompt_diverges(setup):
    P, U, cfg, store, final = setup
    unet = P.UNet(cfg)
    text = P.embed_tokens(P.PromptTokens(NEW), cfg)
    maps = {lid: store.get((1, lid, P.Role.CROSS_ATTN_MAP)) for lid in unet.cross_layers}
    lat = P.initial_latent(cfg)
    ctrl = unet.forward(lat, 1, text, U.ControlledMode(cfg, maps, P.SharedTokenMap.from_ids(OLD, NEW), len(NEW)))
    dense = unet.forward(lat, 1, text, U.DenseMode(cfg.groups))
    assert not np.array_equal(ctrl, dense)
    # and it matches the CPU oracle's controlled step
    from oracle import sparsedit_oracle as O
    net = O.build_net(cfg)
    omaps = {lid: maps[lid] for lid in unet.cross_layers}
    want = O.forward(net, lat, 1, text, O.ControlledOps(net, omaps, O.lcs_pairs(OLD, NEW), len(NEW)))
    assert np.abs(ctrl - want).max() <= 1e-4
