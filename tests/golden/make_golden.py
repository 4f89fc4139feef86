"""Generate the golden vectors that pin the CPU oracle (and the CUDA path).

Run in the build container, where the read-only reference package exists:

    python tests/golden/make_golden.py [/root/reference/pkg/src]

It imports the REAL reference `sparsedit` package (never copied into this
repo), runs it on seeded inputs and writes small .npz fixtures next to this
script. The fixtures are committed; nothing at test / bench time reads
/root/reference.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src"
sys.path.insert(0, REF)

import sparsedit as sd  # noqa: E402
from sparsedit import sparse as sp  # noqa: E402
from sparsedit import unet as un  # noqa: E402

OLD = (3, 5, 7, 11)
NEW = (3, 5, 9, 11)
TINY = dict(latent_h=32, latent_w=32, channels=(8, 16), blocks_per_level=1, groups=4, steps=6,
            t1=2, t2=3, text_dim=8, seed=7)
TINY2 = dict(latent_h=32, latent_w=32, channels=(8, 16, 16), blocks_per_level=2, groups=4, steps=4,
             t1=1, t2=2, text_dim=8, seed=5, gate_fraction=0.2)
MEDIUM = dict(latent_h=64, latent_w=64, channels=(8, 16, 32), blocks_per_level=1, groups=4, steps=20,
              t1=5, t2=10, text_dim=16, seed=11)


def r4(g, *s):
    return g.standard_normal(s).astype(np.float32)


def ops_golden():
    g = np.random.Generator(np.random.PCG64(2024))
    out = {}
    # dense conv (tensors.py:97)
    x = r4(g, 1, 5, 9, 11)
    w = (g.standard_normal((6, 5, 3, 3)) / np.sqrt(45)).astype(np.float32)
    b = (0.1 * g.standard_normal(6)).astype(np.float32)
    out.update(conv_x=x, conv_w=w, conv_b=b, conv_y=sd.conv2d(x, sd.ConvWeights(w, b, 1)))
    # group norm (tensors.py:129)
    x = r4(g, 1, 8, 6, 6) * 3 + 1
    gam = (1 + 0.1 * g.standard_normal(8)).astype(np.float32)
    bet = (0.1 * g.standard_normal(8)).astype(np.float32)
    y, m, v = sd.group_norm(x, 4, gam, bet, 1e-5)
    out.update(gn_x=x, gn_gamma=gam, gn_beta=bet, gn_y=y, gn_mean=m, gn_var=v)
    # attention (tensors.py:203)
    q, k, vv = r4(g, 7, 5), r4(g, 9, 5), r4(g, 9, 4)
    out.update(att_q=q, att_k=k, att_v=vv, att_y=sd.attention(q, k, vv, 0.37))
    # sparse conv / gn / attention (sparse.py:184-338)
    x = r4(g, 1, 4, 16, 16)
    w = (g.standard_normal((6, 4, 3, 3)) / 6.0).astype(np.float32)
    b = (0.1 * g.standard_normal(6)).astype(np.float32)
    cached = r4(g, 1, 6, 16, 16)
    mask = sd.BinaryMask(g.random((16, 16)) < 0.2)
    plan = sd.select_gather_plan(mask, (3, 3))
    ctx = sp.SparseLayerContext(step=1, layer_id=0, cached_output=cached)
    out.update(sc_x=x, sc_w=w, sc_b=b, sc_cached=cached, sc_mask=mask.bits,
               sc_y=sd.sparse_conv(x, sd.ConvWeights(w, b, 1), plan, ctx, mask))
    x = r4(g, 1, 8, 16, 16)
    cached = r4(g, 1, 8, 16, 16)
    mean, var = r4(g, 1, 4), (0.5 + g.random((1, 4))).astype(np.float32)
    gam = g.standard_normal(8).astype(np.float32)
    bet = g.standard_normal(8).astype(np.float32)
    ctx = sp.SparseLayerContext(step=1, layer_id=0, cached_output=cached, cached_mean=mean, cached_var=var)
    out.update(sg_x=x, sg_cached=cached, sg_mean=mean, sg_var=var, sg_gamma=gam, sg_beta=bet,
               sg_mask=mask.bits, sg_y=sd.sparse_group_norm(x, ctx, gam, bet, 1e-5, mask))
    s = 1 / np.sqrt(8)
    wq, wk, wv = [(g.standard_normal((8, 8)) * s).astype(np.float32) for _ in range(3)]
    mask3 = sd.BinaryMask(g.random((16, 16)) < 0.3)
    ctx = sp.SparseLayerContext(step=1, layer_id=0, cached_output=cached)
    out.update(sa_x=x, sa_wq=wq, sa_wk=wk, sa_wv=wv, sa_cached=cached, sa_mask=mask3.bits,
               sa_y=sd.sparse_self_attention(x, wq, wk, wv, 0.35, ctx, mask3),
               sa_dense=sp.dense_self_attention(x, wq, wk, wv, 0.35))
    tk, tv = r4(g, 6, 8), r4(g, 6, 8)
    ya = sd.sparse_cross_attention(x, tk, tv, wq, 0.35, ctx, mask3)
    yd, mp = sp.dense_cross_attention(x, tk, tv, wq, 0.35)
    out.update(ca_tk=tk, ca_tv=tv, ca_y=ya, ca_dense=yd, ca_map=mp)
    # accumulate_diff (masks.py:117)
    xs = [r4(g, 1, 4, 16, 16) for _ in range(10)]
    ys = [a + (0.3 * g.standard_normal(a.shape)).astype(np.float32) for a in xs]
    d = sd.accumulate_diff(xs, ys, 3, 8)
    out.update(ad_x=np.stack(xs), ad_y=np.stack(ys), ad_values=d.values, ad_degenerate=d.degenerate)
    # otsu on continuous and coarse maps (masks.py:147)
    maps, eps, obj = [], [], []
    for i in range(12):
        if i % 3 == 0:
            m = g.random((32, 32)).astype(np.float32)
        elif i % 3 == 1:
            m = np.clip(np.concatenate([0.2 + 0.1 * g.random(700), 0.7 + 0.2 * g.random(324)]), 0, 1)
            m = m.astype(np.float32).reshape(32, 32)
        else:
            m = (g.integers(0, 9, (32, 32)) / 8.0).astype(np.float32)
        r = sd.otsu_threshold(sd.DiffMap(m, False))
        maps.append(m); eps.append(r.epsilon); obj.append(r.objective)
    out.update(otsu_maps=np.stack(maps), otsu_eps=np.array(eps), otsu_obj=np.array(obj))
    # dilation / pyramid / plans
    bits = g.random((32, 32)) < 0.03
    out.update(dl_in=bits, dl_r1=sd.dilate(sd.BinaryMask(bits), 1).bits,
               dl_r2=sd.dilate(sd.BinaryMask(bits), 2).bits)
    pyr = sd.build_pyramid(sd.BinaryMask(bits), 4)
    for i, lv in enumerate(pyr.levels):
        out[f"pyr_{i}"] = lv.bits
    plan_masks, plan_cost, plan_blocks, plan_origins = [], [], [], []
    for i in range(8):
        pm = g.random((24, 24)) < (0.02 + 0.1 * i)
        p = sd.select_gather_plan(sd.BinaryMask(pm), (3, 3))
        plan_masks.append(pm); plan_cost.append(p.cost); plan_blocks.append(p.block)
        org = np.full((144, 2), -1, np.int32)
        org[: len(p.origins)] = np.array(p.origins, np.int32).reshape(-1, 2)
        plan_origins.append(org)
    out.update(plan_masks=np.stack(plan_masks), plan_cost=np.array(plan_cost),
               plan_blocks=np.array(plan_blocks), plan_origins=np.stack(plan_origins))
    p10 = sd.select_gather_plan(sd.BinaryMask.full(8, 8), (3, 3), candidates=(10,))
    p5 = sd.select_gather_plan(sd.BinaryMask(plan_masks[3]), (5, 5))
    out.update(plan_c10=np.array([*p10.block, p10.cost, len(p10.origins)]),
               plan_k5=np.array([*p5.block, p5.cost, len(p5.origins)]))
    np.savez_compressed(HERE / "ops.npz", **out)


def pipeline_golden(name, cfgd, rand_mask_seed=None):
    cfg = un.UNetConfig(**cfgd)
    unet = un.UNet(cfg)
    out = {"config_json": np.array(str(cfgd))}
    out["init_latent"] = un.initial_latent(cfg)
    out["embed_old"] = un.embed_tokens(un.PromptTokens(OLD), cfg)
    out["time_bias"] = unet.time_bias
    out["stem_w"] = unet.stem.weights.weight
    out["out_b"] = unet.out_conv.weights.bias
    blk = unet.enc_blocks[0][0]
    out["sa_wq"] = blk["self_attn"].wq
    out["ca_wk_text"] = blk["cross_attn"].wk_text
    out["gn_gamma"] = blk["norm"].gamma

    def gen():
        store = sd.CacheStore(async_transfer=False)
        final = un.generate_dense(un.PromptTokens(OLD), cfg, store)
        return store, final

    store, final = gen()
    out["final_old"] = final
    T = cfg.steps
    for t in (1, T):
        out[f"step_latent_{t}"] = store.get((t, 0, sd.Role.STEP_LATENT))
        for lid in (0, 1, 2, 3, 4, len(unet.layers) - 1):
            out[f"out_{t}_{lid}"] = store.get((t, lid, sd.Role.LAYER_OUTPUT))
        out[f"mean_{t}_2"] = store.get((t, 2, sd.Role.NORM_MEAN))
        out[f"map_{t}_4"] = store.get((t, 4, sd.Role.CROSS_ATTN_MAP))
    store.close()
    masks = {"center10": sd.centered_square_mask(cfg.latent_h, cfg.latent_w, 0.1),
             "full": sd.BinaryMask.full(cfg.latent_h, cfg.latent_w)}
    if rand_mask_seed is not None:
        rg = np.random.Generator(np.random.PCG64(rand_mask_seed))
        masks["rand"] = sd.dilate(sd.BinaryMask(rg.random((cfg.latent_h, cfg.latent_w)) < 0.1 / 9), 1)
    for mname, m in masks.items():
        store, _ = gen()
        session = un.EditSession.create(OLD, NEW, cfg, store, user_mask=m)
        res = un.edit(session, cfg, store)
        out[f"edit_{mname}_mask"] = m.bits
        out[f"edit_{mname}_latent"] = res.latent
        out[f"edit_{mname}_sparse_macs"] = np.array([l.sparse_macs for l in res.macs.layers], np.int64)
        out[f"edit_{mname}_dense_macs"] = np.array([l.dense_macs for l in res.macs.layers], np.int64)
        if res.plans:
            for lv, p in res.plans.items():
                out[f"edit_{mname}_plan{lv}_cost"] = np.array(p.cost)
                out[f"edit_{mname}_plan{lv}_origins"] = np.array(p.origins, np.int32).reshape(-1, 2)
        store.close()
    # detected-mask path
    store, _ = gen()
    session = un.EditSession.create(OLD, NEW, cfg, store)
    res = un.edit(session, cfg, store)
    out["det_no_edit"] = np.array(res.no_edit)
    out["det_mask"] = res.mask.bits if res.mask is not None else np.zeros((1, 1), bool)
    out["det_latent"] = res.latent
    out["det_sparse_macs"] = np.array([l.sparse_macs for l in res.macs.layers], np.int64)
    out["det_phase1"] = np.array(res.phase1_macs)
    store.close()
    store, _ = gen()
    outcome = un.detect_mask(un.EditSession.create(OLD, NEW, cfg, store), cfg, store)
    out["det_epsilon"] = np.array(outcome.epsilon)
    out["det_control_latent"] = outcome.control_latent
    store.close()
    # identical prompts -> no edit
    store, _ = gen()
    res = un.edit(un.EditSession.create(OLD, OLD, cfg, store), cfg, store)
    out["same_no_edit"] = np.array(res.no_edit)
    store.close()
    np.savez_compressed(HERE / f"{name}.npz", **out)


if __name__ == "__main__":
    ops_golden()
    pipeline_golden("tiny", TINY)
    pipeline_golden("tiny2", TINY2)
    pipeline_golden("medium", MEDIUM, rand_mask_seed=3)
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, os.path.getsize(f))
