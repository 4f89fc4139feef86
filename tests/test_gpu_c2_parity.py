"""Parity at the BENCHMARKED shapes (BASELINE configs[1], [3], [4]) against the CPU oracle.

C2 = the SD-1.5-shape UNet of the bench (320/640/1280/1280 channels, 2 blocks per level,
32 groups, 64x64x4 latent, 77-token 768-wide text, 50-step schedule), 10% centered-square
user mask. Both sides start from the same seeded weights, prompt and initial latent:

  * the oracle (numpy f64-accumulate restatement of the reference, pinned to the reference's
    golden vectors by tests/test_oracle_golden.py) runs the dense caching steps 1..S of the
    old prompt (DenseOps, recording every role) and then sparse steps 1..S of the new prompt
    (SparseOps over that cache; unet.py:874-883, sparse.py:184-338);
  * the GPU records the old prompt's generation into its HBM arena (generate_dense) and steps
    the edit's sparse plan (EditPlan + the captured step graph, the bench's exact path).

Compared: every layer's cached output / GN stats / cross-attention map of dense steps 1..S
(all 64 layers), the mask's active-pixel lists and gather plans (bit-exact), and the stepped
latent after each sparse step (inside the mask: the fresh rows; outside: the cached
generation, bit-exact against the device's own generation).

Bounds (stated in DESIGN.md §2; measured values are printed with -s):
  fp32 mode: latent max-abs <= 1e-4 per sampled step (the north star's 1e-3 final-latent bound
             over 50 steps with margin); layer outputs max-abs <= 2e-4 * max(1, |ref|max)
  tf32x3 mode (fp32 operands on the tensor cores, 3xTF32): the fp32 bounds; 50-step C2 edit
             within 1e-3 of the fp32 edit (test_c2_bf16_full_edit_vs_fp32)
  bf16 mode: latent max-abs <= 2e-3 per sampled step (50 steps extrapolate linearly to
             <= 5e-2, and test_c2_bf16_full_edit_vs_fp32 checks the full 50-step edit);
             layer outputs relative L2 error <= 3e-2
"""

import numpy as np
import pytest

from conftest import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA GPU")]

C2 = dict(latent_h=64, latent_w=64, latent_channels=4, channels=(320, 640, 1280, 1280), blocks_per_level=2,
          groups=32, steps=50, t1=5, t2=10, gate_fraction=0.25, dilation_radius=1, text_dim=768,
          vocab_size=49408, seed=0)
C4 = dict(C2, latent_h=96, latent_w=96, text_dim=1024)
OLD = tuple(range(1, 78))
NEW = tuple(99 if i == 3 else v for i, v in enumerate(OLD))

FP32_LAT_TOL = 1e-4
FP32_LAYER_TOL = 2e-4
TF32X3_LAYER_TOL = 2e-4  # measured 1.3e-5 (split accumulators undo the tensor core's truncating fp32 adds)
BF16_LAT_TOL = 2e-3
BF16_LAYER_REL = 3e-2
BF16_FINAL_TOL = 5e-2


# ----------------------------------------------------------------------------- oracle side
class OracleRun:
    """Dense caching steps 1..S of `old`, then sparse steps 1..S of `new` per mask."""

    def __init__(self, cfg_d, old, S, net=None):
        from oracle import sparsedit_oracle as O
        self.O, self.cfg_d, self.S = O, cfg_d, S
        self.net = net or O.build_net(cfg_d)
        text = O.embed(old, cfg_d)
        sc = O.step_scale(cfg_d)
        lat = O.init_latent(cfg_d)
        self.cache, self.gen_lat = {}, {}
        for t in range(1, S + 1):
            rec = (lambda lid, role, v, _t=t: self.cache.__setitem__((_t, lid, role), v))
            lat = lat - sc * O.forward(self.net, lat, t, text, O.DenseOps(self.net, rec))
            self.gen_lat[t] = lat

    def sparse(self, new, bits, steps=None):
        O, net = self.O, self.net
        text = O.embed(new, self.cfg_d)
        sc = O.step_scale(self.cfg_d)
        pyr = O.pyramid(bits, len(self.cfg_d["channels"]))
        levels = sorted({L.level for L in net.layers if L.gated})
        plans = {lv: O.gather_plan(pyr[lv]) for lv in levels}
        lat = O.init_latent(self.cfg_d)
        out = {}
        for t in range(1, (steps or self.S) + 1):
            lat = lat - sc * O.forward(net, lat, t, text, O.SparseOps(net, pyr, plans, self.cache, t))
            out[t] = lat
        return out, pyr, plans


@pytest.fixture(scope="module")
def c2_oracle():
    return OracleRun(C2, OLD, 2)


@pytest.fixture(scope="module")
def c2_mask():
    from oracle import sparsedit_oracle as O
    return O.centered_square(64, 64, 0.10)


@pytest.fixture(scope="module")
def c2_sparse(c2_oracle, c2_mask):
    return c2_oracle.sparse(NEW, c2_mask)


@pytest.fixture(scope="module")
def P():
    import paper_2305_17423_b200 as P
    yield P
    P.set_precision("fp32")


# ----------------------------------------------------------------------------- GPU side
def _gpu_sparse_steps(P, cfg, store, new, bits, S):
    """Sparse steps 1..S of `new` over the store's generation through the edit path (EditPlan +
    captured step graph); returns the DevicePlan and the full latent (NCHW) after each step."""
    import torch
    from paper_2305_17423_b200 import unet as U
    from paper_2305_17423_b200.engine import DRef, FeatVal
    arena = store.arena
    eng = arena.eng
    kv = eng.text_kv(P.embed_tokens(P.PromptTokens(new), cfg))
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    ep = U.EditPlan(eng, arena, P.BinaryMask(bits), kv, lat0)
    run = U._Runner(eng, ep.plan, True)
    lats = {}
    for t in range(1, S + 1):
        run.step(t)
        out = torch.empty((eng.hw(0), cfg.latent_channels), dtype=torch.float32, device=eng.dev)
        fv = FeatVal(DRef(ep.lat_rows), 0, cfg.latent_channels, ep.dp.index[0], DRef(arena.latent[t]))
        eng.step_dev.fill_(0)
        eng.materialize(fv, DRef(out))  # the product's select-on-read merge (EditPlan.final_latent)
        torch.cuda.synchronize()
        lats[t] = U._to_nchw(out, cfg.latent_channels, cfg.latent_h, cfg.latent_w)
    return ep, lats


def _layer_err(got, ref, precision):
    d = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    if precision != "bf16":
        return float(d.max() / max(1.0, float(np.abs(ref).max())))
    return float(np.linalg.norm(d) / max(1e-12, float(np.linalg.norm(ref.astype(np.float64)))))


def _check_generation(P, store, orc, S, precision):
    tol = {"bf16": BF16_LAYER_REL, "tf32x3": TF32X3_LAYER_TOL}.get(precision, FP32_LAYER_TOL)
    worst = (0.0, None)
    O = orc.O
    for t in range(1, S + 1):
        for (tt, lid, role), ref in orc.cache.items():
            if tt != t:
                continue
            got = store.get((t, lid, int(role)))
            e = _layer_err(got.reshape(ref.shape), ref, precision)
            worst = max(worst, (e, (t, lid, role)))
        e = _layer_err(store.get((t, 0, P.Role.STEP_LATENT)), orc.gen_lat[t], precision)
        worst = max(worst, (e, (t, 0, O.STEP_LATENT)))
    print(f"[{precision}] generation steps 1..{S}: worst layer error {worst[0]:.3e} at {worst[1]}")
    assert worst[0] <= tol, worst


def _check_plan(P, ep, pyr, plans):
    for lv, plan in plans.items():
        assert np.array_equal(ep.dp.level_bits(lv), pyr[lv]), lv
        rows = ep.dp.rows[lv][: ep.dp.n_active[lv]].cpu().numpy()
        assert np.array_equal(rows, np.flatnonzero(pyr[lv].ravel())), lv  # row-major active list
        assert list(ep.dp.origins(lv)) == [tuple(o) for o in plan["origins"]], lv
        assert 4 * ep.dp.n_tiles[lv] == plan["cost"], lv


def _check_latents(lats, ref, gen_store, bits, precision, P):
    tol = BF16_LAT_TOL if precision == "bf16" else FP32_LAT_TOL
    errs = []
    for t, got in lats.items():
        errs.append(float(np.abs(got - ref[t]).max()))
        # outside the mask the edit holds the device's own cached generation bit-exactly
        own = gen_store.get((t, 0, P.Role.STEP_LATENT))
        assert np.array_equal(got[:, :, ~bits], own[:, :, ~bits]), t
    print(f"[{precision}] sparse-step latent max-abs per step: {[f'{e:.3e}' for e in errs]} (bound {tol})")
    assert max(errs) <= tol, errs
    return errs


# ----------------------------------------------------------------------------- C2
@pytest.mark.parametrize("precision", ["fp32", "tf32x3", "bf16"])
def test_c2_sampled_steps_vs_oracle(P, c2_oracle, c2_sparse, c2_mask, precision):
    """BASELINE configs[1] at its exact shapes: generation cache + sparse steps vs the oracle."""
    P.set_precision(precision)
    cfg = P.UNetConfig(**C2)
    store = P.CacheStore()
    P.generate_dense(P.PromptTokens(OLD), cfg, store, record="full")
    _check_generation(P, store, c2_oracle, c2_oracle.S, precision)
    ref, pyr, plans = c2_sparse
    ep, lats = _gpu_sparse_steps(P, cfg, store, NEW, c2_mask, c2_oracle.S)
    _check_plan(P, ep, pyr, plans)
    assert ep.dp.n_active[:2] == [400, 100]
    _check_latents(lats, ref, store, c2_mask, precision, P)
    store.close()


def test_c2_bf16_full_edit_vs_fp32(P, c2_mask):
    """The whole 50-step C2 edit in bf16 (the bench's precision) and in tf32x3 against the same
    edit in fp32 (which the sampled-step test pins to the oracle at <= 1e-4 per step): final
    latent within each mode's bound, outside-mask latents bit-exact against each mode's own
    generation."""
    cfg = P.UNetConfig(**C2)
    out = {}
    for precision in ("fp32", "tf32x3", "bf16"):
        P.set_precision(precision)
        store = P.CacheStore()
        final = P.generate_dense(P.PromptTokens(OLD), cfg, store, record="engine")
        res = P.edit(P.EditSession.create(OLD, NEW, cfg, store, user_mask=P.BinaryMask(c2_mask)), cfg, store)
        assert np.array_equal(res.latent[:, :, ~c2_mask], final[:, :, ~c2_mask])
        out[precision] = (final, res.latent)
        store.close()
    gen_err = float(np.abs(out["bf16"][0] - out["fp32"][0]).max())
    edit_err = float(np.abs(out["bf16"][1] - out["fp32"][1]).max())
    print(f"C2 50-step bf16 vs fp32: generation {gen_err:.3e}, edit final latent {edit_err:.3e} (bound {BF16_FINAL_TOL})")
    assert edit_err <= BF16_FINAL_TOL and gen_err <= BF16_FINAL_TOL
    # fp32 operands on the tensor cores: the north star's fp32 final-latent bound (1e-3)
    tgen = float(np.abs(out["tf32x3"][0] - out["fp32"][0]).max())
    tedit = float(np.abs(out["tf32x3"][1] - out["fp32"][1]).max())
    print(f"C2 50-step tf32x3 vs fp32: generation {tgen:.3e}, edit final latent {tedit:.3e} (bound 1e-3)")
    assert tedit <= 1e-3 and tgen <= 1e-3


def test_c5_mix_batched_vs_oracle(P):
    """BASELINE configs[4] request mix at C2 shapes: R requests (distinct prompts, own
    generations, 5/10/25% squares at distinct offsets) stepped as ONE stacked bf16 batch;
    each request's first sparse step vs its own oracle run."""
    import torch
    from oracle import sparsedit_oracle as O
    from paper_2305_17423_b200 import unet as U
    P.set_precision("bf16")
    cfg = P.UNetConfig(**C2)
    fracs = (0.05, 0.10, 0.25)
    reqs = []
    for r in range(3):
        old = tuple((i * 7 + r) % 49000 + 1 for i in range(77))
        new = tuple(99 + r if i == 3 else v for i, v in enumerate(old))
        side = int(round((fracs[r] * 64 * 64) ** 0.5))
        y0, x0 = (7 * r + 3) % (64 - side), (13 * r + 1) % (64 - side)
        bits = np.zeros((64, 64), bool)
        bits[y0:y0 + side, x0:x0 + side] = True
        reqs.append((old, new, bits))
    stores = [P.CacheStore() for _ in reqs]
    P.generate_dense_batch([P.PromptTokens(o) for o, _, _ in reqs], cfg, stores)
    eng = U.get_engine(cfg, "bf16")
    stacked = stores[0].arena.stacked
    kvs = [eng.text_kv(P.embed_tokens(P.PromptTokens(n), cfg)) for _, n, _ in reqs]
    lat0 = U._to_nhwc(P.initial_latent(cfg), eng.dev)
    bp = U.BatchedEditPlan(eng, stacked, [P.BinaryMask(b) for _, _, b in reqs], kvs, [lat0] * len(reqs))
    U._Runner(eng, bp.plan, True).step(1)
    torch.cuda.synchronize()
    rows0 = bp.lists[0][0].cpu().numpy()
    lat_rows = bp.lat_rows.cpu().numpy()
    net = O.build_net(C2)
    start, errs = 0, []
    for r, (old, new, bits) in enumerate(reqs):
        orc = OracleRun(C2, old, 1, net=net)
        ref, _, _ = orc.sparse(new, bits)
        n = int(bits.sum())
        pix = rows0[start:start + n] - r * 64 * 64
        assert np.array_equal(pix, np.flatnonzero(bits.ravel()))
        got = lat_rows[start:start + n]  # [n, 4] fresh rows of request r
        want = ref[1][0].reshape(4, -1)[:, pix].T
        errs.append(float(np.abs(got - want).max()))
        start += (n + 15) // 16 * 16
    print(f"C5 mix (R=3, bf16) first sparse step max-abs per request: {[f'{e:.3e}' for e in errs]}")
    assert max(errs) <= BF16_LAT_TOL, errs
    for s in stores:
        s.close()


# ----------------------------------------------------------------------------- C4
def test_c4_sd2_shape_multi_round_vs_oracle(P):
    """BASELINE configs[3]: SD-2 shape (96x96 latent, 1024-wide text), two edit rounds with new
    prompts and masks against ONE HBM-resident generation, first sparse step of each round vs
    the oracle, in fp32 and bf16."""
    from oracle import sparsedit_oracle as O
    orc = OracleRun(C4, OLD, 1)
    rounds = []
    for k, (f, new_tok) in enumerate(((0.10, 99), (0.05, 123))):
        new = tuple(new_tok if i == 3 + k else v for i, v in enumerate(OLD))
        bits = np.roll(O.centered_square(96, 96, f), (5 * k, -7 * k), axis=(0, 1))
        rounds.append((new, bits, orc.sparse(new, bits)))
    cfg = P.UNetConfig(**C4)
    for precision in ("fp32", "bf16"):
        P.set_precision(precision)
        store = P.CacheStore()
        P.generate_dense(P.PromptTokens(OLD), cfg, store, record="full")
        _check_generation(P, store, orc, 1, precision)
        for new, bits, (ref, pyr, plans) in rounds:  # both rounds read the same arena
            ep, lats = _gpu_sparse_steps(P, cfg, store, new, bits, 1)
            _check_plan(P, ep, pyr, plans)
            _check_latents(lats, ref, store, bits, precision, P)
        store.close()
