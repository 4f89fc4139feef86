"""Model + pipeline API (reference unet.py:1-899) over the B200 engine.

Entry points keep the reference names and signatures:
  generate_dense(prompt, config, store=None)       unet.py:680
  detect_mask(session, config, store)              unet.py:709
  edit(session, config, store) -> EditResult       unet.py:823
plus UNetConfig, PromptTokens, SharedTokenMap, EditSession, UNet, initial_latent,
embed_tokens. All compute runs in libfisedit kernels on the GPU; inputs and
outputs at this boundary are float32 NCHW numpy arrays as in the reference.

Precision: `set_precision("fp32")` (default; fp32 operands, fp32 accumulate on SIMT FFMA —
the parity mode), `set_precision("tf32x3")` (fp32 operands on the tcgen05 tensor cores as a
3xTF32 split, fp32 accumulate) or `set_precision("bf16")` (bf16 operands/activations on the
tcgen05 tensor cores, fp32 accumulate, fp32 softmax/GN/latent — the perf mode).
"""

from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass, field

import os
import numpy as np
import torch

from . import _lib as L
from .cache import CacheStore, Role
from .engine import Arena, BatchedSparsePlan, DRef, Engine, FeatVal, SparsePlan, StepPlan, _pad, halo_lists, slab
from .errors import CacheMissError, ConfigError, ContractViolation
from .masks import BinaryMask, DevicePlan, run_detect
from .model import (LayerInfo, UNetConfig, build_registry, embed_ids, initial_latent_np, lcs_pairs,
                    require_tensor4, step_scale)
from .sparse import GatherPlan
from .tensors import LayerMacs, MacsReport, macs_attention, macs_linear

_PRECISION = "fp32"
_ENGINES: dict = {}


def set_precision(p: str) -> None:
    global _PRECISION
    from .engine import PRECISIONS
    if p not in PRECISIONS:
        raise ConfigError(f"precision must be one of {PRECISIONS}, got {p!r}")
    _PRECISION = p


def get_precision() -> str:
    return _PRECISION


def get_engine(config: UNetConfig, precision: str | None = None) -> Engine:
    p = precision or _PRECISION
    key = (config.key(), p, torch.cuda.current_device() if torch.cuda.is_available() else -1)
    eng = _ENGINES.get(key)
    if eng is None:
        eng = Engine(config, p)
        _ENGINES[key] = eng
    return eng


# ---------------------------------------------------------------------------
# prompts and sessions (unet.py:141-244)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class PromptTokens:
    ids: tuple

    def __post_init__(self):
        object.__setattr__(self, "ids", tuple(int(i) for i in self.ids))
        if not self.ids:
            raise ConfigError("prompt must contain at least one token")


def embed_tokens(tokens: PromptTokens, config: UNetConfig) -> np.ndarray:
    return embed_ids(tokens.ids, config)


@dataclass(frozen=True)
class SharedTokenMap:
    pairs: tuple

    def __post_init__(self):
        prev = (-1, -1)
        for p in self.pairs:
            if not (p[0] > prev[0] and p[1] > prev[1]):
                raise ContractViolation(f"shared pairs must be strictly increasing, got {self.pairs}")
            prev = p

    @classmethod
    def from_ids(cls, old_ids, new_ids) -> "SharedTokenMap":
        return cls(lcs_pairs(tuple(old_ids), tuple(new_ids)))


@dataclass
class EditSession:
    old_tokens: PromptTokens
    new_tokens: PromptTokens
    shared: SharedTokenMap
    t1: int
    t2: int
    store: CacheStore
    user_mask: BinaryMask | None = None
    schedule: tuple = ()
    mask: BinaryMask | None = None

    @classmethod
    def create(cls, old_ids, new_ids, config: UNetConfig, store: CacheStore, user_mask=None, t1=None, t2=None):
        t1 = config.t1 if t1 is None else t1
        t2 = config.t2 if t2 is None else t2
        if not (1 <= t1 <= t2 <= config.steps):
            raise ConfigError(f"need 1 <= t1 <= t2 <= steps, got t1={t1} t2={t2} steps={config.steps}")
        if user_mask is None and t2 > 10:
            raise ConfigError(f"detection window ends at step 10 at the latest, got t2={t2}")
        if user_mask is not None and user_mask.shape != (config.latent_h, config.latent_w):
            raise ConfigError(f"user mask shape {user_mask.shape} != latent {(config.latent_h, config.latent_w)}")
        old, new = PromptTokens(tuple(old_ids)), PromptTokens(tuple(new_ids))
        return cls(old, new, SharedTokenMap.from_ids(old.ids, new.ids), t1, t2, store, user_mask,
                   tuple(range(1, config.steps + 1)))


# ---------------------------------------------------------------------------
# UNet (layer registry + MAC accounting; unet.py:305-426)
# ---------------------------------------------------------------------------

class UNet:
    """Layer registry with stable ids (cache keys) and analytic MACs; weights live on the engine."""

    def __init__(self, config: UNetConfig):
        self.config = config
        hl, topo = build_registry(config, with_params=False)
        self.layers: list[LayerInfo] = [h.info for h in hl]
        self._cin = {h.info.layer_id: h.c_in for h in hl}
        self.topo = topo
        self.cross_layers = [i.layer_id for i in self.layers if i.kind == "cross_attn"]
        self._by_id = {i.layer_id: i for i in self.layers}

    def info(self, layer_id: int) -> LayerInfo:
        return self._by_id[layer_id]

    # -- per-layer objects with the reference attributes (built lazily: seeded host params) --
    def layer_objects(self) -> dict:
        if getattr(self, "_objs", None) is None:
            from .modes import make_layers
            hl, topo = build_registry(self.config, with_params=True)
            self._objs = make_layers(hl)
            self._time_bias = topo["time_bias"]
        return self._objs

    @property
    def time_bias(self):
        self.layer_objects()
        return self._time_bias

    @property
    def stem(self):
        return self.layer_objects()[self.topo["stem"]]

    @property
    def out_conv(self):
        return self.layer_objects()[self.topo["out"]]

    @property
    def down(self):
        return [self.layer_objects()[i] for i in self.topo["down"]]

    @property
    def fuse(self):
        return {l: self.layer_objects()[i] for l, i in self.topo["fuse"].items()}

    @property
    def enc_blocks(self):
        o = self.layer_objects()
        return [[{k: o[v] for k, v in b.items()} for b in lv] for lv in self.topo["enc"]]

    @property
    def dec_blocks(self):
        o = self.layer_objects()
        return {l: [{k: o[v] for k, v in b.items()} for b in lv] for l, lv in self.topo["dec"].items()}

    def forward(self, latent, t, text_emb, mode):
        """One denoiser evaluation through the reference mode protocol (unet.py:430-458)."""
        from .modes import forward
        return forward(self, latent, t, text_emb, mode)

    def conv_cin(self, lid):
        return self._cin[lid]

    def layer_macs(self, info: LayerInfo, px: int, n_text: int) -> int:
        c = info.channels
        if info.kind == "conv":
            return px * c * self._cin[info.layer_id] * 9
        if info.kind == "norm":
            return 0
        if info.kind == "self_attn":
            return 3 * macs_linear(px, c, c) + macs_attention(px, px, c)
        return macs_linear(px, c, c) + 2 * macs_linear(n_text, self.config.text_dim, c) + macs_attention(px, n_text, c)

    def dense_step_macs(self, n_text: int) -> dict:
        return {i.layer_id: self.layer_macs(i, i.h * i.w, n_text) for i in self.layers}

    def sparse_step_macs(self, n_text, active, tile_cost) -> dict:
        """Per-layer MACs of one SparseMode step (unet.py:604-663): gated convs count plan.cost,
        gated attention the active-pixel count, ungated layers are dense."""
        out = {}
        for i in self.layers:
            if not i.gated:
                out[i.layer_id] = self.layer_macs(i, i.h * i.w, n_text)
            elif i.kind == "conv":
                out[i.layer_id] = self.layer_macs(i, tile_cost[i.level], n_text)
            else:
                out[i.layer_id] = self.layer_macs(i, active[i.level], n_text)
        return out


def initial_latent(config: UNetConfig) -> np.ndarray:
    return initial_latent_np(config)


def _initial_latent_dev(eng: Engine) -> torch.Tensor:
    """The seeded initial latent (NHWC rows) on the engine's device, generated once per engine
    (a constant of the config's seed; read-only for its users)."""
    t = getattr(eng, "_lat_init", None)
    if t is None:
        t = eng._lat_init = _to_nhwc(initial_latent_np(eng.config), eng.dev)
    return t


_UNETS: dict = {}


def _unet_of(config: UNetConfig) -> "UNet":
    """The layer registry / MAC model of a config (immutable metadata), built once per config."""
    u = _UNETS.get(config.key())
    if u is None:
        u = _UNETS[config.key()] = UNet(config)
    return u


def _to_nhwc(a: np.ndarray, dev) -> torch.Tensor:
    n, c, h, w = a.shape
    return torch.from_numpy(np.ascontiguousarray(a[0].reshape(c, h * w).T)).to(dev)


def _to_nchw(t: torch.Tensor, c, h, w) -> np.ndarray:
    return t.float().reshape(h, w, c).permute(2, 0, 1).reshape(1, c, h, w).contiguous().cpu().numpy()


# ---------------------------------------------------------------------------
# pipeline
# ---------------------------------------------------------------------------

class _Runner:
    """Drives Engine steps for t in a range: eagerly or through one captured CUDA graph."""

    def __init__(self, eng: Engine, plan, use_graph: bool, ns: int = 0):
        self.eng, self.plan, self.use_graph, self.ns = eng, plan, use_graph, ns
        self.graph = None
        self.launches_per_step = None

    def step(self, t: int):
        """One step on the current CUDA stream (each concurrently driven request owns a namespace
        `ns` of scratch buffers and step counter, and its own stream)."""
        eng = self.eng
        eng.ns = self.ns
        eng.step_dev.fill_(t)
        if not self.use_graph:
            eng.run_step(self.plan)
            return
        if self.graph is None:
            # warm (allocates scratch), then capture one step; replays read t from step_dev
            n0 = eng.launches
            eng.run_step(self.plan)
            self.launches_per_step = eng.launches - n0
            torch.cuda.synchronize()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            import gc
            gc_on = gc.isenabled()
            gc.disable()  # a collection inside the capture could destroy other graphs (invalidating it)
            try:
                # capture_begin / capture_end directly: torch.cuda.graph() empties the caching
                # allocator before every capture (cudaFree of every cached block: up to ~0.5 s
                # with a large arena resident, measured in edit_batch)
                with torch.cuda.stream(s):
                    g.capture_begin()
                    try:
                        eng.run_step(self.plan)
                    finally:
                        g.capture_end()
            finally:
                if gc_on:
                    gc.enable()
            torch.cuda.current_stream().wait_stream(s)
            self.graph = g
            return
        self.graph.replay()

    def run(self, t0, t1):
        for t in range(t0, t1 + 1):
            self.step(t)


def _use_graphs():
    return True


def generate_dense(prompt: PromptTokens, config: UNetConfig, store: CacheStore | None = None, *,
                   record: str = "full", precision: str | None = None, _arena: Arena | None = None) -> np.ndarray:
    """Dense generation; records the generation into an HBM arena bound to `store` (unet.py:680-696).

    record="full" keeps every reference role (LAYER_OUTPUT, NORM stats, maps, latents);
    record="engine" keeps only what edits read (features, gated stats, maps, latents).
    """
    eng = get_engine(config, precision)
    text = embed_tokens(prompt, config)
    kv = eng.text_kv(text)
    T = config.steps
    hw = eng.hw(0)
    if _arena is not None:  # a view of a stacked arena (generate_dense_batch)
        arena = _arena
        latents = arena.latent
    elif store is not None:
        arena = Arena(eng, text.shape[0], full=(record == "full"))
        latents = arena.latent
    else:
        arena = None
        latents = torch.empty((T + 1, hw, config.latent_channels), dtype=torch.float32, device=eng.dev)
    latents[0].copy_(_to_nhwc(initial_latent_np(config), eng.dev))
    _Runner(eng, StepPlan(eng, kv, latents, arena), _use_graphs()).run(1, T)
    if store is not None:
        arena.prompt = tuple(prompt.ids)
        store._bind(eng, arena)
    return _to_nchw(latents[T], config.latent_channels, config.latent_h, config.latent_w)


@dataclass
class _MacsCounter:
    per_layer: dict = field(default_factory=lambda: defaultdict(int))

    def add(self, layer_id, macs):
        self.per_layer[layer_id] += macs

    @property
    def total(self):
        return sum(self.per_layer.values())


@dataclass
class DetectOutcome:
    no_edit: bool
    mask: BinaryMask | None
    epsilon: float
    control_latent: np.ndarray | None
    phase1_macs: _MacsCounter
    from_user_mask: bool = False
    _control_dev: object = None
    diff: object = None


def _arena_of(store: CacheStore, config: UNetConfig, t_first: int):
    a = store.arena if store is not None else None
    if a is None:
        unet = UNet(config)
        lid = next(i.layer_id for i in unet.layers if i.gated)
        raise CacheMissError(t_first, lid, "layer_output")
    if a.eng.config.key() != config.key():
        # the kernels would read the recorded slabs with another model's shapes (reference:
        # ContractViolation / CacheMissError on a cached-shape mismatch, sparse.py:174-181)
        raise ContractViolation(f"store holds a generation of a different UNetConfig "
                                f"({a.eng.config.key()} != {config.key()})")
    return a


def detect_mask(session: EditSession, config: UNetConfig, store: CacheStore) -> DetectOutcome:
    """Controlled steps 1..t2 on device, then the fused diff/Otsu/dilate kernel (unet.py:709-752)."""
    macs = _MacsCounter()
    if session.user_mask is not None:
        return DetectOutcome(session.user_mask.is_empty(), session.user_mask, 0.0, None, macs, True)
    arena = _arena_of(store, config, 1)
    eng = get_engine(config, arena.eng.precision)
    text = embed_tokens(session.new_tokens, config)
    n_new = text.shape[0]
    kv = eng.text_kv(text)
    pairs = session.shared.pairs
    verbatim = len(pairs) == n_new and n_new == arena.n_text
    po = torch.tensor([p[0] for p in pairs] or [0], dtype=torch.int32, device=eng.dev)
    pn = torch.tensor([p[1] for p in pairs] or [0], dtype=torch.int32, device=eng.dev)
    pairs_dev = (po[: len(pairs)], pn[: len(pairs)])
    t2 = session.t2
    hw, cl = eng.hw(0), config.latent_channels
    ys = torch.empty((t2 + 1, hw, cl), dtype=torch.float32, device=eng.dev)
    ys[0].copy_(_to_nhwc(initial_latent_np(config), eng.dev))
    plan = StepPlan(eng, kv, ys, None, ctrl=(arena, verbatim, pairs_dev))
    _Runner(eng, plan, _use_graphs()).run(1, t2)
    unet = UNet(config)
    dense = unet.dense_step_macs(n_new)
    for lid, m in dense.items():
        macs.add(lid, m * t2)
    xr = L.Ref(arena.latent[1].data_ptr(), arena.latent.stride(0) * 4, cl, L.F32)
    yr = L.Ref(ys[1].data_ptr(), ys.stride(0) * 4, cl, L.F32)
    out = run_detect(config.latent_h, config.latent_w, cl, session.t1, t2, config.dilation_radius, xr, yr)
    res = out["result"].cpu().tolist()
    no_edit = bool(out["flags"][0].item())
    control = ys[t2]
    ctrl_np = _to_nchw(control, cl, config.latent_h, config.latent_w)
    if no_edit:
        return DetectOutcome(True, None, float(res[0]), ctrl_np, macs, False, control)
    mask = BinaryMask(out["mask"].cpu().numpy().astype(bool).reshape(config.latent_h, config.latent_w))
    return DetectOutcome(False, mask, float(res[0]), ctrl_np, macs, False, control)


@dataclass
class EditResult:
    latent: np.ndarray
    macs: MacsReport
    cache_stats: object
    mask: BinaryMask | None
    no_edit: bool
    phase1_macs: int
    phase2_macs: int
    plans: dict = field(default_factory=dict)


def _build_report(unet: UNet, n_text, config, counters):
    dense = unet.dense_step_macs(n_text)
    tot = defaultdict(int)
    for c in counters:
        for lid, m in c.per_layer.items():
            tot[lid] += m
    return MacsReport([LayerMacs(i.layer_id, i.kind, dense[i.layer_id] * config.steps, tot.get(i.layer_id, 0))
                       for i in unet.layers])


class EditPlan:
    """Device-side plan of one edit: mask pyramid lists + the sparse step plan."""

    def __init__(self, eng: Engine, arena: Arena, mask: BinaryMask, kv, lat0_full: torch.Tensor):
        cfg = eng.config
        self.dp = DevicePlan(torch.from_numpy(mask.bits.astype(np.uint8).ravel()).to(eng.dev),
                             cfg.latent_h, cfg.latent_w, cfg.levels)
        lists = {l: (self.dp.rows[l], self.dp.index[l], self.dp.n_active[l]) for l in range(cfg.levels)}
        n0 = self.dp.n_active[0]
        rows0 = self.dp.rows[0][:n0].long()
        self.lat_rows = lat0_full.index_select(0, rows0).contiguous()
        self.plan = SparsePlan(eng, kv, arena, lists, self.lat_rows)

    def final_latent(self, eng: Engine, arena: Arena) -> torch.Tensor:
        cfg = eng.config
        out = torch.empty((eng.hw(0), cfg.latent_channels), dtype=torch.float32, device=eng.dev)
        fv = FeatVal(DRef(self.lat_rows), 0, cfg.latent_channels, self.dp.index[0], DRef(arena.latent[cfg.steps]))
        eng.step_dev.fill_(0)
        eng.materialize(fv, DRef(out))
        return out


_GRAPH_CACHE_SIZE = 4  # captured edit-step graphs kept per cached generation (CacheStore.graph_cache)


def _cached_runner(eng: Engine, store: CacheStore, start: int, ep: "EditPlan", kv):
    """Step runner of an edit, reusing a captured step graph when an earlier edit on the same
    cached generation had the same active-row counts per level (same launch shapes): the new
    edit's row lists, pixel->row maps, start latent rows and text K/V are copied (device to
    device) into the buffers that graph reads, instead of capturing a new one. The graphs are
    owned by the store (CacheStore.graph_cache: freed with it, or by close())."""
    if not _use_graphs():
        return _Runner(eng, ep.plan, _use_graphs())
    graphs = store.graph_cache()
    n_text = next(iter(kv.values()))[0].shape[0]
    gated = tuple(n for l, n in enumerate(ep.dp.n_active) if eng.gated[l])  # only gated levels shape launches
    key = (id(eng), start, gated, n_text)
    hit = graphs.get(key)
    if hit is None:
        runner = _Runner(eng, ep.plan, True)
        graphs[key] = (runner, ep, kv)
        if len(graphs) > _GRAPH_CACHE_SIZE:
            graphs.popitem(last=False)
        return runner
    runner, ep0, kv0 = hit
    graphs.move_to_end(key)
    for l in range(len(ep.dp.rows)):
        ep0.dp.rows[l].copy_(ep.dp.rows[l])
        ep0.dp.index[l].copy_(ep.dp.index[l])
    ep0.lat_rows.copy_(ep.lat_rows)
    for lid, tens in kv.items():
        for dst, src in zip(kv0[lid], tens):
            if dst is not None:
                dst.copy_(src)
    # the caller keeps using `ep` for results: point it at the buffers the graph updates
    ep.lat_rows = ep0.lat_rows
    ep.dp.index = ep0.dp.index
    return runner


def edit(session: EditSession, config: UNetConfig, store: CacheStore) -> EditResult:
    """Incremental regeneration for the edited prompt (unet.py:823-899) on the B200 engine."""
    unet = _unet_of(config)
    n_new = len(session.new_tokens.ids)
    outcome = detect_mask(session, config, store)
    session.mask = outcome.mask
    phase2 = _MacsCounter()
    cl, H, W, T = config.latent_channels, config.latent_h, config.latent_w, config.steps
    if outcome.no_edit:
        arena = _arena_of(store, config, T)
        latent = _to_nchw(arena.latent[T], cl, H, W)
        rep = _build_report(unet, n_new, config, [outcome.phase1_macs])
        return EditResult(latent, rep, store.stats(), outcome.mask, True, outcome.phase1_macs.total, 0)
    mask = outcome.mask
    start = 1 if outcome.from_user_mask else session.t2 + 1
    arena = _arena_of(store, config, start)
    eng = get_engine(config, arena.eng.precision)
    kv = eng.text_kv(embed_tokens(session.new_tokens, config))
    if outcome.from_user_mask:
        lat0 = _initial_latent_dev(eng)
    else:
        m = torch.from_numpy(mask.bits.ravel().copy()).to(eng.dev)[:, None]
        lat0 = torch.where(m, outcome._control_dev, arena.latent[session.t2])
    plans = {}
    # the host-side accounting (MACs, gather plans -- its tile read-back is a device sync) runs
    # before the steps are queued or while they execute, so only the final latent copy waits on them
    if mask.all_active():
        _add_dense_macs(phase2, unet, n_new, T - start + 1)
        rep = _build_report(unet, n_new, config, [outcome.phase1_macs, phase2])
        final = _dense_edit(eng, kv, lat0, start)
    else:
        ep = EditPlan(eng, arena, mask, kv, lat0)
        _add_sparse_macs(phase2, unet, n_new, ep.dp, T - start + 1)
        plans = _gather_plans(unet, ep.dp)
        rep = _build_report(unet, n_new, config, [outcome.phase1_macs, phase2])
        _cached_runner(eng, store, start, ep, kv).run(start, T)
        final = ep.final_latent(eng, arena)
    latent = _to_nchw(final, cl, H, W)
    return EditResult(latent, rep, store.stats(), mask, False, outcome.phase1_macs.total, phase2.total, plans)


def _dense_edit(eng: Engine, kv, lat0: torch.Tensor, start: int) -> torch.Tensor:
    """Full-mask edit: plain dense steps start..T with fresh statistics (unet.py:860,877-878)."""
    cfg = eng.config
    latents = torch.empty((cfg.steps + 1, eng.hw(0), cfg.latent_channels), dtype=torch.float32, device=eng.dev)
    latents[start - 1].copy_(lat0)
    _Runner(eng, StepPlan(eng, kv, latents, None), _use_graphs()).run(start, cfg.steps)
    return latents[cfg.steps]


def _add_dense_macs(counter: _MacsCounter, unet: UNet, n_text: int, n_steps: int):
    for lid, m_ in unet.dense_step_macs(n_text).items():
        counter.add(lid, m_ * n_steps)


def _add_sparse_macs(counter: _MacsCounter, unet: UNet, n_text: int, dp: DevicePlan, n_steps: int):
    """SparseMode MACs (unet.py:604-663): gated convs count plan.cost, attention active pixels."""
    cost = {l: 4 * dp.n_tiles[l] for l in range(unet.config.levels)}
    for lid, m_ in unet.sparse_step_macs(n_text, dp.n_active, cost).items():
        counter.add(lid, m_ * n_steps)


def _gather_plans(unet: UNet, dp: DevicePlan) -> dict:
    cfg = unet.config
    plans = {}
    for l in sorted({i.level for i in unet.layers if i.gated}):
        org = dp.origins(l)
        plans[l] = GatherPlan((4, 4), (2, 2), (3, 3), org, 4 * len(org), (cfg.latent_h >> l, cfg.latent_w >> l))
    return plans


# reference-compatible names of the per-layer mode protocol (unet.py:464-663,676,781)
from .modes import ControlledMode, DenseMode, SparseMode  # noqa: E402
from .modes import _MacsCounter as _ModeMacsCounter  # noqa: E402,F401
from .modes import sparse_contexts as _sparse_contexts  # noqa: E402


def _step_scale(config: UNetConfig):
    return step_scale(config)


# ---------------------------------------------------------------------------
# batched requests: R edits of one model stepped as one stacked batch
# ---------------------------------------------------------------------------

def generate_dense_batch(prompts, config: UNetConfig, stores, *, precision: str | None = None) -> list:
    """Dense generations of R prompts recorded into ONE stacked arena (generation r = image r of
    every slab), each bound to its CacheStore; `edit_batch` then steps their edits together.
    Returns the R final latents (NCHW numpy), as R generate_dense calls would."""
    if len(prompts) != len(stores) or not prompts:
        raise ContractViolation("generate_dense_batch needs one store per prompt")
    eng = get_engine(config, precision)
    stacked = Arena(eng, 0, full=False, batch=len(prompts))
    finals = []
    for r, (p, st) in enumerate(zip(prompts, stores)):
        view = stacked.view(r, len(p.ids))
        finals.append(generate_dense(p, config, st, record="engine", precision=precision, _arena=view))
    return finals


def stack_text_kv(eng: Engine, kvs):
    """Stack R prompts' text K [n, C] / V^T [C, n] per cross layer, each padded to a multiple of
    16 keys (zeros), plus the key segments [2R] of each request."""
    R = len(kvs)
    lid0 = next(iter(kvs[0]))
    nts = [kv[lid0][0].shape[0] for kv in kvs]
    ks = _pad(max(nts))
    out = {}
    for lid in kvs[0]:
        c = kvs[0][lid][0].shape[1]
        K = torch.zeros((R * ks, c), dtype=eng.act, device=eng.dev)
        VT = torch.zeros((c, R * ks), dtype=eng.act, device=eng.dev)
        MT = torch.zeros((R * ks, c), dtype=eng.act, device=eng.dev)
        for r, kv in enumerate(kvs):
            k, vt, _, mt = kv[lid]
            K[r * ks: r * ks + nts[r]] = k
            VT[:, r * ks: r * ks + nts[r]] = vt[:, :nts[r]]
            MT[r * ks: r * ks + nts[r]] = mt
        out[lid] = (K, VT, None, MT)
    kseg = torch.tensor([v for r in range(R) for v in (r * ks, r * ks + nts[r])], dtype=torch.int32, device=eng.dev)
    return out, kseg


class BatchedEditPlan:
    """Device plan of R edits over one stacked arena: per-request mask pyramids, concatenated
    row lists (each request's run padded to 16 rows), stacked pixel->row maps, attention
    segments and the BatchedSparsePlan that steps them as one batch."""

    def __init__(self, eng: Engine, stacked: Arena, masks, kvs, lat0s, stacked_kv=None):
        """kvs: per-request text K/V dicts (Engine.text_kv), or None with stacked_kv =
        Engine.text_kv_stacked(...) (one GEMM pair per cross layer for all requests)."""
        cfg = eng.config
        R = stacked.batch
        if not (len(masks) == len(lat0s) == R and (kvs is None or len(kvs) == R)):
            raise ContractViolation(f"need {R} masks / prompts / start latents for a {R}-request arena")
        if eng.act != torch.bfloat16:
            raise ContractViolation("batched edits run in bf16 (fused segment attention)")
        dev, i32 = eng.dev, torch.int32
        self.R = R
        # all R masks in one host->device copy, all R plan kernels before one read-back of their counts
        bits_d = torch.from_numpy(np.stack([m.bits.astype(np.uint8).ravel() for m in masks])).to(dev)
        self.dps = [DevicePlan(bits_d[r], cfg.latent_h, cfg.latent_w, cfg.levels, sync=False) for r in range(R)]
        DevicePlan.finish_all(self.dps)
        lists, qsegs, row_img = {}, {}, {}
        for l in range(cfg.levels):
            hw = eng.hw(l)
            if not eng.gated[l]:
                seg = [v for r in range(R) for v in (r * hw, (r + 1) * hw)]
                qsegs[l] = (torch.tensor(seg, dtype=i32, device=dev), R, hw)
                continue
            rows, idx, seg, img = [], [], [], []
            start = 0
            for r, dp in enumerate(self.dps):
                n = dp.n_active[l]
                npad = _pad(n)
                rr = dp.rows[l][:n] + r * hw
                if npad > n:  # padding rows repeat a live row of the request (never read back)
                    rr = torch.cat([rr, rr[:1].expand(npad - n)])
                ii = dp.index[l]
                idx.append(torch.where(ii >= 0, ii + start, ii))
                rows.append(rr)
                seg += [start, start + n]
                img.append(torch.full((npad,), r, dtype=i32, device=dev))
                start += npad
            rows_t = torch.cat(rows).to(i32).contiguous() if start else torch.zeros(1, dtype=i32, device=dev)
            lists[l] = (rows_t, torch.cat(idx).to(i32).contiguous(), start)
            qsegs[l] = (torch.tensor(seg, dtype=i32, device=dev), R, max(1, max(dp.n_active[l] for dp in self.dps)))
            row_img[l] = torch.cat(img).contiguous() if start else torch.zeros(1, dtype=i32, device=dev)
        self.lists = lists
        lat0 = torch.cat(list(lat0s), 0)
        r0, _, n0 = lists[0]
        self.lat_rows = lat0.index_select(0, r0[:n0].long()).contiguous()
        if stacked_kv is not None:
            kv, kseg, max_keys = stacked_kv
        else:
            kv, kseg = stack_text_kv(eng, kvs)
            lid0 = next(iter(kvs[0]))
            max_keys = max(kv_[lid0][0].shape[0] for kv_ in kvs)
        self.kv = kv
        # halo-mode GEMM rows of the gated levels' convs (framed runs of adjacent pixels; the rows'
        # outputs land at each request's compact row positions, engine.halo_lists)
        halo = {}
        for l in lists:
            hw = eng.hw(l)
            hl, wl = eng.grid(l)
            px_parts, out_parts, start = [], [], 0
            for r, dp in enumerate(self.dps):
                n = dp.n_active[l]
                px_parts.append(dp.rows[l][:n].long() + r * hw)
                out_parts.append(torch.arange(start, start + n, device=dev))
                start += _pad(n)
            if start == 0:
                continue
            pix, outi = halo_lists(torch.cat(px_parts).cpu().numpy(), torch.cat(out_parts).cpu().numpy(), hl, wl)
            halo[l] = (torch.from_numpy(pix).to(dev), torch.from_numpy(outi).to(dev), int(pix.size))
        self.halo = halo
        self.plan = BatchedSparsePlan(eng, kv, stacked, lists, self.lat_rows, qsegs, kseg, row_img, max_keys,
                                      halo=halo)

    def final_latents(self, eng: Engine, stacked: Arena) -> torch.Tensor:
        """[R * hw, Cl] f32: fresh rows where masked, the cached generation elsewhere."""
        cfg = eng.config
        out = torch.empty((self.R * eng.hw(0), cfg.latent_channels), dtype=torch.float32, device=eng.dev)
        fv = FeatVal(DRef(self.lat_rows), 0, cfg.latent_channels, self.lists[0][1], DRef(stacked.latent[cfg.steps]))
        eng.step_dev.fill_(0)
        eng.materialize(fv, DRef(out), n_img=self.R)
        return out


def edit_batch(sessions, config: UNetConfig) -> list:
    """Edits whose stores come from one `generate_dense_batch` (any subset of its generations, one
    session each), stepped as ONE stacked batch.

    Per request this matches `edit(session, config, session.store)` (unet.py:823-899) up to the
    bf16 bound: masks (user or detected) and prompts are per request; all requests must share
    the sparse phase's first step (same t2 with detection, or all user masks). Generations of the
    batch without a session ride along with an empty mask (no active rows) and are not returned.
    Returns one EditResult per session, in the given order."""
    if not sessions:
        return []
    views = [s.store.arena for s in sessions]
    stacked = getattr(views[0], "stacked", None)
    idx = [getattr(v, "index", -1) for v in views]
    if stacked is None or any(getattr(v, "stacked", None) is not stacked for v in views) or \
            len(set(idx)) != len(idx) or min(idx) < 0 or max(idx) >= stacked.batch:
        raise ContractViolation("edit_batch needs stores of one generate_dense_batch, one session each")
    order = sorted(range(len(sessions)), key=lambda i: views[i].index)
    sessions = [sessions[i] for i in order]
    views = [views[i] for i in order]
    outcomes = [detect_mask(s, config, s.store) for s in sessions]
    starts = {1 if o.from_user_mask else s.t2 + 1 for s, o in zip(sessions, outcomes)}
    if len(starts) != 1:
        raise ContractViolation(f"batched edits must share the sparse phase's first step, got {sorted(starts)}")
    start = starts.pop()
    eng = get_engine(config, stacked.eng.precision)
    cl, H, W, T = config.latent_channels, config.latent_h, config.latent_w, config.steps
    masks, lat0s = [], []
    lat_init = None
    for s, o, v in zip(sessions, outcomes, views):
        s.mask = o.mask
        # a no-edit request rides along with an empty mask: its latent stays the cached one
        masks.append(o.mask if o.mask is not None else BinaryMask(np.zeros((H, W), dtype=bool)))
        if o.from_user_mask or o.mask is None:
            if lat_init is None:  # the seeded initial latent is the same for every request
                lat_init = _initial_latent_dev(eng)
            lat0s.append(lat_init)
        else:
            m = torch.from_numpy(o.mask.bits.ravel().copy()).to(eng.dev)[:, None]
            lat0s.append(torch.where(m, o._control_dev, v.latent[s.t2]))
    # an all-active mask is a plain dense edit with fresh GroupNorm statistics (unet.py:860,877-878),
    # not a sparse step over the old generation's cached statistics: such requests ride in the
    # stacked batch with an empty mask (their rows are never read back) and are stepped densely
    full = [o.mask is not None and o.mask.all_active() for o in outcomes]
    batch_masks = [BinaryMask(np.zeros((H, W), dtype=bool)) if f else m for f, m in zip(full, masks)]
    texts = [embed_tokens(s.new_tokens, config) for s in sessions]
    # generations of the stacked batch without a session: empty mask, any prompt / start latent
    nb = stacked.batch
    slot = {v.index: r for r, v in enumerate(views)}
    empty = BinaryMask(np.zeros((H, W), dtype=bool))
    if len(slot) < nb and lat_init is None:
        lat_init = _initial_latent_dev(eng)
    b_masks = [batch_masks[slot[i]] if i in slot else empty for i in range(nb)]
    b_lat0 = [lat0s[slot[i]] if i in slot else lat_init for i in range(nb)]
    b_texts = [texts[slot[i]] if i in slot else texts[0] for i in range(nb)]
    skv = eng.text_kv_stacked(b_texts)
    bp = BatchedEditPlan(eng, stacked, b_masks, None, b_lat0, stacked_kv=skv)
    DevicePlan.fetch_tiles_all(bp.dps)  # (one transfer, before the steps are queued)
    _Runner(eng, bp.plan, _use_graphs() and os.environ.get("FIS_BATCH_GRAPH", "1") != "0").run(start, T)
    final = bp.final_latents(eng, stacked)
    hw = eng.hw(0)
    img = [v.index for v in views]  # stacked image of each (sorted) session
    for r, f in enumerate(full):
        if f:
            final[img[r] * hw:(img[r] + 1) * hw] = _dense_edit(eng, eng.text_kv(texts[r]), lat0s[r], start)
    # per-request accounting on the host while the queued steps run (no device sync in it)
    unet = _unet_of(config)
    acct = []
    for r, (s, o) in enumerate(zip(sessions, outcomes)):
        n_new = len(s.new_tokens.ids)
        phase2 = _MacsCounter()
        plans = {}
        if not o.no_edit:
            if full[r]:
                _add_dense_macs(phase2, unet, n_new, T - start + 1)
            else:
                _add_sparse_macs(phase2, unet, n_new, bp.dps[img[r]], T - start + 1)
                plans = _gather_plans(unet, bp.dps[img[r]])
        acct.append((_build_report(unet, n_new, config, [o.phase1_macs, phase2]), phase2, plans))
    fin = final.view(nb, H, W, cl).permute(0, 3, 1, 2).contiguous().cpu().numpy()  # one D2H
    results = [None] * len(sessions)
    for r, ((s, o), (rep, phase2, plans)) in enumerate(zip(zip(sessions, outcomes), acct)):
        results[order[r]] = EditResult(fin[img[r]:img[r] + 1], rep, s.store.stats(), o.mask, o.no_edit,
                                       o.phase1_macs.total, phase2.total, plans)
    return results
