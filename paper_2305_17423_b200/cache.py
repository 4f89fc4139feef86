"""HBM-resident activation cache with the reference CacheStore interface.

Replaces sparsedit's tiered CacheStore (cache.py:281-679). A generation
recorded by `generate_dense` lives in an `Arena` of per-step device slabs that
edits read in place (select-on-read) and never mutate (C2: ~1.2 GB bf16 per
50-step request, ~140 requests per B200). Beyond HBM, generations tier to
pinned host memory under `hot_budget` (LRU, copy-engine transfers on a side
stream, `prefetch` promotes ahead of the edit) and persist to a spill file in
the reference's layout (`flush_all` / `open_spill`, spill.py).

`get` returns float32 NCHW numpy arrays (the reference payload type); `put`
accepts them and, for keys backed by the arena (e.g. STEP_LATENT), writes the
device slab too, so device-side consumers see user overrides (as the
reference's detection fixtures do, test_unet.py:244-258).
"""

from __future__ import annotations

import enum
import os
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from .errors import CacheMissError, ContractViolation


class Role(enum.IntEnum):
    LAYER_OUTPUT = 0
    NORM_MEAN = 1
    NORM_VAR = 2
    CROSS_ATTN_MAP = 3
    STEP_LATENT = 4
    LAYER_INPUT = 5
    # engine roles (this framework): conv-input features of gated levels, keyed by producer
    FEATURE = 6
    POOLED = 7


class CacheKey(NamedTuple):
    step: int
    layer_id: int
    role: Role


def _as_key(key) -> CacheKey:
    step, layer_id, role = key
    return CacheKey(int(step), int(layer_id), Role(role))


@dataclass(frozen=True)
class CacheStats:
    hot_bytes: int
    cold_bytes: int
    total_bytes: int
    transfer_count: int
    transfer_bytes: int
    prefetch_hits: int
    blocking_loads: int
    pool_reuses: int
    pool_peak: int
    evict_warnings: int

    def to_json(self) -> dict:
        return dict(self.__dict__)


class BufferPool:
    """API-compatible stub of the CPU scratch pool (cache.py:182-213): device
    workspaces are owned by the engine, so nothing is pooled here."""

    def __init__(self):
        self.reuses = 0
        self.outstanding = 0
        self.peak = 0

    def acquire(self, shape) -> np.ndarray:
        self.outstanding += 1
        self.peak = max(self.peak, self.outstanding)
        return np.zeros(tuple(int(s) for s in shape), dtype=np.float32)

    def release(self, buf) -> None:
        self.outstanding -= 1


def _nhwc_to_nchw(t: torch.Tensor, c, h, w) -> np.ndarray:
    return t.float().reshape(h, w, c).permute(2, 0, 1).reshape(1, c, h, w).contiguous().cpu().numpy()


def _nchw_to_nhwc(a: np.ndarray) -> torch.Tensor:
    n, c, h, w = a.shape
    return torch.from_numpy(np.ascontiguousarray(a[0].reshape(c, h * w).T))


class _Tiers:
    """Process-wide LRU of the stores that hold a generation (reference cache.py:358-400).

    The unit of residency is a whole generation: the edit kernels address every step of a slab
    as base + t * stride, so a generation is either all in HBM ("hot") or all in pinned host
    memory ("cold", moved by the copy engine on a side stream). When the hot generations exceed
    the smallest `hot_budget` of the registered stores, the least recently used ones other than
    the one being edited go cold; a generation that alone exceeds the budget stays hot and
    counts an evict warning (reference cache.py:378-382)."""

    def __init__(self):
        import weakref
        from collections import OrderedDict
        self._ref = weakref.ref
        self.order: "OrderedDict[int, object]" = OrderedDict()
        self.streams = {}

    def stream(self, dev):
        st = self.streams.get(dev)
        if st is None:
            st = self.streams[dev] = torch.cuda.Stream(device=dev)
        return st

    def live(self):
        out = []
        for k, r in list(self.order.items()):
            s = r()
            if s is None:
                del self.order[k]
            else:
                out.append(s)
        return out

    def touch(self, store):
        self.order[id(store)] = self._ref(store)
        self.order.move_to_end(id(store))
        self.enforce(store)

    def forget(self, store):
        self.order.pop(id(store), None)

    def enforce(self, keep):
        stores = self.live()
        budgets = [s.hot_budget for s in stores if s.hot_budget is not None]
        if not budgets:
            return
        budget = min(budgets)
        hot = [s for s in stores if s._state == "hot" and s._arena is not None]
        total = sum(s._arena.nbytes() for s in hot)
        for s in hot:  # LRU first
            if total <= budget:
                break
            if s is keep or not s._movable():
                continue
            nb = s._arena.nbytes()
            s._to_host()
            total -= nb
        if total > budget and keep is not None:
            keep._evict_warnings += 1


_TIERS = _Tiers()


class CacheStore:
    """(step, layer, role)-keyed store over one cached generation: an HBM arena ("hot"), its
    pinned host copy ("cold"), or a spill file opened with `open_spill` ("disk")."""

    def __init__(self, hot_budget=None, spill_path=None, async_transfer=True, load_delay=0.0):
        self.hot_budget = hot_budget
        self.spill_path = spill_path
        self._async = async_transfer
        self._extra: dict[CacheKey, np.ndarray] = {}
        self._arena = None  # engine.Arena (device) when hot
        self._host = None  # engine.Arena of pinned host tensors when cold
        self._engine = None
        self._state = "empty"  # empty | hot | cold | arriving | disk
        self._event = None
        self._disk = None  # open_spill: (cache.bin path, sidecar path, footer)
        self._current_step = 0
        self._pool = BufferPool()
        self._closed = False
        self._transfer_count = self._transfer_bytes = 0
        self._prefetch_hits = self._blocking_loads = self._evict_warnings = 0

    # -- arena binding (done by generate_dense) --------------------------------
    def _bind(self, engine, arena):
        self._engine, self._arena, self._state = engine, arena, "hot"
        _TIERS.touch(self)

    @property
    def arena(self):
        """The device arena, promoted from the host / disk tier first if needed."""
        self._ensure_hot()
        return self._arena

    def _movable(self) -> bool:
        # views of a stacked generate_dense_batch arena share their slabs with the other requests
        return self._arena is not None and getattr(self._arena, "stacked", None) is None

    # -- tiers -------------------------------------------------------------------
    def _to_host(self):
        """Hot -> cold: copy every slab to pinned host memory on the transfer stream, drop the
        device slabs and the step graphs captured over them."""
        a = self._arena
        st = _TIERS.stream(a.latent.device)
        st.wait_stream(torch.cuda.current_stream(a.latent.device))

        def to_host(t):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t, non_blocking=True)
            return h

        with torch.cuda.stream(st):
            host = a.map_tensors(to_host)
        st.synchronize()
        self.graph_cache().clear()
        self._host, self._arena, self._state = host, None, "cold"
        self._transfer_count += 1
        self._transfer_bytes += host.nbytes()

    def _start_to_device(self):
        """Cold -> arriving: copy-engine H2D of every slab on the transfer stream."""
        dev = self._engine.dev
        st = _TIERS.stream(dev)
        with torch.cuda.stream(st):
            self._arena = self._host.map_tensors(lambda h: h.to(dev, non_blocking=True))
            self._event = torch.cuda.Event()
            self._event.record(st)
        self._state = "arriving"
        self._transfer_count += 1
        self._transfer_bytes += self._host.nbytes()

    def _ensure_hot(self):
        if self._state == "arriving":
            torch.cuda.current_stream(self._engine.dev).wait_event(self._event)
            self._prefetch_hits += 1
            self._state, self._host, self._event = "hot", None, None
            _TIERS.touch(self)
        elif self._state == "cold":
            self._blocking_loads += 1
            self._start_to_device()
            torch.cuda.current_stream(self._engine.dev).wait_event(self._event)
            self._state, self._host, self._event = "hot", None, None
            _TIERS.touch(self)
        elif self._state == "disk":
            self._blocking_loads += 1
            self._load_spill()
            _TIERS.touch(self)
        elif self._state == "hot":
            _TIERS.order.move_to_end(id(self)) if id(self) in _TIERS.order else None

    # -- spill files (f4) --------------------------------------------------------
    @classmethod
    def open_spill(cls, path, **kwargs) -> "CacheStore":
        """Open a spill written by `flush_all` (reference cache.py:316-339): entries are read
        from the file on `get`; the first edit loads the whole generation back into HBM from
        the engine sidecar. A reference-written spill (no sidecar) serves `get` only."""
        from . import spill
        store = cls(**kwargs)
        footer = spill.read_footer(path)
        side = str(path) + ".engine"
        store._disk = (str(path), side if os.path.exists(side) else None, footer)
        store._state = "disk"
        return store

    def _load_spill(self):
        from . import spill
        from .model import UNetConfig
        from .unet import get_engine
        path, side, footer = self._disk
        meta = footer.get("fisedit")
        if meta is None or side is None:
            raise ContractViolation(f"{path} holds no engine slabs (written by the reference?): regenerate it "
                                    "with this engine to edit against it")
        eng = get_engine(UNetConfig.from_json(meta["config"]), meta["precision"])
        from .engine import Arena
        arena = Arena.__new__(Arena)
        arena.eng, arena.n_text, arena.full, arena.T, arena.batch = eng, meta["n_text"], meta["full"], eng.config.steps, 1
        arena.prompt = tuple(meta["prompt"])
        arena.latent, arena.feature, arena.stats, arena.maps, arena.outputs = None, {}, {}, {}, {}
        side_footer = spill.read_footer(side)
        with open(side, "rb") as f:
            for rec, name in zip(side_footer["entries"], side_footer["fisedit"]["slabs"]):
                t = spill.decode_slab(spill.read_record(f, rec["offset"], rec["length"]), eng.dev)
                kind = name[0]
                if kind == "latent":
                    arena.latent = t
                elif kind == "feature":
                    arena.feature[tuple(name[1:])] = t
                elif kind in ("mean", "var"):
                    m, v = arena.stats.get(name[1], (None, None))
                    arena.stats[name[1]] = (t, v) if kind == "mean" else (m, t)
                elif kind == "map":
                    arena.maps[name[1]] = t
                else:
                    arena.outputs[name[1]] = t
        self._engine, self._arena, self._state = eng, arena, "hot"
        self._transfer_count += 1
        self._transfer_bytes += arena.nbytes()

    def _write_spill(self, path):
        """cache.bin in the reference layout (reference roles, NCHW float32) + the engine sidecar."""
        from . import spill
        a, e = self._arena, self._engine
        cfg = e.config
        w = spill.SpillWriter(path)
        for k in self.keys():
            if k.role in (Role.FEATURE, Role.POOLED):
                continue
            v = self.get(k)
            w.append(k.step, k.layer_id, int(k.role), spill.encode_payload(v), v.nbytes)
        meta = {"config": cfg.to_json(), "precision": e.precision, "prompt": list(getattr(a, "prompt", ())),
                "n_text": a.n_text, "full": a.full, "sidecar": os.path.basename(str(path)) + ".engine"}
        w.finish(meta)
        sw = spill.SpillWriter(str(path) + ".engine")
        names = []
        for i, (name, t) in enumerate(a.slabs()):
            sw.append(0, i, int(Role.FEATURE), spill.encode_slab(t), t.numel() * t.element_size())
            names.append([n if not isinstance(n, tuple) else list(n) for n in name])
        sw.finish({"slabs": names})
        self._transfer_count += 1
        self._transfer_bytes += a.nbytes()

    def _disk_get(self, k: CacheKey):
        from . import spill
        path, _, footer = self._disk
        for rec in footer["entries"]:
            if (rec["step"], rec["layer"], rec["role"]) == (k.step, k.layer_id, int(k.role)):
                with open(path, "rb") as f:
                    return spill.decode_payload(spill.read_record(f, rec["offset"], rec["length"]))
        return None

    # -- arena-backed entries -----------------------------------------------------
    def _arena_tensor(self, k: CacheKey):
        a, e = self._arena, self._engine
        if a is None or not (0 <= k.step <= a.T):
            return None
        if k.role == Role.STEP_LATENT and k.layer_id == 0 and k.step >= 1:
            return a.latent[k.step], (e.config.latent_channels, e.config.latent_h, e.config.latent_w)
        info = e.info.get(k.layer_id)
        if info is None or k.step < 1:
            return None
        if k.role == Role.LAYER_OUTPUT and k.layer_id in a.outputs:
            return a.outputs[k.layer_id][k.step], (info.channels, info.h, info.w)
        if k.role in (Role.NORM_MEAN, Role.NORM_VAR) and k.layer_id in a.stats:
            return a.stats[k.layer_id][int(k.role) - 1][k.step].reshape(1, -1), None
        if k.role == Role.CROSS_ATTN_MAP and k.layer_id in a.maps:
            return a.maps[k.layer_id][k.step], None
        return None

    # -- public operations ------------------------------------------------------
    def put(self, key, payload, overwrite: bool = False) -> None:
        k = _as_key(key)
        if isinstance(payload, CompactTensor):
            payload = payload.materialize()
        if not isinstance(payload, np.ndarray):
            raise ContractViolation(f"unsupported payload type {type(payload)}")
        if payload.dtype != np.float32:
            raise ContractViolation(f"payloads must be float32, got {payload.dtype}")
        if self.contains(k) and not overwrite:
            raise ContractViolation(f"key {k} already present (pass overwrite=True)")
        if self._state in ("cold", "arriving", "disk"):
            self._ensure_hot()
        hit = self._arena_tensor(k)
        if hit is not None:
            t, shape = hit
            src = _nchw_to_nhwc(payload) if shape is not None else torch.from_numpy(payload.reshape(t.shape))
            t.copy_(src.to(t.device, t.dtype))
            if k in self._extra:
                del self._extra[k]
            return
        self._extra[k] = payload.copy()

    def get(self, key):
        k = _as_key(key)
        if k in self._extra:
            return self._extra[k]
        if self._state == "disk":
            v = self._disk_get(k)
            if v is None:
                raise CacheMissError(k.step, k.layer_id, k.role.name.lower())
            return v
        if self._state in ("cold", "arriving"):
            self._ensure_hot()
        hit = self._arena_tensor(k)
        if hit is None:
            raise CacheMissError(k.step, k.layer_id, k.role.name.lower())
        t, shape = hit
        if shape is None:
            return t.float().cpu().numpy().copy()
        return _nhwc_to_nchw(t, *shape)

    def contains(self, key) -> bool:
        k = _as_key(key)
        return k in set(self.keys())

    def keys(self) -> list[CacheKey]:
        out = list(self._extra)
        if self._state == "disk":
            return out + [CacheKey(r["step"], r["layer"], Role(r["role"])) for r in self._disk[2]["entries"]]
        a = self._arena if self._arena is not None else self._host
        if a is not None:
            for t in range(1, a.T + 1):
                out.append(CacheKey(t, 0, Role.STEP_LATENT))
                for lid in a.outputs:
                    out.append(CacheKey(t, lid, Role.LAYER_OUTPUT))
                for lid in a.stats:
                    out += [CacheKey(t, lid, Role.NORM_MEAN), CacheKey(t, lid, Role.NORM_VAR)]
                for lid in a.maps:
                    out.append(CacheKey(t, lid, Role.CROSS_ATTN_MAP))
        return out

    def set_current_step(self, step: int) -> None:
        self._current_step = step

    def prefetch(self, step: int) -> None:
        """Start promoting a cold generation to HBM on the copy engine (non-blocking); the next
        edit finds it arrived (a prefetch hit). The step argument is kept for the reference
        signature: residency is per generation (see _Tiers)."""
        if self._state == "cold":
            self._start_to_device()

    def drain(self) -> None:
        """Wait for an in-flight prefetch (makes the counters deterministic, reference cache.py:603-610)."""
        if self._state == "arriving":
            self._event.synchronize()

    def evict(self) -> None:
        """Apply the HBM budget now (LRU generations other than the most recent go cold)."""
        if self._state == "hot":
            _TIERS.enforce(self)

    def flush_all(self) -> None:
        """Persist the generation to `spill_path` (cache.bin + engine sidecar); the reference
        flushes every hot entry cold (cache.py:580-600), here the HBM copy also stays usable."""
        if self.spill_path is None:
            raise ContractViolation("flush_all needs a spill_path")
        self._ensure_hot()
        if self._arena is None:
            raise ContractViolation("nothing to flush: no generation is bound to this store")
        self._write_spill(self.spill_path)

    def compact(self, mask) -> None:
        """No-op: the edit engine reads the pristine generation in place."""

    def acquire_buffer(self, shape):
        return self._pool.acquire(shape)

    def release_buffer(self, buf) -> None:
        self._pool.release(buf)

    @property
    def buffer_pool(self) -> BufferPool:
        return self._pool

    def stats(self) -> CacheStats:
        host = sum(v.nbytes for v in self._extra.values())
        hot = self._arena.nbytes() if self._arena is not None and self._state == "hot" else 0
        cold = self._host.nbytes() if self._host is not None else 0
        if self._state == "disk":
            cold = sum(r["bytes"] for r in self._disk[2]["entries"])
        return CacheStats(hot + host, cold, hot + host + cold, self._transfer_count, self._transfer_bytes,
                          self._prefetch_hits, self._blocking_loads, self._pool.reuses, self._pool.peak,
                          self._evict_warnings)

    def hot_keys(self):
        return set(self.keys()) if self._state == "hot" else set(self._extra)

    def graph_cache(self) -> dict:
        """Captured edit-step graphs over this store's generation (unet._cached_runner). Owned by
        the store, not the arena: a graph's plan references the arena, so keeping them here
        avoids a reference cycle (whose collection could run inside a later graph capture) and
        frees them deterministically with the store or on close()."""
        g = getattr(self, "_graphs", None)
        if g is None:
            from collections import OrderedDict
            g = self._graphs = OrderedDict()
        return g

    def close(self) -> None:
        if getattr(self, "_graphs", None):
            self._graphs.clear()
        _TIERS.forget(self)
        self._arena = self._host = None
        self._state = "empty"
        self._extra.clear()
        self._closed = True

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


@dataclass(frozen=True)
class CompactTensor:
    """A layer output kept only at the pixels outside an edit mask (reference cache.py:64-92).

    `values` [n, c, n_stored] holds the stored (mask-complement) pixels in row-major pixel
    order; `index` lists either the active or the stored pixel ids, whichever list is shorter
    (`index_is_active` says which). The HBM arena never compacts (edits read the pristine
    generation); this type exists for callers of the reference payload API.
    """

    shape: tuple
    values: np.ndarray
    index: np.ndarray
    index_is_active: bool

    @property
    def nbytes(self) -> int:
        return int(self.values.nbytes + self.index.nbytes)

    def stored_positions(self) -> np.ndarray:
        hw = int(self.shape[2]) * int(self.shape[3])
        if not self.index_is_active:
            return self.index.astype(np.int64)
        keep = np.ones(hw, dtype=bool)
        keep[self.index.astype(np.int64)] = False
        return np.flatnonzero(keep)

    def materialize(self) -> np.ndarray:
        """Full float32 tensor: stored pixels restored, zeros at the active ones."""
        n, c, h, w = (int(v) for v in self.shape)
        out = np.zeros((n, c, h * w), dtype=np.float32)
        out[:, :, self.stored_positions()] = self.values
        return out.reshape(n, c, h, w)


def compact_tensor(arr: np.ndarray, mask_bits: np.ndarray) -> CompactTensor:
    """Drop the mask-active pixels of a (n, c, h, w) payload (reference cache.py:95-105)."""
    n, c, h, w = arr.shape
    bits = np.asarray(mask_bits, dtype=bool).ravel()
    stored, active = np.flatnonzero(~bits), np.flatnonzero(bits)
    vals = arr.reshape(n, c, h * w)[:, :, stored].copy()
    use_active = active.size <= stored.size
    idx = (active if use_active else stored).astype(np.int32)
    return CompactTensor((n, c, h, w), vals, idx, use_active)


def materialize_payload(payload):
    """Full ndarray of a payload (CompactTensor materialised, arrays returned as is)."""
    return payload.materialize() if isinstance(payload, CompactTensor) else payload
