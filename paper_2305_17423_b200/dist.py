"""Request-level data parallelism across the GPUs of one node (SURVEY §8 e).

Edit requests are independent (own cached generation, mask, prompts), so they are
statically sharded across ranks by estimated cost with no collective in the step
path. The only communication is (i) timing reductions and (ii) one final gather of
the edited latents (64 KB per C2 request) to rank 0 — NCCL over NVLink on GPUs,
gloo in the CPU tests.
"""

from __future__ import annotations

import heapq

import numpy as np
import torch
import torch.distributed as dist


def request_cost(mask_bits: np.ndarray) -> int:
    """Estimated sparse-step cost of a request: active 2x2 tiles at level 0 plus active pixels
    (the M of the level-0 gather-GEMMs, which dominate the gated work)."""
    b = np.asarray(mask_bits, bool)
    h, w = b.shape
    tiles = b[: h - h % 2, : w - w % 2].reshape(h // 2, 2, w // 2, 2).any(axis=(1, 3)).sum()
    return int(tiles) * 4 + int(b.sum())


def shard_requests(costs, world_size: int):
    """Longest-processing-time-first assignment. Returns a list of request-index lists per rank,
    each sorted ascending; deterministic (ties broken by request index, then rank)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0, r) for r in range(world_size)]
    out = [[] for _ in range(world_size)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(x) for x in out]


def is_dist() -> bool:
    return dist.is_available() and dist.is_initialized()


def max_over_ranks(x: float, device=None) -> float:
    if not is_dist():
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(local: dict, world_size: int, device=None):
    """Gather {request index: latent ndarray} from every rank to rank 0 (one collective per edit
    batch). Latents are fixed-shape float32, so this is a tensor all_gather, not pickling."""
    if not is_dist():
        return dict(local)
    keys = sorted(local)
    n_local = torch.tensor([len(keys)], device=device)
    counts = [torch.zeros_like(n_local) for _ in range(world_size)]
    dist.all_gather(counts, n_local)
    maxn = int(max(c.item() for c in counts))
    shape = next(iter(local.values())).shape if local else None
    shape_t = torch.tensor(list(shape) if shape else [0, 0, 0, 0], device=device)
    shapes = [torch.zeros_like(shape_t) for _ in range(world_size)]
    dist.all_gather(shapes, shape_t)
    shape = tuple(int(v) for v in max(shapes, key=lambda s: int(s.prod())).tolist())
    numel = int(np.prod(shape))
    buf = torch.zeros((maxn, numel + 1), dtype=torch.float32, device=device)
    for i, k in enumerate(keys):
        buf[i, 0] = k
        buf[i, 1:] = torch.from_numpy(np.ascontiguousarray(local[k], np.float32).ravel())
    bufs = [torch.zeros_like(buf) for _ in range(world_size)]
    dist.all_gather(bufs, buf)
    out = {}
    for r, b in enumerate(bufs):
        for i in range(int(counts[r].item())):
            out[int(b[i, 0].item())] = b[i, 1:].cpu().numpy().reshape(shape)
    return out
