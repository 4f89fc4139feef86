"""On-disk persistence of a cached generation (reference cache.py:119-276).

`cache.bin` keeps the reference's spill-file layout so either implementation can read the
other's reference-role entries:

  record  = u64 step, u64 layer, u64 role, u8 role (repeated as a check), u64 payload length,
            payload                                             (all little endian)
  payload = kind 0: u8 0, u8 ndim, 6 x u64 dims (zero padded), f32 data      (dense array)
            kind 1: u8 1, 4 x u64 shape, u64 index length, u8 index-is-active,
                    i32 index, f32 stored values                            (CompactTensor)
  footer  = JSON {"entries": [{step, layer, role, offset, length, bytes, compacted}, ...],
                  "fisedit": {...}}, u64 JSON length, 8-byte magic b"SPCACHE1"

The reference reads only the "entries" list of the footer; the "fisedit" object carries what
this engine needs to rebuild its HBM arena (config, precision, prompt, record mode).

The engine's own slabs (the conv-input features of the gated levels, which the reference does
not have) go to a sidecar `<spill>.engine` with the same record framing and payload kind 2:
u8 2, u8 dtype (0 f32, 1 bf16), u8 ndim, 6 x u64 dims, raw little-endian data -- one record
per whole [T+1, rows, C] slab (role = FEATURE, layer = the feature's ordinal).
"""

from __future__ import annotations

import json
import os
import struct

import numpy as np
import torch

from .errors import ContractViolation

MAGIC = b"SPCACHE1"
_REC = struct.Struct("<3QBQ")


def encode_payload(payload) -> bytes:
    from .cache import CompactTensor
    if isinstance(payload, CompactTensor):
        head = struct.pack("<B4QQB", 1, *[int(v) for v in payload.shape], int(payload.index.size),
                           1 if payload.index_is_active else 0)
        return head + payload.index.astype("<i4").tobytes() + np.ascontiguousarray(payload.values, "<f4").tobytes()
    a = np.ascontiguousarray(payload, dtype="<f4")
    if a.ndim > 6:
        raise ContractViolation(f"payload rank {a.ndim} > 6")
    dims = list(a.shape) + [0] * (6 - a.ndim)
    return struct.pack("<BB6Q", 0, a.ndim, *dims) + a.tobytes()


def decode_payload(buf: bytes):
    from .cache import CompactTensor
    kind = buf[0]
    if kind == 0:
        ndim = buf[1]
        dims = struct.unpack_from("<6Q", buf, 2)[:ndim]
        return np.frombuffer(buf, dtype="<f4", offset=50).reshape(dims).astype(np.float32)
    if kind == 1:
        n, c, h, w, nidx, is_active = struct.unpack_from("<4QQB", buf, 1)
        off = 42
        index = np.frombuffer(buf, dtype="<i4", count=nidx, offset=off).astype(np.int32)
        off += 4 * nidx
        stored = h * w - nidx if is_active else nidx
        values = np.frombuffer(buf, dtype="<f4", offset=off).reshape(n, c, stored).astype(np.float32)
        return CompactTensor((n, c, h, w), values, index, bool(is_active))
    raise ContractViolation(f"unknown payload kind {kind}")


def encode_slab(t: torch.Tensor) -> bytes:
    """kind 2: a device slab's raw bytes (f32 or bf16), copied to the host once."""
    code = {torch.float32: 0, torch.bfloat16: 1}[t.dtype]
    host = t.detach().contiguous().view(torch.int16 if code else torch.float32).cpu().numpy()
    dims = list(t.shape) + [0] * (6 - t.dim())
    return struct.pack("<BBB6Q", 2, code, t.dim(), *dims) + host.tobytes()


def decode_slab(buf: bytes, device) -> torch.Tensor:
    if buf[0] != 2:
        raise ContractViolation(f"engine record of kind {buf[0]}, expected 2")
    code, ndim = buf[1], buf[2]
    dims = struct.unpack_from("<6Q", buf, 3)[:ndim]
    raw = np.frombuffer(buf, dtype="<i2" if code else "<f4", offset=51).reshape(dims)
    t = torch.from_numpy(raw.copy())
    return (t.view(torch.bfloat16) if code else t).to(device)


class SpillWriter:
    """Append records, then `finish(extra)` writes the JSON footer and the magic."""

    def __init__(self, path):
        self.path = str(path)
        self.f = open(self.path, "wb")
        self.index = []

    def append(self, step: int, layer: int, role: int, payload_buf: bytes, nbytes: int, compacted=False):
        off = self.f.tell()
        self.f.write(_REC.pack(int(step), int(layer), int(role), int(role) & 0xFF, len(payload_buf)))
        self.f.write(payload_buf)
        self.index.append({"step": int(step), "layer": int(layer), "role": int(role), "offset": off,
                           "length": _REC.size + len(payload_buf), "bytes": int(nbytes), "compacted": bool(compacted)})

    def finish(self, extra: dict | None = None):
        blob = json.dumps({"entries": self.index, **({"fisedit": extra} if extra else {})}).encode("utf-8")
        self.f.write(blob)
        self.f.write(struct.pack("<Q", len(blob)))
        self.f.write(MAGIC)
        self.f.close()


def read_footer(path) -> dict:
    with open(path, "rb") as f:
        f.seek(0, os.SEEK_END)
        end = f.tell()
        if end < 16:
            raise ContractViolation(f"{path} is not a spill file (too short)")
        f.seek(end - 16)
        n, magic = struct.unpack("<Q8s", f.read(16))
        if magic != MAGIC:
            raise ContractViolation(f"{path} is missing the spill index footer")
        f.seek(end - 16 - n)
        return json.loads(f.read(n).decode("utf-8"))


def read_record(f, offset: int, length: int) -> bytes:
    f.seek(offset)
    buf = f.read(length)
    step, layer, role, role8, plen = _REC.unpack_from(buf)
    if role8 != (role & 0xFF) or plen != length - _REC.size:
        raise ContractViolation(f"corrupt spill record at offset {offset} in {getattr(f, 'name', '?')}")
    return buf[_REC.size:]
