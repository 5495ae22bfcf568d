"""AQKV workload files (R/src/workload_io.cpp:65-159, R/../SPEC.md:82) with a
bf16 dtype extension.

Layout, little-endian: magic "AQKV", version u32 = 1, head_count u32, n u64,
d u32, dtype u8, 3 reserved bytes; then per head the Q, K and V rows
(row-major).  dtype 0 = f32 (byte-identical to the reference's writer),
dtype 1 = bf16 (this extension: half the bytes, exactly the values the
tcgen05 path consumes).  Errors carry the reference's DecodeErrorKind names
and messages.
"""
from __future__ import annotations

import enum
import os
import struct

import numpy as np
import torch

MAGIC = b"AQKV"
VERSION = 1
DTYPE_F32 = 0
DTYPE_BF16 = 1
_HEADER = struct.Struct("<4sIIQIB3x")


class DecodeErrorKind(enum.Enum):
    BadMagic = "BadMagic"
    BadVersion = "BadVersion"
    Truncated = "Truncated"
    ShapeMismatch = "ShapeMismatch"
    EmptyWorkload = "EmptyWorkload"
    NonFinite = "NonFinite"
    Io = "Io"


class DecodeError(RuntimeError):
    def __init__(self, kind: DecodeErrorKind, what: str):
        super().__init__(what)
        self.kind = kind


def write_workload(path: str, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                   dtype: str = "f32") -> None:
    """q, k, v: [heads, n, d] (one K/V per head, as the reference stores them)."""
    if q.dim() != 3 or q.shape[0] == 0:
        raise DecodeError(DecodeErrorKind.EmptyWorkload, "write_workload: empty workload")
    if q.shape != k.shape or q.shape != v.shape:
        raise DecodeError(DecodeErrorKind.ShapeMismatch, "write_workload: heads must share (n, d)")
    heads, n, d = q.shape
    code = {"f32": DTYPE_F32, "bf16": DTYPE_BF16}[dtype]
    tdt = torch.float32 if code == DTYPE_F32 else torch.bfloat16
    try:
        with open(path, "wb") as f:
            f.write(_HEADER.pack(MAGIC, VERSION, heads, n, d, code))
            for h in range(heads):
                for x in (q[h], k[h], v[h]):
                    arr = x.detach().to("cpu", tdt).contiguous()
                    raw = arr.view(torch.int16).numpy() if code == DTYPE_BF16 else arr.numpy()
                    f.write(raw.astype(raw.dtype.newbyteorder("<"), copy=False).tobytes())
    except OSError as exc:
        raise DecodeError(DecodeErrorKind.Io, f"write_workload: cannot open {path}") from exc


def read_workload(path: str):
    """Returns (q, k, v) as [heads, n, d] tensors (f32 or bf16, as stored)."""
    if not os.path.exists(path):
        raise DecodeError(DecodeErrorKind.Io, f"read_workload: cannot open {path}")
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 4:
        raise DecodeError(DecodeErrorKind.Truncated, "read_workload: truncated header")
    if data[:4] != MAGIC:
        raise DecodeError(DecodeErrorKind.BadMagic, "read_workload: bad magic")
    if len(data) < _HEADER.size:
        raise DecodeError(DecodeErrorKind.Truncated, "read_workload: truncated header")
    _, version, heads, n, d, code = _HEADER.unpack_from(data)
    if version != VERSION:
        raise DecodeError(DecodeErrorKind.BadVersion,
                          f"read_workload: version mismatch (got {version})")
    if heads == 0:
        raise DecodeError(DecodeErrorKind.EmptyWorkload, "read_workload: empty workload")
    if n == 0 or d == 0:
        raise DecodeError(DecodeErrorKind.ShapeMismatch,
                          "read_workload: shape mismatch, n and d must be >= 1")
    if code not in (DTYPE_F32, DTYPE_BF16):
        raise DecodeError(DecodeErrorKind.ShapeMismatch, "read_workload: unsupported dtype")
    es = 4 if code == DTYPE_F32 else 2
    per = n * d * es
    out = ([], [], [])
    off = _HEADER.size
    for h in range(heads):
        for t in range(3):
            if off + per > len(data):
                raise DecodeError(DecodeErrorKind.Truncated,
                                  f"read_workload: truncated payload at head {h}")
            if code == DTYPE_F32:
                arr = torch.from_numpy(np.frombuffer(data, "<f4", n * d, off).copy())
            else:
                arr = torch.from_numpy(np.frombuffer(data, "<i2", n * d, off).copy()).view(
                    torch.bfloat16)
            out[t].append(arr.view(n, d))
            off += per
        if not all(torch.isfinite(x[-1].float()).all() for x in out):
            raise DecodeError(DecodeErrorKind.NonFinite,
                              f"read_workload: non-finite value in head {h}")
    return tuple(torch.stack(x) for x in out)
