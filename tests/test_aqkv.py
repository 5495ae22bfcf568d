"""AQKV files (R/src/workload_io.cpp) and the bf16 extension: f32 files are
byte-identical to the reference's own writer and readable by it; every
decode error kind of the reference is reproduced."""
import ctypes as C
import os
import struct

import pytest
import torch

from oracle.oracle import REF_PATH
from paper_2505_23520_b200 import aqkv


def rand(h=2, n=16, d=8, seed=11):
    g = torch.Generator().manual_seed(seed)
    return [torch.randn(h, n, d, generator=g) for _ in range(3)]


def test_roundtrip_f32_and_bf16(tmp_path):
    q, k, v = rand()
    p = str(tmp_path / "w.aqkv")
    aqkv.write_workload(p, q, k, v)
    q2, k2, v2 = aqkv.read_workload(p)
    assert torch.equal(q, q2) and torch.equal(k, k2) and torch.equal(v, v2)
    aqkv.write_workload(p, q, k, v, dtype="bf16")
    q3, k3, v3 = aqkv.read_workload(p)
    assert q3.dtype == torch.bfloat16 and torch.equal(q3, q.bfloat16())
    assert os.path.getsize(p) == 28 + 3 * q.numel() * 2


@pytest.mark.skipif(not os.path.exists(REF_PATH), reason="oracle/_ref not built")
def test_f32_bytes_match_reference_writer(tmp_path):
    L = C.CDLL(REF_PATH)
    L.ref_write_workload.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64] + [C.c_void_p] * 3
    L.ref_read_workload.argtypes = [C.c_char_p]
    L.ref_read_workload.restype = C.c_int64
    q, k, v = rand(3, 32, 8, seed=5)
    ours, theirs = str(tmp_path / "ours.aqkv"), str(tmp_path / "ref.aqkv")
    aqkv.write_workload(ours, q, k, v)
    assert L.ref_write_workload(theirs.encode(), 3, 32, 8, q.data_ptr(), k.data_ptr(),
                                v.data_ptr()) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert L.ref_read_workload(ours.encode()) == 3


@pytest.mark.parametrize("mutate,kind", [
    (lambda b: b"XQKV" + b[4:], aqkv.DecodeErrorKind.BadMagic),
    (lambda b: b[:4] + struct.pack("<I", 2) + b[8:], aqkv.DecodeErrorKind.BadVersion),
    (lambda b: b[:10], aqkv.DecodeErrorKind.Truncated),
    (lambda b: b[:-4], aqkv.DecodeErrorKind.Truncated),
    (lambda b: b[:8] + struct.pack("<I", 0) + b[12:], aqkv.DecodeErrorKind.EmptyWorkload),
    (lambda b: b[:24] + bytes([7]) + b[25:], aqkv.DecodeErrorKind.ShapeMismatch),
    (lambda b: b[:28] + struct.pack("<f", float("nan")) + b[32:], aqkv.DecodeErrorKind.NonFinite),
])
def test_decode_errors(tmp_path, mutate, kind):
    q, k, v = rand(1, 4, 2)
    p = str(tmp_path / "w.aqkv")
    aqkv.write_workload(p, q, k, v)
    b = open(p, "rb").read()
    open(p, "wb").write(mutate(b))
    with pytest.raises(aqkv.DecodeError) as ei:
        aqkv.read_workload(p)
    assert ei.value.kind == kind
    with pytest.raises(aqkv.DecodeError) as ei:
        aqkv.read_workload(str(tmp_path / "missing.aqkv"))
    assert ei.value.kind == aqkv.DecodeErrorKind.Io
