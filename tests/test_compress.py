"""Compression pipeline: mgr::compress / decompress
(pipeline.hpp:149-198, pipeline.cpp:381-547) with the decompose, the
quantizer's error-bound search and the zigzag-varint coding on the GPU and
the codec on the host.  Under the exact arithmetic policy the containers are
byte-identical to the reference's; decompressed fields are bit-identical."""
import struct

import numpy as np
import pytest

from paper_2105_12764_b200 import container, errors

CASES = [  # (shape, dtype, nonuniform, error bound)
    ((17, 9, 5), "float64", False, 1e-3),
    ((33, 17, 9), "float32", True, 1e-2),
    ((65, 33), "float64", False, 1e-6),
    ((12, 10, 9), "float32", False, 5e-4),
    ((129,), "float64", True, 1e-9),
    ((9, 5, 5, 5), "float64", False, 1e-4),  # 4-D
]


def _field(shape, dtype, nonuni, seed):
    rng = np.random.default_rng(seed)
    coords = [np.cumsum(rng.uniform(0.1, 1.0, n)) for n in shape] if nonuni else None
    v = rng.random(int(np.prod(shape))).astype(dtype)
    return v, coords


def _rebuild_store(data: bytes, streams):
    """A store-codec MGRC container with the given per-class raw streams."""
    codec, dt, shape, coords, levels = container._compressed_header(data)
    head = 4 + 4 + 8 * len(shape) + 8 * sum(shape) + 8 + 24
    out = bytearray(data[:head])
    out[5] = 0  # codec id: store
    at = head
    for s in streams:
        count, _raw, enc = struct.unpack("<QQQ", data[at:at + 24])
        at += 24 + enc
        out += struct.pack("<QQQ", count, len(s), len(s)) + s
    return bytes(out)


def _streams(data: bytes):
    codec, dt, shape, coords, levels = container._compressed_header(data)
    at = 4 + 4 + 8 * len(shape) + 8 * sum(shape) + 8 + 24
    out = []
    for _ in range(levels + 1):
        count, raw, enc = struct.unpack("<QQQ", data[at:at + 24])
        assert codec == 0 and raw == enc
        out.append(data[at + 24:at + 24 + enc])
        at += 24 + enc
    return out


# ---- CPU: the reference pipeline pinned, header parse -------------------------
def test_reference_pipeline_pinned(oracle_mod):
    if not oracle_mod.available("ref"):
        pytest.skip("oracle/_ref not built")
    v, coords = _field((17, 9, 5), "float64", False, 1)
    data, b, m = oracle_mod.ref_compress(v, (17, 9, 5), 1e-3, 1)
    assert m <= 1e-3 and b > 0
    back = oracle_mod.ref_decompress(data, v.size, np.float64)
    assert np.abs(back - v).max() <= 1e-3
    codec, dt, shape, _, levels = container._compressed_header(data)
    assert (codec, dt, shape) == (1, 8, (17, 9, 5)) and levels == 2
    with pytest.raises(oracle_mod.OracleError) as ei:
        oracle_mod.ref_compress(v, (17, 9, 5), 0.0)
    assert ei.value.code == 10  # InvalidBound
    with pytest.raises(errors.CorruptFile, match="bad magic"):
        container._compressed_header(b"MGRX" + data[4:])


# ---- GPU --------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("codec", [0, 1], ids=["store", "zlib"])
def test_gpu_compress_bytes_match_reference(case, codec, oracle_mod):
    import torch

    from paper_2105_12764_b200 import Plan

    if not oracle_mod.available("ref"):
        pytest.skip("oracle/_ref not built")
    shape, dt, nonuni, eb = CASES[case]
    v, coords = _field(shape, dt, nonuni, 100 + case)
    ref, rb, rm = oracle_mod.ref_compress(v, shape, eb, codec, coords)
    plan = Plan(shape, dt, coords=coords)  # exact policy
    d = torch.from_numpy(v).cuda()
    data, b, m = plan.compress(d, eb, codec)
    assert (b, m) == (rb, rm)
    assert data == ref
    out, e2, b2, m2, c2 = plan.decompress(ref)
    assert (e2, b2, m2, c2) == (eb, rb, rm, codec)
    assert np.array_equal(out.cpu().numpy(), oracle_mod.ref_decompress(ref, v.size, dt))
    plan.close()


@pytest.mark.gpu
def test_gpu_compress_fast_policy_meets_bound():
    import torch

    from paper_2105_12764_b200 import Plan

    shape = (129, 65, 33)
    v, _ = _field(shape, "float32", False, 7)
    plan = Plan(shape, "float32", fast=True)
    for eb in (1e-2, 1e-4):
        data, b, m = plan.compress(torch.from_numpy(v).cuda(), eb, 1)
        assert m <= eb
        out, *_ = plan.decompress(data)
        assert float((out.cpu() - torch.from_numpy(v)).abs().max()) <= eb
    plan.close()


@pytest.mark.gpu
def test_gpu_compress_api_mirror_and_errors(oracle_mod):
    from paper_2105_12764_b200 import TensorGrid, make_grid

    v, coords = _field((33, 17, 9), "float64", True, 3)
    g = make_grid((33, 17, 9), v, coords)
    r = container.compress(g, 1e-4)
    assert r.report.codec == "zlib" and r.report.measured_max_abs_error <= 1e-4
    d = container.decompress(r.bytes)
    assert isinstance(d.grid, TensorGrid)
    assert float(np.abs(d.grid.values.cpu().numpy() - v).max()) <= 1e-4
    with pytest.raises(errors.InvalidBound):
        container.compress(g, 0.0)
    with pytest.raises(errors.InvalidBound):
        container.compress(g, 1e-3, codec="lz4")


@pytest.mark.gpu
@pytest.mark.parametrize("damage,msg", [
    ("truncate", "truncated varint stream"),
    ("trailing", "trailing bytes in varint stream"),
    ("overflow", "varint overflow"),
])
def test_gpu_varint_errors_match_reference(damage, msg, oracle_mod):
    import torch  # noqa: F401

    from paper_2105_12764_b200 import Plan

    if not oracle_mod.available("ref"):
        pytest.skip("oracle/_ref not built")
    shape = (17, 9, 5)
    v, _ = _field(shape, "float64", False, 5)
    ref, _, _ = oracle_mod.ref_compress(v, shape, 1e-3, 0)
    s = _streams(ref)
    s1 = bytearray(s[1])
    if damage == "truncate":
        s1[-1] |= 0x80          # the last element never terminates
    elif damage == "trailing":
        s1 += b"\x00"           # one element too many
    else:
        s1 = bytearray(b"\xff" * 10 + b"\x01") + s1[1:]  # 11-byte first element
    bad = _rebuild_store(ref, [s[0], bytes(s1)] + s[2:])
    plan = Plan(shape, "float64")
    with pytest.raises(errors.CorruptFile, match=msg):
        plan.decompress(bad)
    with pytest.raises(oracle_mod.OracleError) as ei:
        oracle_mod.ref_decompress(bad, v.size, np.float64)
    assert ei.value.code == 8  # the reference raises CorruptFile too
    plan.close()
