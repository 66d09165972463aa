"""MGRF container: files written from the device class
buffer are byte-identical to the reference writer's (pipeline.cpp:180-206),
reads mirror read_refactored (prefix reads, CorruptFile / MissingClass), and
the GPU CRC-32 equals mgr::crc32 / zlib.crc32.

Golden containers: tests/golden/mgrf/*.mgrf, written by the reference itself
(tests/golden/make_mgrf_golden.py)."""
import os
import zlib

import numpy as np
import pytest

from paper_2105_12764_b200 import container, errors

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mgrf")
NAMES = ["c3d_f64", "c3d_f32_nonuni", "c2d_f32", "c2d_f64_nonuni", "c1d_f64",
         "c4d_f32_nonuni"]


def _case(name):
    z = np.load(os.path.join(GOLD, "cases.npz"))
    shape = tuple(int(x) for x in z[f"{name}/shape"])
    coords = None
    if f"{name}/coords0" in z:
        coords = [z[f"{name}/coords{d}"] for d in range(len(shape))]
    return dict(values=z[f"{name}/values"], classes=z[f"{name}/classes"], shape=shape,
                coords=coords, levels=int(z[f"{name}/levels"]),
                consumed=[int(x) for x in z[f"{name}/consumed"]],
                path=os.path.join(GOLD, f"{name}.mgrf"))


# ---- CPU: the header reader and the CRC oracle ------------------------------
@pytest.mark.parametrize("name", NAMES)
def test_header_parse_matches_golden(name):
    c = _case(name)
    h = container.read_refactored_header(c["path"])
    assert h.shape == c["shape"] and h.levels == c["levels"]
    assert h.np_dtype == c["classes"].dtype
    raw = open(c["path"], "rb").read()
    assert h.header_bytes + sum(r.bytes for r in h.class_records) == len(raw)
    off = h.header_bytes
    for rec in h.class_records:  # payload CRCs: zlib's crc32 == mgr::crc32
        assert zlib.crc32(raw[off:off + rec.bytes]) == rec.crc
        off += rec.bytes
    # the payload is the flat class buffer, class 0 first
    assert raw[h.header_bytes:] == c["classes"].tobytes()
    # prefix byte counts of the reference's read_refactored
    acc = h.header_bytes
    for k, rec in enumerate(h.class_records):
        acc += rec.bytes
        assert acc == c["consumed"][k]


def test_reference_crc32_is_zlib(oracle_mod):
    if not oracle_mod.available("ref"):
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    for n in (0, 1, 7, 511, 512, 513, 4096 + 3, 100003):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert oracle_mod.ref_crc32(b) == zlib.crc32(b)


@pytest.mark.parametrize("mutate,exc,msg", [
    (lambda b: b"MGRX" + b[4:], errors.CorruptFile, "bad magic"),
    (lambda b: b[:4] + b"\x02" + b[5:], errors.CorruptFile, "unsupported version 2"),
    (lambda b: b[:5] + b"\x01" + b[6:], errors.CorruptFile, "unsupported endianness"),
    (lambda b: b[:6] + b"\x05" + b[7:], errors.CorruptFile, "unsupported dtype 5"),
    (lambda b: b[:20], errors.CorruptFile, "unexpected end of data"),
])
def test_header_errors_match_reference(tmp_path, oracle_mod, mutate, exc, msg):
    c = _case("c3d_f64")
    p = tmp_path / "bad.mgrf"
    p.write_bytes(mutate(open(c["path"], "rb").read()))
    with pytest.raises(exc, match=msg):
        container.read_refactored_header(p)
    if oracle_mod.available("ref"):  # the reference raises the same type
        with pytest.raises(oracle_mod.OracleError) as ei:
            oracle_mod.ref_read_refactored(str(p), c["classes"].size, np.float64)
        assert ei.value.code == 8  # CorruptFile (errors.hpp; mgrg.h MGRG_CORRUPT_FILE)


# ---- GPU: device CRC, byte-identical writes, reads -------------------------
@pytest.mark.gpu
def test_gpu_crc32_matches_zlib():
    import torch

    rng = np.random.default_rng(9)
    big = rng.integers(0, 256, 5 * (1 << 20) + 77, dtype=np.uint8)
    d = torch.from_numpy(big).cuda()
    for off, n in [(0, 0), (0, 1), (3, 15), (0, 512), (1, 513), (5, 16383), (0, 16384),
                   (7, 16385), (0, 1 << 20), (13, (1 << 20) + 1000), (0, big.size),
                   (11, big.size - 11)]:
        assert container.crc32(d[off:off + n]) == zlib.crc32(big[off:off + n].tobytes()), (off, n)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_write_is_byte_identical_to_reference(tmp_path, name):
    import torch

    from paper_2105_12764_b200 import Plan

    c = _case(name)
    plan = Plan(c["shape"], c["values"].dtype.name, coords=c["coords"])  # exact policy
    d = plan.decompose(torch.from_numpy(c["values"]).cuda())
    assert np.array_equal(d.cpu().numpy(), c["classes"])
    p = tmp_path / "ours.mgrf"
    n = plan.write_refactored(d, p)
    raw = open(c["path"], "rb").read()
    assert n == len(raw)
    assert p.read_bytes() == raw
    assert plan.class_crc32(d) == [r.crc for r in container.read_refactored_header(p).class_records]
    plan.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_read_prefixes_match_reference(name):
    from paper_2105_12764_b200 import Plan

    c = _case(name)
    plan = Plan(c["shape"], c["values"].dtype.name, coords=c["coords"])
    offs = plan.class_offsets
    for k in range(c["levels"] + 1):
        t, loaded, used = plan.read_refactored(c["path"], k)
        assert loaded == k and used == c["consumed"][k]
        got = t.cpu().numpy()
        assert np.array_equal(got[: offs[k + 1]], c["classes"][: offs[k + 1]])
        assert not got[offs[k + 1]:].any()  # past the prefix: never written
    with pytest.raises(errors.MissingClass):
        plan.read_refactored(c["path"], c["levels"] + 1)
    plan.close()


@pytest.mark.gpu
def test_gpu_read_corruption_and_truncation(tmp_path):
    from paper_2105_12764_b200 import Plan

    c = _case("c3d_f32_nonuni")
    plan = Plan(c["shape"], "float32", coords=c["coords"])
    h = container.read_refactored_header(c["path"])
    raw = bytearray(open(c["path"], "rb").read())
    start2 = h.header_bytes + sum(r.bytes for r in h.class_records[:2])
    bad = bytearray(raw)
    bad[start2 + 5] ^= 0x40  # inside class 2
    p = tmp_path / "bad.mgrf"
    p.write_bytes(bytes(bad))
    plan.read_refactored(p, 1)  # the prefix before the damage still reads
    with pytest.raises(errors.CorruptFile, match="crc mismatch in class 2"):
        plan.read_refactored(p)
    q = tmp_path / "short.mgrf"
    q.write_bytes(bytes(raw[: start2 + 3]))
    plan.read_refactored(q, 1)
    with pytest.raises(errors.MissingClass, match="class 2 payload is truncated"):
        plan.read_refactored(q, 2)
    plan.close()


@pytest.mark.gpu
def test_gpu_fast_plan_container_reads_in_reference(tmp_path, oracle_mod):
    """A 129^3 f32 FAST-policy decompose written from the device is read back
    by the reference's read_refactored, CRCs and all."""
    import torch

    from paper_2105_12764_b200 import Plan

    if not oracle_mod.available("ref"):
        pytest.skip("oracle/_ref not built")
    shape = (129, 129, 129)
    v = np.random.default_rng(3).random(int(np.prod(shape))).astype(np.float32)
    plan = Plan(shape, "float32", fast=True)
    d = plan.decompose(torch.from_numpy(v).cuda())
    p = tmp_path / "big.mgrf"
    plan.write_refactored(d, p)
    got, loaded, used = oracle_mod.ref_read_refactored(str(p), v.size, np.float32)
    assert loaded == plan.levels and used == os.path.getsize(p)
    assert np.array_equal(got, d.cpu().numpy())
    # and through the RefactoredData-level mirror
    r = container.read_refactored(p)
    assert r.classes_loaded == plan.levels
    n2 = container.write_refactored(r.data, tmp_path / "again.mgrf")
    assert n2 == used and (tmp_path / "again.mgrf").read_bytes() == p.read_bytes()
    plan.close()
