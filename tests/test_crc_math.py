"""Host-side check of the GPU CRC-32 algebra (paper_2105_12764_b200/csrc/
crc32.cuh): the lane-stream decomposition of a segment (64 bytes per lane
per 2 KiB quad, Horner with Z_2048, butterfly with Z_64 .. Z_1024, 1-3
trailing 512-byte blocks folded 16 bytes per lane and appended with
Z_{512*rem}) and the combine (segment runs, pairwise tree, head / tail
bytes, init term) reproduce zlib.crc32 -- the reference's mgr::crc32
(pipeline.cpp:13-28).  Pure Python on small buffers."""
import zlib

import numpy as np
import pytest

_T = []
for i in range(256):
    c = i
    for _ in range(8):
        c = (c >> 1) ^ (0xEDB88320 if c & 1 else 0)
    _T.append(c)


def crc0(data: bytes, c: int = 0) -> int:
    """CRC register after `data` from register c (no init / final xor)."""
    for b in data:
        c = _T[(c ^ b) & 255] ^ (c >> 8)
    return c


def zshift(v: int, n: int) -> int:
    """Z_n: feed n zero bytes."""
    return crc0(bytes(n), v)


def segment_value(seg: bytes) -> int:
    """crc0 of a segment of whole 512-byte blocks, computed the way
    crc_blocks2_kernel does (32 lanes)."""
    nblk = len(seg) // 512
    nquad, rem = nblk // 4, nblk % 4
    acc = [0] * 32
    for q in range(nquad):
        for a in range(32):
            piece = seg[q * 2048 + 64 * a: q * 2048 + 64 * a + 64]
            acc[a] = zshift(acc[a], 2048) ^ crc0(piece)
    for k in range(5):  # butterfly: acc[a] = Z_{64*2^k}(acc[a]) ^ acc[a + 2^k]
        s = 1 << k
        acc = [zshift(acc[a], 64 * s) ^ (acc[a + s] if a + s < 32 else 0) for a in range(32)]
    v = acc[0]
    if rem:
        h = [0] * 32
        for b in range(4 * nquad, nblk):
            for a in range(32):
                h[a] = zshift(h[a], 512) ^ crc0(seg[b * 512 + 16 * a: b * 512 + 16 * a + 16])
        for k in range(5):
            s = 1 << k
            h = [zshift(h[a], 16 * s) ^ (h[a + s] if a + s < 32 else 0) for a in range(32)]
        v = zshift(v, 512 * rem) ^ h[0]
    return v


def gpu_style_crc(data: bytes, head: int, seglog: int, runs: int = 8) -> int:
    """crc32_ranges for one range: head bytes, segments of 2^seglog blocks,
    per-thread runs folded then a pairwise tree, tail, init term."""
    n = len(data)
    body = data[head:]
    nblk = len(body) // 512
    segb = 1 << seglog
    nseg = (nblk + segb - 1) // segb
    seg = [segment_value(body[i * segb * 512: min((i + 1) * segb, nblk) * 512])
           for i in range(nseg)]
    per = 1
    while runs * per < nseg:
        per *= 2
    run = []
    for t in range(runs):
        v = 0
        for i in range(min(t * per, nseg), min(t * per + per, nseg)):
            nb = min(segb, nblk - i * segb)
            v = zshift(v, 512 * nb) ^ seg[i]
        run.append(v)
    full = per * segb
    w = 1
    while w < runs:
        for t in range(0, runs, 2 * w):
            if (t + w) * per < nseg:
                g0, g1 = (t + w) * full, min((t + 2 * w) * full, nblk)
                run[t] = zshift(run[t], 512 * (g1 - g0)) ^ run[t + w]
        w *= 2
    c = crc0(data[:head])
    c = zshift(c, 512 * nblk) ^ run[0]
    c = crc0(body[nblk * 512:], c)
    return c ^ zshift(0xFFFFFFFF, n) ^ 0xFFFFFFFF


@pytest.mark.parametrize("nbytes,head,seglog", [
    (512 * 8, 0, 3), (512 * 9 + 100, 0, 3), (512 * 11 + 7, 5, 3), (512 * 30 + 511, 11, 3),
    (512 * 3, 0, 3), (300, 0, 3), (0, 0, 3), (512 * 17, 15, 4)])
def test_gpu_crc_algebra_matches_zlib(nbytes, head, seglog):
    rng = np.random.default_rng(nbytes + head)
    data = rng.integers(0, 256, nbytes, dtype=np.uint8).tobytes()
    head = min(head, nbytes)
    assert gpu_style_crc(data, head, seglog) == zlib.crc32(data)
