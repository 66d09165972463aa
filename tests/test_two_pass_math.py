"""Host-side check of the two-pass long-fiber Thomas algebra
(paper_2105_12764_b200/csrc/thomas_2pass.cuh, tables built in csrc/mgrg.cu
upload_geometry): a fiber solved chunk by chunk from zero carries, the
chunk-level carry recurrences with the fiber-independent PF / Q / PB table
entries, and the chunk re-solve from the exact carries reproduce the plain
sequential sweeps of thomas_fiber (kernels.hpp:143-151).  numpy, float64."""
import numpy as np
import pytest


def _factors(h):
    """Thomas factors of a mass-matrix-shaped tridiagonal system (diagonal
    2(h_l + h_r), off-diagonal h: TridiagonalOperator::build, kernels.hpp:
    98-136, up to its constant scale): forward multipliers fwd, reciprocal
    pivots ip, backward multipliers g = -ip * h."""
    m = len(h) + 1
    diag = np.empty(m)
    diag[0] = 2 * h[0]
    diag[-1] = 2 * h[-1]
    diag[1:-1] = 2 * (h[:-1] + h[1:])
    off = h  # sub/super diagonal
    fwd = np.zeros(m)
    ip = np.empty(m)
    piv = diag[0]
    ip[0] = 1 / piv
    for i in range(1, m):
        fwd[i] = -off[i - 1] / piv
        piv = diag[i] + fwd[i] * off[i - 1]
        ip[i] = 1 / piv
    g = np.zeros(m)
    g[:-1] = -ip[:-1] * off
    return fwd, ip, g


def _sequential(f, fwd, ip, g):
    v = np.empty_like(f)
    acc = 0.0
    for i in range(len(f)):
        acc = f[i] + fwd[i] * acc
        v[i] = acc
    x = np.empty_like(f)
    z = 0.0
    for i in range(len(f) - 1, -1, -1):
        z = ip[i] * v[i] + g[i] * z
        x[i] = z
    return x


def _tables(fwd, ip, g, C):
    """Per chunk (PF, Q, PB) exactly as mgrg.cu builds them."""
    m = len(fwd)
    K = (m + C - 1) // C
    ck = np.zeros((K, 3))
    for k in range(K):
        a, b = k * C, min(m, k * C + C)
        pfi = np.cumprod(fwd[a:b])
        x = 0.0
        for j in range(b - 1, a - 1, -1):
            x = ip[j] * pfi[j - a] + (g[j] * x if j + 1 < b else 0.0)
        ck[k] = (pfi[-1], x, np.prod(g[a:b]))
    return ck


def _two_pass(f, fwd, ip, g, C):
    m = len(f)
    ck = _tables(fwd, ip, g, C)
    K = len(ck)
    E = np.empty(K)
    S = np.empty(K)
    for k in range(K):  # pass 1: zero carries
        a, b = k * C, min(m, k * C + C)
        acc, vl = 0.0, np.empty(b - a)
        for i in range(a, b):
            acc = f[i] + fwd[i] * acc
            vl[i - a] = acc
        E[k] = vl[-1]
        x = 0.0
        for i in range(b - 1, a - 1, -1):
            x = ip[i] * vl[i - a] + (g[i] * x if i + 1 < b else 0.0)
        S[k] = x
    c = np.empty(K)  # carry: forward then backward
    cin = 0.0
    for k in range(K):
        c[k] = cin
        cin = ck[k, 0] * cin + E[k]
    d = np.empty(K)
    din = 0.0
    for k in range(K - 1, -1, -1):
        d[k] = din
        din = ck[k, 2] * din + (S[k] + ck[k, 1] * c[k])
    out = np.empty(m)  # pass 2: re-solve from the exact carries
    for k in range(K):
        a, b = k * C, min(m, k * C + C)
        acc, v = c[k], np.empty(b - a)
        for i in range(a, b):
            acc = f[i] + fwd[i] * acc
            v[i - a] = acc
        x = d[k]
        for i in range(b - 1, a - 1, -1):
            x = ip[i] * v[i - a] + g[i] * x
            out[i] = x
    return out


@pytest.mark.parametrize("m,C", [(4097, 16), (4501, 16), (1025, 32), (37, 16), (16, 16), (17, 16)])
@pytest.mark.parametrize("uniform", [True, False])
def test_two_pass_equals_sequential(m, C, uniform):
    rng = np.random.default_rng(m * 31 + C + uniform)
    h = np.full(m - 1, 1.0 / (m - 1)) if uniform else rng.uniform(0.1, 1.0, m - 1)
    fwd, ip, g = _factors(h)
    f = rng.standard_normal(m)
    ref = _sequential(f, fwd, ip, g)
    got = _two_pass(f, fwd, ip, g, C)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
