"""Test infrastructure: a numpy model of the tensor path's number format
(paper_1009_0881_b200/csrc/ix_gemm.cu), used only as a checker.

Every fp32 row of M (a row for A = M W^T, a column for C = V^T M) is
scaled by 256 s, s = scale_of(row max) (the row maximum at [2^30, 2^31)),
and rounded to X = d1 2^24 + d2 2^16 + d3 2^8 + d4 (31-bit fixed point:
entries within 2^7 of the maximum are exact).  Every fp64 factor row (a row of W, a column of V) is scaled
by s_f = fscale_of(row max) and rounded to Y = e1 2^24 + e2 2^16 + e3 2^8 + e4
(31-bit).  The kernel forms the digit products d_i e_j of weight classes
c = i + j - 2 <= 3 (the rest are <= 2^-32 of the largest product), sums them
by class exactly in int32, and returns 2^16 (G0 2^24 + G1 2^16 + G2 2^8 +
G3) / (s s_f).  Here the integer sums are fp64 matrix products of small
integers (|sum| < 2^31, exact), combined in exact int64 and rounded once to
fp64, as the kernel does.  Model and kernel agree up to the fp64 rounding of
the kernel's split-K sum (~1e-16 relative).
"""
import numpy as np

XMAX = 8355711.0  # 2^23 - 0x8080 - 1


def scale_of(mx):
    mx = np.asarray(mx, np.float32).astype(np.float64)
    _, e = np.frexp(mx)
    k = np.clip(23 - e, -125, 125)
    s = np.ldexp(1.0, k)
    s = np.where(mx * s > XMAX, s * 0.5, s)
    return np.where(mx > 0, s, 1.0)


def fscale_of(mx):
    """factor scale: the fp64 row maximum rounded UP to fp32, then 2^(30 - e)"""
    mx = np.asarray(mx, np.float64)
    mx32 = mx.astype(np.float32).astype(np.float64)
    mx32 = np.where(mx32 < mx, np.nextafter(mx.astype(np.float32), np.float32(np.inf)).astype(np.float64), mx32)
    _, e = np.frexp(mx32)
    return np.where(mx > 0, np.ldexp(1.0, 30 - e), 1.0)


def digits(x, s):
    """four balanced digits of fp32 M entries on the 31-bit grid
    X = round(x 256 s) (half-even: the kernel's F2I; x 256 s is exact)"""
    X = np.rint(np.asarray(x, np.float32).astype(np.float64) * (256.0 * s))
    out = []
    for _ in range(3):
        d = np.mod(X + 128, 256) - 128
        out.append(d)
        X = (X - d) / 256
    out.append(X)
    return out[::-1]  # d1, d2, d3, d4


def fdigits(f, s):
    """four balanced digits of an fp64 factor row on its 31-bit grid"""
    X = np.rint(np.asarray(f, np.float64) * s)
    out = []
    for _ in range(3):
        d = np.mod(X + 128, 256) - 128
        out.append(d)
        X = (X - d) / 256
    out.append(X)
    return out[::-1]  # e1, e2, e3, e4


def _combine(a, b, sa, sb):
    """sum over the contraction of a (rows x K: three M digits) and b (K x
    cols: four factor digits)."""
    G = [np.zeros((a[0].shape[0], b[0].shape[1])) for _ in range(4)]
    for i in range(4):
        for j in range(4):
            if i + j <= 3:  # weight classes >= 4 (<= 2^-32 of the largest product) are not formed
                G[i + j] += a[i] @ b[j]
    G = [np.rint(g).astype(np.int64) for g in G]
    S = ((G[0] * 256 + G[1]) * 256 + G[2]) * 256 + G[3]
    return S.astype(np.float64) * 65536.0 / (sa[:, None] * sb[None, :])


def product_A(M, W):
    """A = M W^T (m x r) as the tensor path computes it (W fp64)."""
    M = np.asarray(M, np.float32)
    W = np.asarray(W, np.float64)
    sm = scale_of(M.max(axis=1))
    sw = fscale_of(W.max(axis=1))
    dm = digits(M, sm[:, None])
    dw = [d.T for d in fdigits(W, sw[:, None])]
    return _combine(dm, dw, sm, sw)


def product_C(V, M):
    """C = V^T M (r x n) as the tensor path computes it (V fp64)."""
    V = np.asarray(V, np.float64)
    M = np.asarray(M, np.float32)
    sv = fscale_of(V.max(axis=0))
    sm = scale_of(M.max(axis=0))
    dv = fdigits(V, sv[None, :])                # m x r each
    dm = [d.T for d in digits(M, sm[None, :])]  # n x m each
    return _combine(dm, dv, sm, sv).T           # (M^T V)^T


def gram_error(M, V, W):
    """||M - V W||_F through the Gram identity with the model's C."""
    M64, V64, W64 = (np.asarray(a, np.float32).astype(np.float64) for a in (M, V, W))
    C = product_C(V, M)
    e2 = (M64 * M64).sum() - 2.0 * (C * W64).sum() + ((V64.T @ V64) * (W64 @ W64.T)).sum()
    return float(np.sqrt(max(e2, 0.0)))
