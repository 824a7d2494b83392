"""Test infrastructure: a numpy model of the tensor path's number format
(paper_1009_0881_b200/csrc/ix_gemm.cu), used only as a checker.

Every fp32 operand row (a row of M for A = M W^T, a column of M for
C = V^T M, a row of W / a column of V on the factor side) is scaled by the
power of two s = scale_of(row max), rounded once to the nearest integer X
(round-half-even, as the kernel's single FFMA), and split into balanced
base-256 digits X = d1 2^16 + d2 2^8 + d3.  The kernel accumulates
    G0 = sum d1 e1,  G1 = sum d1 e2 + d2 e1,  G2 = sum d1 e3 + d2 e2 + d3 e1
exactly in int32 and returns 2^16 (G0 2^16 + G1 2^8 + G2) / (s_x s_f).  The
integer sums here are fp64 matrix products of small integers (|sum| < 2^31),
so they are exact too: the model and the kernel agree up to the fp64
rounding of the kernel's split-K sum (~1e-16 relative).
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


def digits(x, s):
    X = np.rint(np.asarray(x, np.float32).astype(np.float64) * s)
    d3 = np.mod(X + 128, 256) - 128
    Xp = (X - d3) / 256
    d2 = np.mod(Xp + 128, 256) - 128
    d1 = (Xp - d2) / 256
    return d1, d2, d3


def _combine(a, b, sa, sb):
    """sum over the contraction of a (rows x K digits) and b (K x cols digits)."""
    a1, a2, a3 = a
    b1, b2, b3 = b
    G0 = a1 @ b1
    G1 = a1 @ b2 + a2 @ b1
    G2 = a1 @ b3 + a2 @ b2 + a3 @ b1
    S = G0 * 65536.0 + G1 * 256.0 + G2
    return S * 65536.0 / (sa[:, None] * sb[None, :])


def product_A(M, W):
    """A = M W^T (m x r) as the tensor path computes it."""
    M = np.asarray(M, np.float32)
    W = np.asarray(W, np.float32)
    sm = scale_of(M.max(axis=1))
    sw = scale_of(W.max(axis=1))
    dm = digits(M, sm[:, None])
    dw = [d.T for d in digits(W, sw[:, None])]
    return _combine(dm, dw, sm, sw)


def product_C(V, M):
    """C = V^T M (r x n) as the tensor path computes it."""
    V = np.asarray(V, np.float32)
    M = np.asarray(M, np.float32)
    sv = scale_of(V.max(axis=0))
    sm = scale_of(M.max(axis=0))
    dv = [d.T for d in digits(V, sv[None, :])]
    dm = digits(M, sm[None, :])
    return _combine(dv, dm, sv, sm)


def gram_error(M, V, W):
    """||M - V W||_F through the Gram identity with the model's C."""
    M64, V64, W64 = (np.asarray(a, np.float32).astype(np.float64) for a in (M, V, W))
    C = product_C(V, M)
    e2 = (M64 * M64).sum() - 2.0 * (C * W64).sum() + ((V64.T @ V64) * (W64 @ W64.T)).sum()
    return float(np.sqrt(max(e2, 0.0)))
