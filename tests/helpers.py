"""Host-side decoding helpers for tests (reference tableau.hpp:135-157 semantics)."""
import numpy as np


def geometry(n):
    k = (n + 63) // 64
    return k, 64 * k


def xz_bits(n, layout, x, z, g, q):
    k, npad = geometry(n)
    if layout == 0:
        j = g // 64 if g < n else k + (g - n) // 64
        b = g % 64 if g < n else (g - n) % 64
        w = q * 2 * k + j
        return (int(x[w]) >> b) & 1, (int(z[w]) >> b) & 1
    col = g if g < n else npad + (g - n)
    w = (q // 64) * 2 * npad + col
    return (int(x[w]) >> (q % 64)) & 1, (int(z[w]) >> (q % 64)) & 1


def sign_bit(n, s, g):
    k, _ = geometry(n)
    half, idx = (0, g) if g < n else (k, g - n)
    return (int(s[half + idx // 64]) >> (idx % 64)) & 1


def generator_str(n, layout, x, z, s, g):
    out = "-" if sign_bit(n, s, g) else "+"
    for q in range(n):
        xb, zb = xz_bits(n, layout, x, z, g, q)
        out += "IXZY"[xb + 2 * zb]
    return out


def set_bit(n, layout, plane, g, q, v=1):
    k, npad = geometry(n)
    if layout == 0:
        j = g // 64 if g < n else k + (g - n) // 64
        b = g % 64 if g < n else (g - n) % 64
        w = q * 2 * k + j
    else:
        col = g if g < n else npad + (g - n)
        w = (q // 64) * 2 * npad + col
        b = q % 64
    m = np.uint64(1) << np.uint64(b)
    plane[w] = (plane[w] | m) if v else (plane[w] & ~m)


def set_sign(n, s, g, v=1):
    k, _ = geometry(n)
    half, idx = (0, g) if g < n else (k, g - n)
    m = np.uint64(1) << np.uint64(idx % 64)
    s[half + idx // 64] = (s[half + idx // 64] | m) if v else (s[half + idx // 64] & ~m)


def empty(n):
    k, npad = geometry(n)
    return (np.zeros(npad * 2 * k, dtype=np.uint64), np.zeros(npad * 2 * k, dtype=np.uint64),
            np.zeros(2 * k, dtype=np.uint64))
