"""TEST INFRASTRUCTURE ONLY — numpy restatement of the device ES generation (es.cuh).

Checker for `ls_es_*` / `es.optimize_device`: Philox4x32-10 (Salmon, Moraes,
Dror, Shaw, SC'11; pinned below by the Random123 known-answer vectors), the
Box-Muller pairing the device uses, and the reference's ES arithmetic:
ThetaEncoding.decode (ls/es.py:57-62), _shape_fitness (ls/es.py:65-71) and the
es_step update (ls/es.py:74-93), with scores from oracle/oracle.c.  Only tests/
import this module.
"""

from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)

# Random123 kat_vectors, philox4x32_10: (counter, key) -> output
PHILOX_KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 over uint32 arrays (or scalars); returns 4 uint64 arrays < 2^32."""
    c = [np.asarray(x, np.uint64) & MASK32 for x in (c0, c1, c2, c3)]
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for r in range(10):
        if r:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        n0 = (p1 >> np.uint64(32)) ^ c[1] ^ np.uint64(k0)
        n2 = (p0 >> np.uint64(32)) ^ c[3] ^ np.uint64(k1)
        c = [n0, p1 & MASK32, n2, p0 & MASK32]
    return c


def normals(seed: int, generation: int, population: int, dim: int) -> np.ndarray:
    """Noise [population, dim] of one generation: Philox block (member, pair, generation, 0)
    keyed by the 64-bit seed, Box-Muller on (u1 in (0, 1], u2 in [0, 1))."""
    out = np.zeros((population, dim), np.float64)
    i = np.arange(population, dtype=np.uint64)
    for q in range((dim + 1) // 2):
        c = philox4x32_10(i, q, generation, 0, seed & 0xFFFFFFFF, seed >> 32)
        a = ((c[1] << np.uint64(32)) | c[0]) >> np.uint64(11)
        b = ((c[3] << np.uint64(32)) | c[2]) >> np.uint64(11)
        u1 = (a + np.uint64(1)).astype(np.float64) * 2.0 ** -53
        u2 = b.astype(np.float64) * 2.0 ** -53
        rad = np.sqrt(-2.0 * np.log(u1))
        ang = 6.283185307179586 * u2
        out[:, 2 * q] = rad * np.cos(ang)
        if 2 * q + 1 < dim:
            out[:, 2 * q + 1] = rad * np.sin(ang)
    return out


def decode(theta: np.ndarray, sizes) -> np.ndarray:
    """ThetaEncoding.decode per row: clip(round_half_even(x), 0, n - 1) (ls/es.py:57-62)."""
    return np.clip(np.rint(np.asarray(theta, np.float64)), 0, np.asarray(sizes) - 1).astype(np.int64)


def shape_fitness(values: np.ndarray) -> np.ndarray:
    """Centred ranks on [-0.5, 0.5] (ls/es.py:65-71)."""
    n = len(values)
    if n == 1 or np.ptp(values) == 0:
        return np.zeros(n)
    order = np.argsort(np.argsort(values, kind="stable"), kind="stable")
    return order / (n - 1) - 0.5


def es_update(theta, alpha, sigma, population, values, noise, rank_normalize=True):
    """theta + alpha/(n*sigma) * (weights @ noise) (ls/es.py:90-93)."""
    weights = shape_fitness(values) if rank_normalize else values
    return theta + (alpha / (population * sigma)) * (weights @ noise)
