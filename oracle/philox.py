"""Philox4x32-10 counter-based RNG and the injected Gaussian noise (oracle side).

Test infrastructure only (see oracle/__init__.py).

The paper does not name its noise source; SURVEY.md §8(c) O4 / Q21 fixes a
counter layout so that the noise of entry (X, j) is independent of schedule,
batching and pipelining:  key = (seed lo32, seed hi32), counter = (X, j, e//4, 0)
for flat element e of the chunk [C, T', h, w]; Box–Muller in fp64 on the pair
(w0, w1) for e%4 in {0,1} and (w2, w3) for e%4 in {2,3}; cos for even e%4, sin
for odd.  Philox4x32-10 itself is Salmon et al. (Random123, SC'11), pinned by
its published known-answer vectors (tests/golden/philox_kat.txt).
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """ctr: 4 arrays (or scalars) of uint32; key: 2 uint32.  Returns 4 uint32 arrays."""
    c = [np.asarray(x, dtype=np.uint64) & MASK for x in ctr]
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return [x.astype(np.uint32) for x in c]


def gaussian_noise(seed: int, X: int, j: int, numel: int) -> np.ndarray:
    """eps_{X,j}[e], e = 0..numel-1, in fp64."""
    e = np.arange(numel, dtype=np.uint64)
    grp = e // np.uint64(4)
    q = (e % np.uint64(4)).astype(np.int64)
    w = philox4x32_10((np.full_like(grp, X), np.full_like(grp, j), grp, np.zeros_like(grp)),
                      (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF))
    first = np.where(q < 2, w[0], w[2]).astype(np.float64)
    second = np.where(q < 2, w[1], w[3]).astype(np.float64)
    u1 = (first + 0.5) * 2.0 ** -32
    u2 = (second + 0.5) * 2.0 ** -32
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * np.pi * u2
    return np.where(q % 2 == 0, rad * np.cos(ang), rad * np.sin(ang))
