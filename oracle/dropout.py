"""Dropout with RNG replay (oracle) — TEST INFRASTRUCTURE ONLY.

The reference draws dropout masks from leantape.core.Rng (core.py:100-124):
numpy's Philox4x64-10 bit generator keyed [seed, stream], doubles from
``Generator.random()``; SPEC.md forward_dropout keeps an element when its
uniform is >= p and scales survivors by 1/(1-p) (SPEC.md DropoutConfig).  The
mask is a pure function of (seed, stream, p, numel), which is what lets the
MemSave variant keep only the key (saved.py:91-108).

``philox4x64_10`` restates the generator block function independently of
numpy (counter incremented before each block, so element i uses word i % 4 of
block i // 4 + 1); tests pin it against ``np.random.Philox`` itself.
``philox4x32_10`` restates the product's default (cheaper) generator, pinned
against the Random123 known-answer vectors.
"""

from __future__ import annotations

import numpy as np

_M0, _M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_W0, _W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
_MASK = (1 << 64) - 1


def philox4x64_10(ctr, key):
    """One Philox4x64-10 block (pure-Python loops: small cases only)."""
    c = [int(v) & _MASK for v in ctr]
    k0, k1 = int(key[0]) & _MASK, int(key[1]) & _MASK
    for r in range(10):
        if r:
            k0, k1 = (k0 + _W0) & _MASK, (k1 + _W1) & _MASK
        p0, p1 = _M0 * c[0], _M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k0, p1 & _MASK, (p0 >> 64) ^ c[3] ^ k1, p0 & _MASK]
    return c


def uniforms_restated(seed: int, stream: int, n: int) -> np.ndarray:
    """U_i = (word_i >> 11) * 2^-53 from the restated block function."""
    words = []
    for blk in range(1, (n + 3) // 4 + 1):
        words += philox4x64_10([blk, 0, 0, 0], [seed, stream])
    return np.array([(w >> 11) * 2.0 ** -53 for w in words[:n]], dtype=np.float64)


def uniforms(seed: int, stream: int, n: int) -> np.ndarray:
    """The reference generator itself: Rng(seed, stream).uniform((n,))."""
    return np.random.Generator(np.random.Philox(key=[seed, stream])).random(n)


def philox4x32_10(ctr, key):
    """Philox4x32-10 (Salmon et al. 2011, Random123), vectorised over blocks:
    ctr is a (4, B) uint64 array of 32-bit words, key a pair of 32-bit words."""
    m0, m1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
    w0, w1 = 0x9E3779B9, 0xBB67AE85
    lo32 = np.uint64(0xFFFFFFFF)
    c = [np.asarray(v, dtype=np.uint64) & lo32 for v in ctr]
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    for r in range(10):
        if r:
            k0, k1 = (k0 + w0) & 0xFFFFFFFF, (k1 + w1) & 0xFFFFFFFF
        p0, p1 = m0 * c[0], m1 * c[2]  # < 2^64: exact in uint64
        c = [(p1 >> np.uint64(32)) ^ c[1] ^ np.uint64(k0), p1 & lo32,
             (p0 >> np.uint64(32)) ^ c[3] ^ np.uint64(k1), p0 & lo32]
    return c


def words_philox4x32(seed: int, stream: int, n: int) -> np.ndarray:
    """The product's default generator (include/memsave_b200.h MS_RNG_PHILOX4X32):
    key = seed (lo, hi), counter = (j lo, j hi, stream lo, stream hi) for block j;
    element 4j + i takes word i."""
    nb = (n + 3) // 4
    j = np.arange(nb, dtype=np.uint64)
    lo32 = np.uint64(0xFFFFFFFF)
    ctr = [j & lo32, j >> np.uint64(32), np.full(nb, stream & 0xFFFFFFFF, np.uint64),
           np.full(nb, (stream >> 32) & 0xFFFFFFFF, np.uint64)]
    c = philox4x32_10(ctr, (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF))
    return np.stack(c, axis=1).reshape(-1)[:n]


def dropout_mask(seed: int, stream: int, p: float, n: int,
                 generator: str = "reference") -> np.ndarray:
    if generator == "reference":
        return uniforms(seed, stream, n) >= p
    import math
    return words_philox4x32(seed, stream, n) >= np.uint64(math.ceil(p * 2.0 ** 32))


def dropout_fwd(x, seed: int, stream: int, p: float, generator: str = "reference"):
    x = np.asarray(x, dtype=np.float64)
    m = dropout_mask(seed, stream, p, x.size, generator).reshape(x.shape)
    return np.where(m, x / (1.0 - p), 0.0), m


def dropout_bwd(g, seed: int, stream: int, p: float, generator: str = "reference"):
    """dX = G ⊙ mask / (1 − p) with the mask replayed from the key."""
    return dropout_fwd(g, seed, stream, p, generator)[0]
