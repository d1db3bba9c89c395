"""O5: Philox4x32-10 counter-based generator (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Salmon et al. (SC'11, "Parallel random numbers: as easy as 1, 2, 3"), written
out with Python integers.  Round: (hi0, lo0) = M0 * c0, (hi1, lo1) = M1 * c2,
c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); the key is bumped by the Weyl
constants between rounds.  Pinned by the published known-answer vectors
(tests/golden/philox_kat.json).

The stream layout used by `spec_accept` (reading Z8):
key = (seed_lo, seed_hi), counter = (b, step_lo, step_hi, block); the words of
sequence b are block 0's 4 outputs, then block 1's, ...; rnd[b][j] for j < gamma
are the accept tests and (rnd[b][gamma], rnd[b][gamma+1]) the 64-bit final draw.
"""
from __future__ import annotations

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    c0, c1, c2, c3 = (int(x) & MASK32 for x in ctr)
    k0, k1 = (int(x) & MASK32 for x in key)
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK32
        hi1, lo1 = p1 >> 32, p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return (c0, c1, c2, c3)


def philox_words(seed: int, step: int, B: int, words_per_seq: int) -> np.ndarray:
    """uint32 [B, words_per_seq] in the layout described above."""
    out = np.zeros((B, words_per_seq), dtype=np.uint32)
    key = (seed & MASK32, (seed >> 32) & MASK32)
    for b in range(B):
        for blk in range((words_per_seq + 3) // 4):
            r = philox4x32_10((b, step & MASK32, (step >> 32) & MASK32, blk), key)
            for i in range(4):
                w = 4 * blk + i
                if w < words_per_seq:
                    out[b, w] = r[i]
    return out
