"""Philox4x32-10 counter-based generator and the RStS index-set sampler (oracle side).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this module.
The CUDA path implements the same published algorithm independently
(``paper_2305_09044_b200/csrc/sampler.cu``); the two share no code.

Paper passages:
  * PAPER.md:229 (Sec. 4.3) "we randomly and uniformly select s_k lateral slices of Z_k".
  * PAPER.md:268 (Alg. 1 line 4) "Randomly generate index set I_i ... set I_k = {1..I_k}".
The paper does not say how the uniform selection is drawn; reading R11 fixes it:
sampling without replacement, keys from Philox4x32-10 (Salmon et al., SC'11) with
key = (seed lo32, seed hi32) and counter = (i, m, k, t); the s_m indices with the smallest
(key, i) pairs are selected and returned in ascending order.
"""
import numpy as np

# Philox4x32 round constants (multipliers) and Weyl key increments (Salmon et al. 2011).
PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = np.uint64(0x9E3779B9)
PHILOX_W1 = np.uint64(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox4x32 rounds on uint32 counter words (numpy arrays, broadcastable).

    One round: p0 = M0*c0, p1 = M1*c2 (64-bit products);
    (c0,c1,c2,c3) <- (hi(p1)^c1^k0, lo(p1), hi(p0)^c3^k1, lo(p0)); then the key is
    bumped by (W0, W1) mod 2^32 before the next round.
    Returns the four output words as uint64 arrays holding 32-bit values.
    """
    c0 = np.asarray(c0, dtype=np.uint64) & _MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & _MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & _MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & _MASK32
    k0 = np.uint64(int(k0) & 0xFFFFFFFF)
    k1 = np.uint64(int(k1) & 0xFFFFFFFF)
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + PHILOX_W0) & _MASK32
            k1 = (k1 + PHILOX_W1) & _MASK32
        p0 = PHILOX_M0 * c0          # < 2^64, exact in uint64
        p1 = PHILOX_M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return c0, c1, c2, c3


def sample_keys(seed, t, k, m, I_m):
    """kappa_i = (out0 << 32) | out1 of Philox(key=seed, ctr=(i, m, k, t)), i in [0, I_m)."""
    i = np.arange(I_m, dtype=np.uint64)
    o0, o1, _, _ = philox4x32_10(i, m, k, t, int(seed) & 0xFFFFFFFF, (int(seed) >> 32) & 0xFFFFFFFF)
    return (o0 << np.uint64(32)) | o1


def sample_indices(seed, t, k, m, I_m, s_m):
    """RStS index set I_m for sweep t, block k (Alg. 1 line 4).

    Uniform without replacement: the s_m indices with the smallest (kappa_i, i); ascending.
    s_m <= 0 or s_m >= I_m means the full index set (no RNG draw).
    """
    if s_m <= 0 or s_m >= I_m:
        return np.arange(I_m, dtype=np.int64)
    kappa = sample_keys(seed, t, k, m, I_m)
    order = np.lexsort((np.arange(I_m), kappa))  # primary key kappa, tie-break on i
    return np.sort(order[:s_m]).astype(np.int64)
