"""Counter-based Gaussian sketch Omega -- TEST INFRASTRUCTURE ONLY.

Alg. 2 step 1 ("Omega ... i.i.d. standard normal"), one Omega for
every level k (eqn:Yk P:834-838, reading R8).  The method draws random numbers;
per the parity rules both sides implement the SAME counter-based generator
independently (this file shares no code with the CUDA path):

  * Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers:
    as easy as 1, 2, 3"): multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key
    increments 0x9E3779B9 / 0xBB67AE85, ten rounds, the key bumped after each.
  * counter of element e (column-major index e = row + col * N of the N x w
    sketch in TREE order) = (e mod 2^32, e >> 32, 0x5350, 0x48); key = the 64-bit
    seed split into (low, high) words  (reading R29).
  * Box-Muller on the first two 53-bit uniforms of the output block:
        u1 = (((c0 << 21) ^ c1) mod 2^53) 2^-53 + 2^-54     (in (0, 1))
        u2 = (((c2 << 21) ^ c3) mod 2^53) 2^-53             (in [0, 1))
        omega = sqrt(-2 ln u1) cos(2 pi u2).
Pinned by the Random123 known-answer vectors of Philox4x32-10 and by the
moments / Kolmogorov-Smirnov distance of N(0,1) (tests/test_oracle_omega.py).
"""
import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """ctr: 4 arrays (uint64 holding 32-bit words), key: 2 ints. Returns 4 arrays."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & MASK32 for c in ctr)
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    for _ in range(10):
        p0 = M0 * c0                       # < 2^64: exact in uint64
        p1 = M1 * c2
        h0, l0 = p0 >> np.uint64(32), p0 & MASK32
        h1, l1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (h1 ^ c1 ^ np.uint64(k0), l1, h0 ^ c3 ^ np.uint64(k1), l0)
        k0 = (k0 + W0) & 0xFFFFFFFF
        k1 = (k1 + W1) & 0xFFFFFFFF
    return c0, c1, c2, c3


def philox_normal(n, w, seed):
    """N x w column-major Gaussian sketch (tree order) of reading R29."""
    e = np.arange(int(n) * int(w), dtype=np.uint64)
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    c0, c1, c2, c3 = philox4x32_10((e & MASK32, e >> np.uint64(32),
                                    np.full_like(e, 0x5350), np.full_like(e, 0x48)),
                                   (seed & 0xFFFFFFFF, seed >> 32))
    m53 = np.uint64((1 << 53) - 1)
    u1 = (((c0 << np.uint64(21)) ^ c1) & m53).astype(np.float64) * 2.0 ** -53 + 2.0 ** -54
    u2 = (((c2 << np.uint64(21)) ^ c3) & m53).astype(np.float64) * 2.0 ** -53
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return z.reshape((int(n), int(w)), order="F")
