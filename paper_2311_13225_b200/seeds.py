"""Host-side splitmix64 stream derivation (planning only; scalar Python ints).

Same contract as the reference's ``derive_seed`` (kernels.py:61-70) and
``_mix64`` (kernels.py:51-55).  The device kernels use the identical finaliser
(csrc/hg_common.cuh); ``kernels.derive_seed`` routes through the C-ABI
(``hg_derive_seed``) and tests check both agree with the golden KATs.
"""

from __future__ import annotations

MASK = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
PHI = 0x2545F4914F6CDD1D


def mix64(x: int) -> int:
    x &= MASK
    x = ((x ^ (x >> 30)) * MIX1) & MASK
    x = ((x ^ (x >> 27)) * MIX2) & MASK
    return x ^ (x >> 31)


def derive_seed(seed: int, *parts: int) -> int:
    state = mix64((seed & MASK) + GOLDEN)
    for p in parts:
        state = mix64(((state + GOLDEN) & MASK) ^ (p & MASK))
    return state
