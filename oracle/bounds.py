"""Closed-form bounds of the paper (TEST INFRASTRUCTURE -- oracle).

Theorem 1: t <= 2 n^{1/log2((d+2)/(d+1))} M^{a_d k^{1/d} n^{1-1/d}},
a_d = c_d / [2 - 2((d+1)/(d+2))^{1-1/d}];  PST constant a_2' (l.109).
Returned as log2 values.
"""
from __future__ import annotations

import math

C_D = {1: 1.0, 2: 2.0, 3: 2.135, 4: 2.280, 5: 2.421}
C_PST = 1.971


def a_d(d: int) -> float:
    return C_D[d] / (2.0 - 2.0 * ((d + 1) / (d + 2)) ** (1.0 - 1.0 / d))


def a2_prime() -> float:
    return C_PST / (2.0 - 2.0 * math.sqrt(2.0 / 3.0))


def theorem1_log2(n: int, M: float, k: float, d: int = 2) -> float:
    return (1.0 + math.log2(n) / math.log2((d + 2) / (d + 1))
            + a_d(d) * k ** (1.0 / d) * n ** (1.0 - 1.0 / d) * math.log2(M))
