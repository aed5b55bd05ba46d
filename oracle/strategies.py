"""Relax-factor strategies of PAPER.md §5.2 -- TEST INFRASTRUCTURE ONLY (see
oracle/core.py header for who may import this).

* Fixed strategy (lines 256-258): omega constant; ``run_algorithm2(omega=w)``.
* Probabilistic strategy (lines 301-303, 322-325, 331): "a roulette wheel is
  used to choose omega ... P(0.5) = P(1.0) = 0.3, P(1.5) = P(2.0) = 0.2", one
  draw per iteration.  The paper does not name a random number
  generator (reading R20): both sides implement SplitMix64
  (Steele, Lea & Flood 2014) -- written here again from its definition, not
  shared with the library -- and map u = (z >> 11) * 2^-53 to omega by the
  cumulative probabilities 0.3, 0.6, 0.8 (R24).
* Enumerating strategy (lines 288-291): omega = argmin over {0, 0.5, ..., 9}
  of f((1 + w) X^{k+1} - w X^k); ties go to the smaller omega.
  Candidate 0 is X^{k+1} itself, so the chosen point never has a larger
  stress than X^{k+1} (the guard of lines 6-8 is implied).
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1

# the roulette wheel's sectors, in the paper's order
ROULETTE = ((0.5, 0.3), (1.0, 0.3), (1.5, 0.2), (2.0, 0.2))
# the enumerated relax factors 0, 0.5, ..., 9 (19 candidates)
ENUM_OMEGAS = tuple(0.5 * i for i in range(19))


class SplitMix64:
    """SplitMix64: state += 0x9E3779B97F4A7C15; z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9; z = (z ^ (z >> 27)) * 0x94D049BB133111EB;
    return z ^ (z >> 31) (all mod 2^64).  Python integers, no numpy wraparound."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        """53-bit uniform in [0, 1)."""
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)


def roulette(u: float) -> float:
    """The sector of P:325's wheel that u in [0, 1) falls in (cumulative order)."""
    acc = 0.0
    for w, p in ROULETTE:
        acc += p
        if u < acc:
            return w
    return ROULETTE[-1][0]


def probabilistic_omega_fn(seed: int):
    """omega_fn(it) for layout.run_algorithm2: one roulette draw per iteration."""
    rng = SplitMix64(seed)
    return lambda it: roulette(rng.uniform())


def enumerate_omega(prob, X_next: np.ndarray, X_prev: np.ndarray, omegas=ENUM_OMEGAS):
    """Lines 288-291: (omega*, f*, fs) with fs[c] = f((1+w_c) X^{k+1} - w_c X^k)
    and omega* the first (smallest) argmin."""
    fs = [prob.f((1.0 + w) * X_next - w * X_prev) for w in omegas]
    c = int(np.argmin(fs))  # first minimum: ties to the smaller omega
    return omegas[c], fs[c], fs
