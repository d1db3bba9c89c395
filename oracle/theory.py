"""Closed forms of the paper used as pins (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Eq.1 (§3.1): Omega(gamma, alpha) = (1 - alpha^(gamma+1)) / (1 - alpha),
the expected number of tokens one verification emits; alpha = 1 gives gamma + 1.
Accepted-count law ("follows a truncated geometric distribution"): with
per-position overlaps beta_i = sum_x min(p_i, q_i)(x),
  P(n = k) = prod_{i<k} beta_i * (1 - beta_k)  for k < gamma,  P(n = gamma) = prod_i beta_i.
"""
from __future__ import annotations

from fractions import Fraction


def omega(gamma: int, alpha):
    if alpha == 1:
        return gamma + 1
    return (1 - alpha ** (gamma + 1)) / (1 - alpha)


def accepted_count_pmf(betas):
    """P(n = k), k = 0..gamma, for per-position overlaps betas (length gamma)."""
    gamma = len(betas)
    pmf = []
    run = Fraction(1) if isinstance(betas[0], Fraction) else 1.0
    for k in range(gamma):
        pmf.append(run * (1 - betas[k]))
        run = run * betas[k]
    pmf.append(run)
    return pmf
