"""Exact rational output distributions of speculative sampling on tiny vocabularies
(TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).  Used by the O4 pins.

Two laws for ONE speculation block (gamma draft positions + one final token),
given per-position target rows p_0..p_gamma and draft rows q_0..q_{gamma-1}, with
each draft token d_j ~ q_j independently (prefix-independent arrays):

* `block_dist_ideal`  - Leviathan et al.'s rule (cited at P:204) in exact
  rationals: accept x w.p. min(1, p(x)/q(x)); on the first rejection emit
  norm(max(0, p - q)); after gamma acceptances emit a bonus token ~ p_gamma.
* `block_dist_discrete` - the law of the implemented integer rule (oracle/accept.py
  docstring) obtained by COUNTING the uniforms that produce each outcome:
    accept count  #{m < 2^29 : m q < p 2^29} = min(2^29, ceil(p 2^29 / q))  (q > 0),
    draw count    #{u < 2^64 : floor(u S / 2^64) in [C_{k-1}, C_k)}
                  = ceil(C_k 2^64 / S) - ceil(C_{k-1} 2^64 / S).
  The threshold pins in tests/test_oracle_accept.py check that the oracle's code
  flips exactly at these integer boundaries.

`joint_first_n` chains blocks along absolute positions and returns the joint law
of the first N emitted tokens; for the ideal rule it must equal prod_t p^(t)(y_t)
(SD is lossless).
"""
from __future__ import annotations

from fractions import Fraction
from math import ceil, floor

TWO29 = 1 << 29
TWO40 = 1 << 40
TWO64 = 1 << 64


def _F(x) -> Fraction:
    return x if isinstance(x, Fraction) else Fraction(float(x))


# ---------------------------------------------------------------- ideal rule
def _ideal_final(p, q):
    """Residual law norm(max(0, p - q)) (q given) or p itself (q None)."""
    if q is None:
        return [_F(x) for x in p]
    r = [max(Fraction(0), _F(a) - _F(b)) for a, b in zip(p, q)]
    s = sum(r)
    if s == 0:
        return [_F(x) for x in p]
    return [x / s for x in r]


def block_dist_ideal(p_rows, q_rows):
    gamma = len(q_rows)
    out = {}

    def rec(j, prefix, mass):
        if mass == 0:
            return
        if j == gamma:
            for y, w in enumerate(_ideal_final(p_rows[gamma], None)):
                if w:
                    out[prefix + (y,)] = out.get(prefix + (y,), 0) + mass * w
            return
        p, q = [_F(x) for x in p_rows[j]], [_F(x) for x in q_rows[j]]
        rej = Fraction(0)
        for x in range(len(p)):
            if q[x] == 0:
                continue
            a = min(Fraction(1), p[x] / q[x])
            rec(j + 1, prefix + (x,), mass * q[x] * a)
            rej += q[x] * (1 - a)
        if rej:
            for y, w in enumerate(_ideal_final(p_rows[j], q_rows[j])):
                if w:
                    out[prefix + (y,)] = out.get(prefix + (y,), 0) + mass * rej * w

    rec(0, (), Fraction(1))
    return out


# ---------------------------------------------------------------- implemented (discretised) rule
def accept_count(p_x, q_x) -> int:
    p, q = _F(p_x), _F(q_x)
    if q == 0:
        return TWO29 if p > 0 else 0
    return min(TWO29, ceil(p * TWO29 / q))


def grid40_exact(row):
    return [floor(_F(x) * TWO40) for x in row]


def discrete_final_weights(p_row, q_row):
    P = grid40_exact(p_row)
    if q_row is not None:
        Q = grid40_exact(q_row)
        W = [a - b if a > b else 0 for a, b in zip(P, Q)]
        if sum(W) == 0:
            W = P
    else:
        W = P
    return W


def draw_counts(W):
    """Number of 64-bit uniforms u mapping to each index under t = floor(u S / 2^64)."""
    S = sum(W)
    counts, c_prev, lo = [], 0, 0
    for w in W:
        c = c_prev + w
        hi = -((-c * TWO64) // S)          # ceil(c 2^64 / S)
        counts.append(hi - lo)
        lo, c_prev = hi, c
    return counts


def _discrete_final_law(p_row, q_row):
    W = discrete_final_weights(p_row, q_row)
    if sum(W) == 0:                         # invalid all-tiny row: lowest-index argmax of p
        vals = [_F(x) for x in p_row]
        k = vals.index(max(vals))
        return [Fraction(int(i == k)) for i in range(len(vals))]
    return [Fraction(c, TWO64) for c in draw_counts(W)]


def block_dist_discrete(p_rows, q_rows):
    gamma = len(q_rows)
    out = {}

    def rec(j, prefix, mass):
        if mass == 0:
            return
        if j == gamma:
            for y, w in enumerate(_discrete_final_law(p_rows[gamma], None)):
                if w:
                    out[prefix + (y,)] = out.get(prefix + (y,), 0) + mass * w
            return
        q = [_F(x) for x in q_rows[j]]
        rej = Fraction(0)
        for x in range(len(q)):
            if q[x] == 0:
                continue
            a = Fraction(accept_count(p_rows[j][x], q_rows[j][x]), TWO29)
            rec(j + 1, prefix + (x,), mass * q[x] * a)
            rej += q[x] * (1 - a)
        if rej:
            for y, w in enumerate(_discrete_final_law(p_rows[j], q_rows[j])):
                if w:
                    out[prefix + (y,)] = out.get(prefix + (y,), 0) + mass * rej * w

    rec(0, (), Fraction(1))
    return out


# ---------------------------------------------------------------- chaining blocks
def joint_first_n(block_fn, P, Q, gamma: int, N: int):
    """Joint law of the first N emitted tokens when block k starts at the absolute
    position where the previous one stopped.  P[t], Q[t] are the target / draft rows
    at absolute position t (prefix independent); P needs >= N + gamma rows."""
    cache = {}

    def block_at(s):
        if s not in cache:
            cache[s] = block_fn([P[s + i] for i in range(gamma + 1)], [Q[s + i] for i in range(gamma)])
        return cache[s]

    out = {}
    frontier = {(): Fraction(1)}
    while frontier:
        nxt = {}
        for prefix, mass in frontier.items():
            for blk, w in block_at(len(prefix)).items():
                seq = prefix + blk
                if len(seq) >= N:
                    key = seq[:N]
                    out[key] = out.get(key, 0) + mass * w
                else:
                    nxt[seq] = nxt.get(seq, 0) + mass * w
        frontier = nxt
    return out
