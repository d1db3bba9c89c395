"""O4: speculative-sampling acceptance (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

The paper uses the rule of Leviathan et al. ("As described in
[leviathan2022fast]") without restating it:

  for j = 0 .. gamma-1: accept draft token x = d_j with probability min(1, p_j(x) / q_j(x));
  at the first rejection j = n, emit a token drawn from norm(max(0, p_n - q_n));
  if all gamma are accepted, emit a bonus token drawn from p_gamma.

Readings where the paper is silent:
  * the accept test uses a 29-bit uniform m = rnd[b][j] >> 3 and is decided
    exactly in fp64:   accept  iff  m * q(x) < p(x) * 2^29   (both products exact);
  * the residual is formed on an integer grid: P_i = floor(p_i 2^40),
    Q_i = floor(q_i 2^40), W_i = max(0, P_i - Q_i); if sum W = 0, W = P; if that is
    also 0 (an invalid all-tiny row), the token is the lowest-index argmax of p;
  * the final draw uses a dedicated 64-bit uniform u = rnd[γ] << 32 | rnd[γ+1]:
    t = floor(u * sum W / 2^64), token = min{k : sum_{i<=k} W_i > t};
  * GREEDY (the paper's experiments decode greedily): accept iff
    argmax p_j == d_j (lowest index on ties); emit argmax p_n.

Outputs per sequence: tokens [d_0 .. d_{n-1}, new, -1 ...] (length gamma+1),
num_accepted = n, committed_len += n + 1.
"""
from __future__ import annotations

import numpy as np

TWO29 = float(1 << 29)
TWO40 = float(1 << 40)


def accept_test(m: int, p_x: float, q_x: float) -> bool:
    """m * q(x) < p(x) * 2^29 in fp64; m < 2^29 and fp32 q give a product with <= 53
    significant bits, and the power-of-two scale of p is exact, so no rounding occurs."""
    return float(m) * float(q_x) < float(p_x) * TWO29


def grid40(row: np.ndarray) -> np.ndarray:
    """floor(x * 2^40) as uint64 for fp32 x in [0, 1] (exact: power-of-two scale, then truncate)."""
    return np.floor(row.astype(np.float64) * TWO40).astype(np.uint64)


def argmax_lowest(row: np.ndarray) -> int:
    return int(np.argmax(row))            # numpy returns the first (lowest-index) maximum


def draw_from_weights(W: np.ndarray, u64: int) -> int:
    """token = min{k : sum_{i<=k} W_i > floor(u64 * sum W / 2^64)} (exact integers)."""
    total = int(W.sum(dtype=np.uint64))
    t = (int(u64) * total) >> 64
    cdf = np.cumsum(W, dtype=np.uint64)
    return int(np.searchsorted(cdf, np.uint64(t), side="right"))


def final_token(p_row: np.ndarray, q_row, u64: int) -> int:
    """Residual draw (q_row given) or bonus draw from p (q_row None)."""
    P = grid40(p_row)
    if q_row is not None:
        Q = grid40(q_row)
        W = np.where(P > Q, P - Q, np.uint64(0))
        if int(W.sum(dtype=np.uint64)) == 0:
            W = P                                   # degenerate residual: fall back to p
    else:
        W = P
    if int(W.sum(dtype=np.uint64)) == 0:
        return argmax_lowest(p_row)                 # invalid all-tiny row
    return draw_from_weights(W, u64)


def spec_accept_sample_one(p, q, d, rnd):
    """One sequence, SAMPLE mode.  p [gamma+1, V], q [gamma, V] fp32, d [gamma], rnd [gamma+2] uint32."""
    gamma = len(d)
    u64 = (int(rnd[gamma]) << 32) | int(rnd[gamma + 1])
    for j in range(gamma):
        x = int(d[j])
        m = int(rnd[j]) >> 3
        if not accept_test(m, p[j, x], q[j, x]):
            return j, final_token(p[j], q[j], u64)
    return gamma, final_token(p[gamma], None, u64)


def spec_accept_greedy_one(p, d):
    gamma = len(d)
    for j in range(gamma):
        if argmax_lowest(p[j]) != int(d[j]):
            return j, argmax_lowest(p[j])
    return gamma, argmax_lowest(p[gamma])


def spec_accept(p, q, d, rnd, mode: str = "sample", committed_len=None):
    """Batched O4.  p [B, gamma+1, V], q [B, gamma, V] fp32, d [B, gamma] int32,
    rnd [B, gamma+2] uint32 -> (out_tokens [B, gamma+1] int32 (-1 padded),
    num_accepted [B] int32, committed_len + n + 1 or None)."""
    B, gamma = d.shape[0], d.shape[1]
    out = np.full((B, gamma + 1), -1, dtype=np.int32)
    nacc = np.zeros(B, dtype=np.int32)
    for b in range(B):
        if mode == "sample":
            n, tok = spec_accept_sample_one(p[b], q[b], d[b], rnd[b])
        else:
            n, tok = spec_accept_greedy_one(p[b], d[b])
        out[b, :n] = d[b, :n]
        out[b, n] = tok
        nacc[b] = n
    new_len = None if committed_len is None else (np.asarray(committed_len) + nacc + 1).astype(np.int32)
    return out, nacc, new_len
