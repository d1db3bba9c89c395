"""Pins for the oracle's speculative acceptance (O4), Philox (O5) and the Eq.1 closed forms.

* Philox: published known-answer vectors (tests/golden/philox_kat.json).
* Eq.1 / truncated-geometric PMF: worked values from SPEC.md S:156-158, S:441 (golden).
* The law of the oracle CODE is measured (binary search for the integer uniform where
  each decision flips) and compared, in exact rationals, with (a) the counting law
  of the stated integer rule and (b) Leviathan's ideal rule: the emitted
  token stream must follow the target distribution (SD is lossless).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import accept as ACC
from oracle import enumerate as EN
from oracle import philox as PH
from oracle import theory as TH

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ Philox
def test_philox_known_answer_vectors():
    g = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for vec in g["vectors"]:
        ctr = [int(x, 16) for x in vec["ctr"]]
        key = [int(x, 16) for x in vec["key"]]
        assert [f"0x{x:08x}" for x in PH.philox4x32_10(ctr, key)] == vec["out"]


def test_philox_words_layout():
    w = PH.philox_words(seed=0x1234_5678_9ABC, step=7, B=3, words_per_seq=6)
    for b in range(3):
        r0 = PH.philox4x32_10((b, 7, 0, 0), (0x5678_9ABC, 0x1234))
        r1 = PH.philox4x32_10((b, 7, 0, 1), (0x5678_9ABC, 0x1234))
        assert list(w[b]) == list(r0) + list(r1[:2])


# ------------------------------------------------------------------ Eq.1
def test_eq1_worked_values():
    g = json.load(open(os.path.join(GOLD, "eq1_examples.json")))
    for e in g["omega"]:
        assert abs(TH.omega(e["gamma"], e["alpha"]) - e["omega"]) < 1e-12
    pmf = TH.accepted_count_pmf([g["pmf"]["alpha"]] * g["pmf"]["gamma"])
    assert np.allclose(pmf, g["pmf"]["pmf"], atol=1e-12)
    # E[n + 1] under the truncated geometric law equals Eq.1
    assert abs(sum((k + 1) * w for k, w in enumerate(pmf)) - 2.952) < 1e-12


# ------------------------------------------------------------------ helpers: exact dyadic rows
def dyadic_rows(rng, n_rows, V, bits=20, zero_frac=0.0):
    """Rows of c_x / 2^bits with sum exactly 1 (exact in fp32 and in Fraction)."""
    rows = []
    for _ in range(n_rows):
        w = rng.random(V) ** 3
        if zero_frac:
            w[rng.random(V) < zero_frac] = 0.0
            if w.sum() == 0:
                w[0] = 1.0
        c = np.floor(w / w.sum() * (1 << bits)).astype(np.int64)
        c[np.argmax(c)] += (1 << bits) - c.sum()
        rows.append((c / float(1 << bits)).astype(np.float32))
    return np.array(rows)


def oracle_accept_count(p_x, q_x):
    """#m in [0, 2^29) the oracle's accept_test accepts (it is monotone in m)."""
    lo, hi = 0, 1 << 29
    while lo < hi:
        mid = (lo + hi) // 2
        if ACC.accept_test(mid, p_x, q_x):
            lo = mid + 1
        else:
            hi = mid
    # monotonicity spot check
    if lo > 0:
        assert ACC.accept_test(lo - 1, p_x, q_x)
    if lo < (1 << 29):
        assert not ACC.accept_test(lo, p_x, q_x)
    return lo


def oracle_final_law(p_row, q_row):
    """Law of oracle.accept.final_token over the 64-bit uniform, measured by binary search
    for the first u at which the returned token reaches each k (token is nondecreasing in u)."""
    V = len(p_row)
    tok = lambda u: ACC.final_token(p_row, q_row, u)
    first = []
    for k in range(V + 1):
        lo, hi = 0, 1 << 64
        while lo < hi:
            mid = (lo + hi) // 2
            if tok(mid) >= k:
                hi = mid
            else:
                lo = mid + 1
        first.append(lo)
    return [Fraction(first[k + 1] - first[k], 1 << 64) for k in range(V)]


def oracle_block_law(p_rows, q_rows):
    """Law of the oracle's one-sequence SAMPLE rule with d_j ~ q_j, assembled from the
    measured decision boundaries of the oracle code."""
    gamma = len(q_rows)
    out = {}

    def rec(j, prefix, mass):
        if mass == 0:
            return
        if j == gamma:
            for y, w in enumerate(oracle_final_law(p_rows[gamma], None)):
                if w:
                    out[prefix + (y,)] = out.get(prefix + (y,), 0) + mass * w
            return
        rej = Fraction(0)
        for x in range(len(q_rows[j])):
            qx = Fraction(float(q_rows[j][x]))
            if qx == 0:
                continue
            a = Fraction(oracle_accept_count(p_rows[j][x], q_rows[j][x]), 1 << 29)
            rec(j + 1, prefix + (x,), mass * qx * a)
            rej += qx * (1 - a)
        if rej:
            for y, w in enumerate(oracle_final_law(p_rows[j], q_rows[j])):
                if w:
                    out[prefix + (y,)] = out.get(prefix + (y,), 0) + mass * rej * w

    rec(0, (), Fraction(1))
    return out


def tv(a, b):
    keys = set(a) | set(b)
    return sum(abs(a.get(k, 0) - b.get(k, 0)) for k in keys) / 2


# ------------------------------------------------------------------ exact enumeration pins
def test_ideal_rule_is_lossless_single_position():
    rng = np.random.default_rng(0)
    p, q = dyadic_rows(rng, 2, 16), dyadic_rows(rng, 1, 16)
    law = EN.block_dist_ideal([p[0], p[1]], [q[0]])
    first = [sum((w for k, w in law.items() if k[0] == y), Fraction(0)) for y in range(16)]
    assert first == [Fraction(float(x)) for x in p[0]]


def test_ideal_rule_joint_first_n_equals_product_of_targets():
    rng = np.random.default_rng(1)
    gamma, V, N = 3, 8, 4
    P = dyadic_rows(rng, N + gamma + 1, V, zero_frac=0.2)
    Q = dyadic_rows(rng, N + gamma + 1, V, zero_frac=0.2)
    law = EN.joint_first_n(EN.block_dist_ideal, P, Q, gamma, N)
    assert sum(law.values()) == 1
    for y, w in law.items():
        expect = Fraction(1)
        for t, yt in enumerate(y):
            expect *= Fraction(float(P[t][yt]))
        assert w == expect


def test_oracle_code_law_equals_counting_law_and_is_near_lossless():
    rng = np.random.default_rng(2)
    gamma, V = 2, 6
    p = dyadic_rows(rng, gamma + 1, V, zero_frac=0.2)
    q = dyadic_rows(rng, gamma, V, zero_frac=0.2)
    measured = oracle_block_law(list(p), list(q))
    counted = EN.block_dist_discrete(list(p), list(q))
    assert measured == counted                       # the code implements the stated integer rule
    ideal = EN.block_dist_ideal(list(p), list(q))
    assert tv(counted, ideal) <= gamma * Fraction(1, 1 << 29) + V * Fraction(1, 1 << 64)


def test_discrete_joint_stream_close_to_target():
    rng = np.random.default_rng(3)
    gamma, V, N = 3, 5, 3
    P = dyadic_rows(rng, N + gamma + 1, V)
    Q = dyadic_rows(rng, N + gamma + 1, V)
    law = EN.joint_first_n(EN.block_dist_discrete, P, Q, gamma, N)
    target = {}
    for y in np.ndindex(*([V] * N)):
        w = Fraction(1)
        for t, yt in enumerate(y):
            w *= Fraction(float(P[t][yt]))
        if w:
            target[tuple(int(v) for v in y)] = w
    assert tv(law, target) <= N * (gamma * Fraction(1, 1 << 29) + V * Fraction(1, 1 << 64))


def test_accepted_count_law_is_product_of_overlaps():
    """P(n = k) = prod_{i<k} beta_i (1 - beta_k), beta = sum min(p, q)  (P:182 truncated geometric)."""
    rng = np.random.default_rng(4)
    gamma, V = 3, 6
    p = dyadic_rows(rng, gamma + 1, V)
    q = dyadic_rows(rng, gamma, V)
    law = EN.block_dist_ideal(list(p), list(q))
    betas = [sum(min(Fraction(float(a)), Fraction(float(b))) for a, b in zip(p[i], q[i])) for i in range(gamma)]
    pmf = TH.accepted_count_pmf(betas)
    got = [sum((w for k, w in law.items() if len(k) - 1 == n), Fraction(0)) for n in range(gamma + 1)]
    assert got == pmf


# ------------------------------------------------------------------ threshold / boundary pins
def test_accept_threshold_flips_at_exact_integer():
    rng = np.random.default_rng(5)
    for _ in range(200):
        p_x = np.float32(rng.random() ** 2)
        q_x = np.float32(rng.random() ** 2 + 1e-6)
        mstar = EN.accept_count(p_x, q_x)          # min(2^29, ceil(p 2^29 / q)) in exact rationals
        if mstar > 0:
            assert ACC.accept_test(mstar - 1, p_x, q_x)
        if mstar < (1 << 29):
            assert not ACC.accept_test(mstar, p_x, q_x)
    assert ACC.accept_test(0, np.float32(0.5), np.float32(0.0))       # q(x) = 0 < p(x): accept
    assert not ACC.accept_test(0, np.float32(0.0), np.float32(0.0))   # both 0: reject


def test_final_draw_boundaries():
    rng = np.random.default_rng(6)
    p = dyadic_rows(rng, 1, 7)[0]
    W = np.array(EN.grid40_exact(p), dtype=np.uint64)
    S, C = int(W.sum()), np.cumsum([int(x) for x in W])
    for k in range(7):
        if W[k] == 0:
            continue
        lo = -((-(int(C[k]) - int(W[k])) * (1 << 64)) // S)
        hi = -((-int(C[k]) * (1 << 64)) // S)
        assert ACC.draw_from_weights(W, lo) == k and ACC.draw_from_weights(W, hi - 1) == k


# ------------------------------------------------------------------ special cases
def _rnd(rng, B, gamma):
    return rng.integers(0, 1 << 32, size=(B, gamma + 2), dtype=np.uint64).astype(np.uint32)


def test_p_equals_q_accepts_everything():
    rng = np.random.default_rng(7)
    B, gamma, V = 64, 4, 50
    p = np.stack([dyadic_rows(rng, gamma + 1, V) for _ in range(B)])
    q = p[:, :gamma].copy()
    d = np.array([[rng.choice(V, p=p[b, j].astype(np.float64) / p[b, j].sum()) for j in range(gamma)] for b in range(B)])
    out, n, newlen = ACC.spec_accept(p, q, d.astype(np.int32), _rnd(rng, B, gamma), committed_len=np.full(B, 10))
    assert np.all(n == gamma) and np.array_equal(out[:, :gamma], d) and np.all(newlen == 10 + gamma + 1)


def test_disjoint_supports_reject_at_zero_and_draw_from_p():
    rng = np.random.default_rng(8)
    B, gamma, V = 32, 3, 20
    p = np.zeros((B, gamma + 1, V), np.float32)
    q = np.zeros((B, gamma, V), np.float32)
    p[:, :, :10] = 0.1
    q[:, :, 10:] = 0.1
    d = rng.integers(10, 20, size=(B, gamma)).astype(np.int32)
    out, n, _ = ACC.spec_accept(p, q, d, _rnd(rng, B, gamma))
    assert np.all(n == 0) and np.all(out[:, 0] < 10) and np.all(out[:, 1:] == -1)


def test_one_hot_sample_equals_greedy():
    rng = np.random.default_rng(9)
    B, gamma, V = 40, 4, 12
    hp = rng.integers(0, V, size=(B, gamma + 1))
    hq = np.where(rng.random((B, gamma)) < 0.7, hp[:, :gamma], rng.integers(0, V, size=(B, gamma)))
    p = np.eye(V, dtype=np.float32)[hp]
    q = np.eye(V, dtype=np.float32)[hq]
    d = hq.astype(np.int32)
    s = ACC.spec_accept(p, q, d, _rnd(rng, B, gamma), "sample")
    g = ACC.spec_accept(p, q, d, None, "greedy")
    assert np.array_equal(s[0], g[0]) and np.array_equal(s[1], g[1])


def test_gamma_zero_is_autoregressive_sampling():
    """gamma = 0: n = 0 and the token is the inverse-CDF draw of p_0 (plain AR decoding)."""
    rng = np.random.default_rng(10)
    V = 9
    p = dyadic_rows(rng, 1, V)[0]
    law = oracle_final_law(p, None)
    assert sum(abs(a - Fraction(float(b))) for a, b in zip(law, p)) <= V * Fraction(1, 1 << 64)
    rnd = _rnd(rng, 5, 0)
    out, n, _ = ACC.spec_accept(p[None, None].repeat(5, 0), np.zeros((5, 0, V), np.float32),
                                np.zeros((5, 0), np.int32), rnd)
    assert np.all(n == 0)
    for b in range(5):
        u = (int(rnd[b, 0]) << 32) | int(rnd[b, 1])
        assert out[b, 0] == ACC.draw_from_weights(ACC.grid40(p), u)


def test_greedy_ties_take_lowest_index():
    p = np.array([[[0.25, 0.25, 0.5, 0.0], [0.4, 0.1, 0.4, 0.1]]], np.float32)
    out, n, _ = ACC.spec_accept(p, np.zeros((1, 1, 4), np.float32), np.array([[2]], np.int32), None, "greedy")
    assert n[0] == 1 and out[0].tolist() == [2, 0]
    out, n, _ = ACC.spec_accept(p, np.zeros((1, 1, 4), np.float32), np.array([[1]], np.int32), None, "greedy")
    assert n[0] == 0 and out[0].tolist() == [2, -1]


def test_residual_zero_falls_back_to_p():
    """p_j(x) < q_j(x) can reject even when p == q elsewhere; residual sum 0 only if p <= q
    everywhere on the 2^-40 grid: then the draw falls back to p (reading Z7)."""
    p = np.array([0.5, 0.5, 0.0], np.float32)
    q = np.array([0.5, 0.5, 0.0], np.float32)
    W = ACC.grid40(p)
    for u in [0, 1 << 63, (1 << 64) - 1]:
        assert ACC.final_token(p, q, u) == ACC.draw_from_weights(W, u)
    tiny = np.array([1e-13, 0.0, 2e-13], np.float32)       # all below 2^-40: argmax fallback
    assert ACC.final_token(tiny, None, 123) == 2
