"""Pins for the tree-speculation oracle (oracle/tree.py)."""
from fractions import Fraction

import numpy as np
import torch

from oracle import accept as ACC
from oracle import attention as OA
from oracle import tree as TR
from tests.helpers import AttnCase
from tests.test_oracle_accept import dyadic_rows


def test_chain_mask_equals_causal_verify():
    case = AttnCase(2, 8, 2, 64, 120, [120, 77], T=5, seed=1)
    mask = np.tile(TR.chain_mask(5), (2, 1))
    o, l = TR.verify_attn_tree(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, mask, case.scale)
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    assert np.array_equal(o, ro) and np.array_equal(l, rl)


def test_tree_mask_matches_torch_sdpa():
    B, T, Hq, Hkv, d, cap = 2, 6, 4, 2, 32, 60
    case = AttnCase(B, Hq, Hkv, d, cap, [60, 31], T=T, seed=2)
    parents = [[-1, 0, 0, 1, 1, 2], [-1, 0, 1, 0, 3, 3]]
    mask = np.stack([TR.tree_mask_from_parents(pp) for pp in parents])
    o, _ = TR.verify_attn_tree(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, mask, case.scale)
    from synth import bf16_bits_to_f32
    q = torch.tensor(bf16_bits_to_f32(case.qv_bits).astype(np.float64))
    k = torch.tensor(bf16_bits_to_f32(case.k_bits).astype(np.float64))
    v = torch.tensor(bf16_bits_to_f32(case.v_bits).astype(np.float64))
    for b in range(B):
        n = int(case.kv_len[b])
        allowed = torch.zeros(T, n, dtype=torch.bool)
        allowed[:, : n - T] = True
        for t in range(T):
            for j in range(T):
                if (int(mask[b, t]) >> j) & 1:
                    allowed[t, n - T + j] = True
        kk = k[b, :, :n].repeat_interleave(Hq // Hkv, 0)
        vv = v[b, :, :n].repeat_interleave(Hq // Hkv, 0)
        with torch.nn.attention.sdpa_kernel(torch.nn.attention.SDPBackend.MATH):
            ref = torch.nn.functional.scaled_dot_product_attention(q[b].transpose(0, 1), kk, vv, attn_mask=allowed,
                                                                   scale=case.scale)
        assert np.max(np.abs(o[b] - ref.transpose(0, 1).numpy())) < 1e-12


def test_tree_mask_from_parents():
    m = TR.tree_mask_from_parents([-1, 0, 0, 1, 2])
    assert m.tolist() == [0b1, 0b11, 0b101, 0b1011, 0b10101]


def test_chain_tree_acceptance_equals_chain_rule():
    rng = np.random.default_rng(3)
    B, gamma, V = 24, 4, 40
    import synth as S
    p, q, d = S.spec_probs(7, B, gamma, V, 0.8)
    rnd = rng.integers(0, 1 << 32, size=(B, gamma + 2), dtype=np.uint64).astype(np.uint32)
    T = gamma + 1
    tokens = np.concatenate([np.full((B, 1), 5, np.int32), d], 1)
    parent = np.tile(np.arange(-1, gamma, dtype=np.int32), (B, 1))
    qt = np.concatenate([q, np.zeros((B, 1, V), np.float32)], 1)      # q of the last node unused
    for mode in ("sample", "greedy"):
        out, n, nodes = TR.spec_accept_tree(p, qt, tokens, parent, rnd, mode)
        ro, rn, _ = ACC.spec_accept(p, q, d, rnd if mode == "sample" else None, mode)
        assert np.array_equal(out, ro) and np.array_equal(n, rn)
        for b in range(B):
            assert nodes[b, : n[b]].tolist() == list(range(1, n[b] + 1))


def _accept_count(fn):
    """# of m in [0, 2^29) accepted by a test monotone in m."""
    lo, hi = 0, 1 << 29
    while lo < hi:
        mid = (lo + hi) // 2
        if fn(mid):
            lo = mid + 1
        else:
            hi = mid
    return lo


def test_two_iid_siblings_are_lossless():
    """Root with two leaf children drawn i.i.d. from q: the law of the first emitted token of
    the oracle's accept_tree_one, measured exactly from its own decision boundaries in the
    uniforms (binary search on m1, m2 and the 64-bit draw), equals p within the grid error."""
    rng = np.random.default_rng(4)
    V = 4
    p_root = dyadic_rows(rng, 1, V)[0]
    q_root = dyadic_rows(rng, 1, V)[0]
    p = np.stack([p_root, dyadic_rows(rng, 1, V)[0], dyadic_rows(rng, 1, V)[0]])
    q = np.stack([q_root, q_root, q_root])
    parent = np.array([-1, 0, 0])
    top = (1 << 29) - 1

    def run(x1, x2, m1, m2, u):
        rnd = np.array([m1 << 3, m2 << 3, u >> 32, u & 0xFFFFFFFF], dtype=np.uint64).astype(np.uint32)
        path, tok = TR.accept_tree_one(p, q, np.array([0, x1, x2]), parent, rnd)
        return (path[0] if path else 0), tok

    law = [Fraction(0)] * V
    for x1 in range(V):
        for x2 in range(V):
            wq = Fraction(float(q_root[x1])) * Fraction(float(q_root[x2]))
            if wq == 0:
                continue
            c1 = _accept_count(lambda m: run(x1, x2, m, top, 0)[0] == 1)
            law[x1] += wq * Fraction(c1, 1 << 29)
            if c1 == 1 << 29:
                continue
            c2 = _accept_count(lambda m: run(x1, x2, top, m, 0)[0] == 2)
            rej1 = 1 - Fraction(c1, 1 << 29)
            law[x2] += wq * rej1 * Fraction(c2, 1 << 29)
            if c2 == 1 << 29:
                continue
            first = []
            for k in range(V + 1):          # first u with final token >= k (nondecreasing in u)
                lo, hi = 0, 1 << 64
                while lo < hi:
                    mid = (lo + hi) // 2
                    if run(x1, x2, top, top, mid)[1] >= k:
                        hi = mid
                    else:
                        lo = mid + 1
                first.append(lo)
            rej2 = 1 - Fraction(c2, 1 << 29)
            for y in range(V):
                law[y] += wq * rej1 * rej2 * Fraction(first[y + 1] - first[y], 1 << 64)
    assert sum(law) == 1
    err = max(abs(a - Fraction(float(b))) for a, b in zip(law, p_root))
    assert err < 1e-8, float(err)


def test_greedy_tree_follows_argmax_child():
    V = 6
    p = np.zeros((1, 4, V), np.float32)
    p[0, 0, 3] = 1.0          # root wants token 3
    p[0, 2, 1] = 1.0          # node 2 (token 3) wants 1
    p[0, 3, 5] = 1.0
    tokens = np.array([[9, 2, 3, 1]], np.int32)
    parent = np.array([[-1, 0, 0, 2]], np.int32)
    out, n, nodes = TR.spec_accept_tree(p, p, tokens, parent, None, "greedy")
    assert n[0] == 2 and out[0].tolist() == [3, 1, 5, -1] and nodes[0].tolist() == [2, 3, -1, -1]


def test_kv_compact_moves_path_rows():
    rng = np.random.default_rng(5)
    kc = rng.integers(0, 1 << 16, size=(2, 3, 30, 8)).astype(np.uint16)
    vc = rng.integers(0, 1 << 16, size=(2, 3, 30, 8)).astype(np.uint16)
    k0, v0 = kc.copy(), vc.copy()
    base = np.array([10, 20])
    nodes = np.array([[2, 5, 6, -1], [1, 3, -1, -1]])
    cnt = np.array([3, 2])
    TR.kv_compact(kc, vc, base, nodes, cnt)
    for b in range(2):
        for i in range(cnt[b]):
            assert np.array_equal(kc[b, :, base[b] + 1 + i], k0[b, :, base[b] + nodes[b, i]])
            assert np.array_equal(vc[b, :, base[b] + 1 + i], v0[b, :, base[b] + nodes[b, i]])
        assert np.array_equal(kc[b, :, : base[b] + 1], k0[b, :, : base[b] + 1])


# ---------------------------------------------------------------- exact law of the tree walk
# The law of the emitted tokens of oracle/tree.accept_tree_one, measured from the CODE's own
# decision boundaries: every accept test is monotone in its 29-bit word m (accept iff m is below
# a threshold), and the final draw is an inverse CDF, monotone in the 64-bit uniform u.  The
# explorer runs the code with the test words fixed one at a time: a word that changes nothing
# is not consumed on that branch (the walk has ended), otherwise its threshold c is found by
# binary search and both branches (accept: m = 0, prob c / 2^29; reject: m = 2^29 - 1) are
# explored.  At a leaf the final token's interval boundaries in u are found by binary search.
# Every probability is an exact rational.
TOP29 = (1 << 29) - 1


def _run_tree(p, q, tokens, parent, ms, u):
    T = len(tokens)
    words = [m << 3 for m in ms] + [TOP29 << 3] * (T - 1 - len(ms))
    rnd = np.array(words + [u >> 32, u & 0xFFFFFFFF], dtype=np.uint64).astype(np.uint32)
    path, tok = TR.accept_tree_one(p, q, np.asarray(tokens), np.asarray(parent), rnd)
    return tuple(int(tokens[c]) for c in path), tok


def _exact_emission_law(p, q, tokens, parent, V):
    """{emitted token tuple (accepted path tokens + new token): Fraction probability}."""
    T = len(tokens)
    law = {}

    def leaf(ms, w):
        first = []
        for k in range(V + 1):          # first u whose final token is >= k
            lo, hi = 0, 1 << 64
            while lo < hi:
                mid = (lo + hi) // 2
                if _run_tree(p, q, tokens, parent, ms, mid)[1] >= k:
                    hi = mid
                else:
                    lo = mid + 1
            first.append(lo)
        path = _run_tree(p, q, tokens, parent, ms, 0)[0]
        for y in range(V):
            if first[y + 1] > first[y]:
                key = path + (y,)
                law[key] = law.get(key, Fraction(0)) + w * Fraction(first[y + 1] - first[y], 1 << 64)

    def explore(ms, w):
        k = len(ms)
        if k == T - 1:
            return leaf(ms, w)
        lo_res = _run_tree(p, q, tokens, parent, ms + [0], 0)
        hi_res = _run_tree(p, q, tokens, parent, ms + [TOP29], 0)
        probe = [_run_tree(p, q, tokens, parent, ms + [0], u) for u in (1 << 62, 1 << 63, 3 << 62)]
        probe_hi = [_run_tree(p, q, tokens, parent, ms + [TOP29], u) for u in (1 << 62, 1 << 63, 3 << 62)]
        if lo_res == hi_res and probe == probe_hi:
            return leaf(ms, w)          # word k is not consumed on this branch
        lo, hi = 0, 1 << 29             # c = #m accepted = first m whose outcome equals m = TOP29's
        while lo < hi:
            mid = (lo + hi) // 2
            if _run_tree(p, q, tokens, parent, ms + [mid], 0)[0] == hi_res[0]:
                hi = mid
            else:
                lo = mid + 1
        c = lo
        if c > 0:
            explore(ms + [0], w * Fraction(c, 1 << 29))
        if c < 1 << 29:
            explore(ms + [TOP29], w * (1 - Fraction(c, 1 << 29)))

    explore([], Fraction(1))
    return law


def _drafts(q_rows_of_node, parent, V):
    """All draft token assignments of the non-root nodes (each drawn from q at its parent) with
    their exact probabilities."""
    T = len(parent)
    import itertools
    for combo in itertools.product(range(V), repeat=T - 1):
        toks = (0,) + combo
        w = Fraction(1)
        for t in range(1, T):
            w *= Fraction(float(q_rows_of_node[parent[t]][toks[t]]))
        if w:
            yield np.array(toks, np.int32), w


def test_three_iid_siblings_are_lossless():
    """Root with THREE leaf children drawn i.i.d. from q (two residual renormalisations, Z22): the
    law of the first emitted token, measured exactly from the code, equals p(root) within the
    grid error (3 tests x 2^-29 + renormalisation floors ~2^-40 per token)."""
    rng = np.random.default_rng(11)
    V = 3
    p_root, q_root = dyadic_rows(rng, 1, V)[0], dyadic_rows(rng, 1, V)[0]
    leaves = dyadic_rows(rng, 3, V)
    p = np.stack([p_root, *leaves])
    q = np.stack([q_root, q_root, q_root, q_root])
    parent = [-1, 0, 0, 0]
    first = [Fraction(0)] * V
    total = Fraction(0)
    for toks, w in _drafts(q, parent, V):
        for emitted, pr in _exact_emission_law(p, q, toks, parent, V).items():
            first[emitted[0]] += w * pr
            total += w * pr
    assert total == 1
    err = max(abs(a - Fraction(float(b))) for a, b in zip(first, p_root))
    assert err < 1e-7, float(err)
    # and it is not trivially p: the draft q differs from p at the root
    assert max(abs(float(a) - float(b)) for a, b in zip(p_root, q_root)) > 0.05


def test_two_level_tree_is_lossless():
    """Root -> {c1, c2} (i.i.d. from q0), c1 -> {c3, c4} (i.i.d. from q1), with targets that
    depend only on the depth (p0 at the root, p1 at depth 1, p2 at depth 2).  The joint law of
    the first three tokens of the output stream -- the step's emitted tokens, continued with fresh
    draws from the next positions' targets when the step emits fewer -- equals p0(y1) p1(y2)
    p2(y3) within the grid error: the walk down an accepted child, the residual draw after the
    siblings' rejections and the bonus draw at a leaf are all exact."""
    rng = np.random.default_rng(12)
    V = 3
    p0, p1, p2 = dyadic_rows(rng, 3, V)
    q0, q1 = dyadic_rows(rng, 2, V)
    targets = [p0, p1, p2]
    parent = [-1, 0, 0, 1, 1]
    p = np.stack([p0, p1, p1, p2, p2])         # p at node t = target at the next position
    q = np.stack([q0, q1, q1, q1, q1])         # q at node t = the draft law of t's children
    joint = {}
    import itertools
    for toks, w in _drafts(q, parent, V):
        for emitted, pr in _exact_emission_law(p, q, toks, parent, V).items():
            L = len(emitted)
            for tail in itertools.product(range(V), repeat=3 - L):  # fresh positions L .. 2
                f = Fraction(1)
                for i, y in enumerate(tail):
                    f *= Fraction(float(targets[L + i][y]))
                key = emitted[:3] + tail
                joint[key] = joint.get(key, Fraction(0)) + w * pr * f
    assert sum(joint.values()) == 1
    err = max(abs(joint.get(k, Fraction(0)) - Fraction(float(p0[k[0]])) * Fraction(float(p1[k[1]])) *
                  Fraction(float(p2[k[2]]))) for k in itertools.product(range(V), repeat=3))
    assert err < 1e-7, float(err)
    assert any(len(e) == 3 for e in _exact_emission_law(p, q, np.array([0, 0, 1, 0, 1], np.int32), parent, V))
