"""GPU parity of the tree-speculation calls vs oracle/tree.py.

md_verify_attn_tree: max-abs <= 2e-3 (out) / 1e-3 (lse) as every attention call, and
bit-identical to md_verify_attn_full for the chain mask (same kernel, same arithmetic).
md_spec_accept_tree and md_kv_compact: bit-exact.
"""
import numpy as np
import pytest
import torch

import paper_2408_11049_b200 as md
import synth as S
from oracle import accept as OACC
from oracle import philox as OPH
from oracle import tree as TR
from tests.helpers import AttnCase

pytestmark = pytest.mark.gpu

ATOL_O = 2e-3
ATOL_LSE = 1e-3


def random_parents(rng, B, T, shape="random"):
    par = np.zeros((B, T), np.int32)
    par[:, 0] = -1
    for b in range(B):
        for t in range(1, T):
            if shape == "chain":
                par[b, t] = t - 1
            elif shape == "star":
                par[b, t] = 0
            else:
                par[b, t] = rng.integers(0, t)
    return par


def _verify_tree(case, mask):
    B, T, Hq, d = case.B, case.T, case.Hq, case.d
    mkl = int(case.kv_len.max())
    out = torch.full((B, T, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, T, Hq), float("nan"), device="cuda")
    ws = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, case.Hkv, d, T, mkl)), dtype=torch.uint8, device="cuda")
    mt = torch.from_numpy(mask.astype(np.uint32).view(np.int32)).cuda()
    md.verify_attn_tree(case.qv, case.k, case.v, case.kv_len_t, mkl, mt, case.scale, out, lse, ws)
    torch.cuda.synchronize()
    return out.cpu().numpy(), lse.cpu().numpy()


TREE_CASES = [
    # name,             B, Hq, Hkv,  d,  T, lengths, shape
    ("llama_rows",      3, 32,  8, 128, 5, [300, 517, 64], "random"),
    ("llama_t8",        2, 32,  8, 128, 8, [700, 130], "random"),
    ("keys_g1",         3,  8,  8, 128, 8, [200, 333, 65], "random"),
    ("keys_g2_d64",     2,  8,  4,  64, 4, [129, 90], "star"),
    ("qwen_rows",       2, 28,  4, 128, 2, [400, 100], "random"),
    ("rows_t16",        2,  4,  4, 128, 16, [260, 77], "random"),
    ("tc_groups_t12",   2, 28,  4, 128, 12, [900, 140], "random"),  # 84 rows: tcgen05 row groups
    ("tc_groups_t16",   2, 32,  4, 128, 16, [700, 20], "star"),     # 128 rows
]


@pytest.mark.parametrize("name,B,Hq,Hkv,d,T,lens,shape", TREE_CASES)
def test_verify_tree_parity(name, B, Hq, Hkv, d, T, lens, shape):
    rng = np.random.default_rng(len(name) * 7 + T)
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, T=T, seed=11).to_cuda()
    par = random_parents(rng, B, T, shape)
    mask = np.stack([TR.tree_mask_from_parents(pp) for pp in par])
    got_o, got_l = _verify_tree(case, mask)
    ref_o, ref_l = TR.verify_attn_tree(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, mask, case.scale)
    assert np.all(np.isfinite(got_o)) and np.all(np.isfinite(got_l))
    eo, el = np.max(np.abs(got_o - ref_o)), np.max(np.abs(got_l - ref_l))
    assert eo <= ATOL_O and el <= ATOL_LSE, (eo, el)


def test_verify_tree_chain_mask_is_verify_full_bitwise():
    B, Hq, Hkv, d, T = 4, 32, 8, 128, 5
    case = AttnCase(B, Hq, Hkv, d, 1500, [1500, 1033, 700, 65], T=T, seed=3, regime=S.Regime("peaky")).to_cuda()
    mask = np.tile(TR.chain_mask(T), (B, 1))
    o_t, l_t = _verify_tree(case, mask)
    mkl = int(case.kv_len.max())
    out = torch.empty((B, T, Hq, d), device="cuda")
    lse = torch.empty((B, T, Hq), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, mkl), dtype=torch.uint8, device="cuda")
    md.verify_attn_full(case.qv, case.k, case.v, case.kv_len_t, mkl, case.scale, out, lse, ws)
    torch.cuda.synchronize()
    assert np.array_equal(o_t, out.cpu().numpy()) and np.array_equal(l_t, lse.cpu().numpy())


def tree_accept_inputs(seed, B, T, V, sigma, shape="random", distinct_siblings=False):
    """p, q [B, T, V] per node (synth.spec_probs rows), tokens drawn from q[parent] by a
    seeded numpy sampler (the drafter, upstream of acceptance), rnd via the Philox oracle."""
    rng = np.random.default_rng(seed)
    p_all, q_all, _ = S.spec_probs(seed, B, T, V, sigma)
    p, q = p_all[:, :T].copy(), q_all.copy()
    par = random_parents(rng, B, T, shape)
    tok = np.zeros((B, T), np.int32)
    for b in range(B):
        used = {}
        for t in range(1, T):
            w = q[b, par[b, t]].astype(np.float64)
            if distinct_siblings:
                for x in used.get(par[b, t], []):
                    w[x] = 0.0
            tok[b, t] = rng.choice(V, p=w / w.sum())
            used.setdefault(par[b, t], []).append(tok[b, t])
    rnd = OPH.philox_words(seed, 2, B, T + 1)
    return p, q, tok, par, rnd


def _run_tree_accept(p, q, tok, par, rnd, mode, committed=None):
    B, T, V = p.shape
    out = torch.empty((B, T), dtype=torch.int32, device="cuda")
    n = torch.empty(B, dtype=torch.int32, device="cuda")
    nodes = torch.empty((B, T), dtype=torch.int32, device="cuda")
    cl = None if committed is None else torch.from_numpy(committed.copy()).cuda()
    md.spec_accept_tree(torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda(), torch.from_numpy(tok).cuda(),
                        torch.from_numpy(par).cuda(), torch.from_numpy(rnd.view(np.int32)).cuda(), out, n, nodes, cl,
                        mode=mode)
    torch.cuda.synchronize()
    return out.cpu().numpy(), n.cpu().numpy(), nodes.cpu().numpy(), None if cl is None else cl.cpu().numpy()


@pytest.mark.parametrize("B,T,V,sigma,shape,distinct", [
    (64, 8, 1000, 1.0, "random", False),
    (32, 16, 5000, 2.5, "star", True),        # many siblings, deep residual histories
    (32, 16, 3000, 0.8, "random", True),
    (16, 6, 128256, 0.9, "random", False),
    (16, 5, 777, 0.5, "chain", False),
    (8, 1, 300, 0.0, "random", False),        # root only: a bonus draw from p
])
def test_spec_accept_tree_sample_bit_exact(B, T, V, sigma, shape, distinct):
    p, q, tok, par, rnd = tree_accept_inputs(B * 13 + T, B, T, V, sigma, shape, distinct)
    committed = np.arange(B, dtype=np.int32) + 50
    out, n, nodes, cl = _run_tree_accept(p, q, tok, par, rnd, "sample", committed)
    ro, rn, rnodes = TR.spec_accept_tree(p, q, tok, par, rnd, "sample")
    assert np.array_equal(out, ro) and np.array_equal(n, rn) and np.array_equal(nodes, rnodes)
    assert np.array_equal(cl, committed + rn + 1)


def test_spec_accept_tree_exercises_sibling_renormalisation():
    """Star trees.  First half of the batch: q lives on the first half of the vocabulary
    where p is small, so whole sibling sets get rejected (n = 0); second half: q mixes in
    p, tokens anywhere, so later siblings get accepted against renormalised residuals."""
    B, T, V = 24, 6, 64
    rng = np.random.default_rng(9)
    p = rng.random((B, T, V)).astype(np.float32)
    p[:, :, : V // 2] *= 0.05
    p /= p.sum(-1, keepdims=True)
    q = np.zeros((B, T, V), np.float32)
    q[:, :, : V // 2] = rng.random((B, T, V // 2)).astype(np.float32)
    q /= q.sum(-1, keepdims=True)
    q[B // 2:] = 0.8 * q[B // 2:] + 0.2 * p[B // 2:]
    q = q.astype(np.float32)
    par = random_parents(rng, B, T, "star")
    tok = rng.integers(0, V // 2, size=(B, T)).astype(np.int32)
    tok[B // 2:] = rng.integers(0, V, size=(B - B // 2, T))
    rnd = OPH.philox_words(77, 0, B, T + 1)
    out, n, nodes, _ = _run_tree_accept(p, q, tok, par, rnd, "sample")
    ro, rn, rnodes = TR.spec_accept_tree(p, q, tok, par, rnd, "sample")
    assert np.array_equal(out, ro) and np.array_equal(n, rn) and np.array_equal(nodes, rnodes)
    assert np.sum(rn) > 0 and np.sum(rn == 0) > 0   # both outcomes occur
    assert np.sum(rnodes[:, 0] > 2) > 0              # a third-or-later sibling accepted


@pytest.mark.parametrize("B,T,V", [(32, 8, 2000), (8, 16, 32000)])
def test_spec_accept_tree_greedy_bit_exact(B, T, V):
    p, q, tok, par, rnd = tree_accept_inputs(5 + T, B, T, V, 0.7)
    rng = np.random.default_rng(1)
    for b in range(B):                 # make some children carry the parent's argmax token
        for t in range(1, T):
            if rng.random() < 0.5:
                tok[b, t] = int(np.argmax(p[b, par[b, t]]))
    out, n, nodes, _ = _run_tree_accept(p, q, tok, par, rnd, "greedy")
    ro, rn, rnodes = TR.spec_accept_tree(p, q, tok, par, None, "greedy")
    assert np.array_equal(out, ro) and np.array_equal(n, rn) and np.array_equal(nodes, rnodes)


def test_spec_accept_tree_chain_equals_spec_accept():
    B, gamma, V = 32, 4, 4096
    p, q, d = S.spec_probs(21, B, gamma, V, 1.0)
    rnd = OPH.philox_words(21, 0, B, gamma + 2)
    T = gamma + 1
    tok = np.concatenate([np.zeros((B, 1), np.int32), d], 1)
    par = np.tile(np.arange(-1, gamma, dtype=np.int32), (B, 1))
    qt = np.concatenate([q, np.zeros((B, 1, V), np.float32)], 1)
    out, n, _, _ = _run_tree_accept(p, qt, tok, par, rnd, "sample")
    ro, rn, _ = OACC.spec_accept(p, q, d, rnd, "sample")
    assert np.array_equal(out, ro) and np.array_equal(n, rn)


def test_kv_compact_bit_exact():
    rng = np.random.default_rng(5)
    B, H, cap, d, T = 4, 8, 300, 128, 8
    kc = rng.integers(0, 1 << 16, size=(B, H, cap, d)).astype(np.uint16)
    vc = rng.integers(0, 1 << 16, size=(B, H, cap, d)).astype(np.uint16)
    base = np.array([10, 200, 0, 291], np.int32)
    nodes = np.full((B, T), -1, np.int32)
    cnt = np.array([3, 0, 7, 4], np.int32)
    paths = [[2, 5, 6], [], [1, 2, 3, 4, 5, 6, 7], [3, 4, 6, 7]]
    for b, pth in enumerate(paths):
        nodes[b, : len(pth)] = pth
    kt = torch.from_numpy(kc.view(np.int16)).view(torch.bfloat16).cuda()
    vt = torch.from_numpy(vc.view(np.int16)).view(torch.bfloat16).cuda()
    md.kv_compact(kt, vt, torch.from_numpy(base).cuda(), torch.from_numpy(nodes).cuda(), torch.from_numpy(cnt).cuda())
    torch.cuda.synchronize()
    TR.kv_compact(kc, vc, base, nodes, cnt)
    assert np.array_equal(kt.cpu().view(torch.int16).numpy().view(np.uint16), kc)
    assert np.array_equal(vt.cpu().view(torch.int16).numpy().view(np.uint16), vc)


def test_tree_step_end_to_end():
    """verify_attn_tree -> spec_accept_tree -> kv_compact on one batch, then a chain verify over
    the compacted cache equals the oracle's attention over the accepted path."""
    B, Hq, Hkv, d, T = 3, 16, 4, 128, 6
    lens = [400, 250, 90]
    case = AttnCase(B, Hq, Hkv, d, 420, lens, T=T, seed=5).to_cuda()
    rng = np.random.default_rng(2)
    par = random_parents(rng, B, T)
    mask = np.stack([TR.tree_mask_from_parents(pp) for pp in par])
    got_o, _ = _verify_tree(case, mask)
    ref_o, _ = TR.verify_attn_tree(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, mask, case.scale)
    assert np.max(np.abs(got_o - ref_o)) <= ATOL_O
    p, q, tok, _, rnd = tree_accept_inputs(3, B, T, 500, 0.6)
    out, n, nodes, _ = _run_tree_accept(p, q, tok, par, rnd, "sample")
    ro, rn, rnodes = TR.spec_accept_tree(p, q, tok, par, rnd, "sample")
    assert np.array_equal(nodes, rnodes)
    base = (case.kv_len - T).astype(np.int32)
    md.kv_compact(case.k, case.v, torch.from_numpy(base).cuda(), torch.from_numpy(nodes).cuda(),
                  torch.from_numpy(n).cuda())
    torch.cuda.synchronize()
    kc, vc = case.k_bits.copy(), case.v_bits.copy()
    TR.kv_compact(kc, vc, base, rnodes, rn)
    assert np.array_equal(case.k.cpu().view(torch.int16).numpy().view(np.uint16), kc)
    assert np.array_equal(case.v.cpu().view(torch.int16).numpy().view(np.uint16), vc)
