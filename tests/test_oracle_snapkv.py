"""Pins for the SnapKV selection and index-list draft attention oracle (
P:1141 SnapKV footnote: observation window 32, average pooling kernel 5)."""
import numpy as np

from oracle import attention as OA
from oracle import snapkv as SK
from synth import k_to_bf16_bits
from tests.helpers import AttnCase


def test_uniform_keys_give_closed_form_votes():
    """All keys equal: a[h,i,j] = 1 / (L-w+i+1), so vote[j] = g * sum_i 1/(L-w+i+1)."""
    g, w, L, d = 3, 4, 20, 8
    rng = np.random.default_rng(0)
    q = k_to_bf16_bits(rng.integers(-32, 32, size=(g, w, d)))
    k = np.tile(k_to_bf16_bits(rng.integers(-32, 32, size=(1, d))), (L, 1))
    vote = SK.snapkv_votes(q, k, L, w, 0.3)
    expect = g * sum(1.0 / (L - w + i + 1) for i in range(w))
    assert np.allclose(vote, expect, rtol=0, atol=1e-14)


def test_avg_pool_kernel5_closed_form():
    v = np.zeros(12)
    v[6] = 1.0
    assert np.array_equal(SK.avg_pool5(v), np.array([0, 0, 0, 0, .2, .2, .2, .2, .2, 0, 0, 0]))
    v = np.zeros(6)
    v[0] = 1.0                        # zero padding: counts the pad, divides by 5
    assert np.allclose(SK.avg_pool5(v), [.2, .2, .2, 0, 0, 0])
    assert np.allclose(SK.avg_pool5(np.ones(7)), [.6, .8, 1, 1, 1, .8, .6])


def test_topk_ties_take_lower_positions():
    pooled = SK.avg_pool5(np.ones(10))           # .6 .8 1 1 1 1 1 1 .8 .6
    assert SK.topk_positions(pooled, 4).tolist() == [2, 3, 4, 5]
    assert SK.topk_positions(pooled, 7).tolist() == [1, 2, 3, 4, 5, 6, 7]
    assert SK.topk_positions(pooled, 20).tolist() == list(range(10))


def test_needle_is_selected_with_its_pool_neighbourhood():
    """A key aligned with every window query dominates the votes: with budget-w = 5 the
    selection is exactly the needle and its +-2 pooling neighbourhood."""
    B, Hq, Hkv, d, L, w = 1, 4, 2, 16, 200, 8
    rng = np.random.default_rng(1)
    qk = rng.integers(-2, 3, size=(B, w, Hq, d))
    kk = rng.integers(-2, 3, size=(B, Hkv, L, d))
    direction = np.sign(rng.standard_normal(d)).astype(int)
    qk = qk + 20 * direction
    kk[0, :, 77] = 40 * direction
    idx, cnt, _ = SK.snapkv_select(k_to_bf16_bits(qk), k_to_bf16_bits(kk), np.array([L]), w, w + 5, 0.25)
    assert cnt[0] == 5
    for h in range(Hkv):
        assert idx[0, h].tolist() == [75, 76, 77, 78, 79]


def test_budget_covering_prompt_keeps_everything():
    case = AttnCase(2, 4, 2, 16, 64, [40, 25], seed=3)
    qo = k_to_bf16_bits(np.random.default_rng(2).integers(-32, 32, size=(2, 8, 4, 16)))
    idx, cnt, _ = SK.snapkv_select(qo, case.k_bits, np.array([40, 25]), 8, 64, 0.25)
    assert cnt.tolist() == [32, 17]
    assert idx[0, 0, :32].tolist() == list(range(32)) and idx[1, 1, :17].tolist() == list(range(17))


def test_group_head_order_does_not_matter():
    rng = np.random.default_rng(4)
    q = k_to_bf16_bits(rng.integers(-32, 32, size=(4, 6, 16)))
    k = k_to_bf16_bits(rng.integers(-32, 32, size=(90, 16)))
    v1 = SK.snapkv_votes(q, k, 90, 6, 0.25)
    v2 = SK.snapkv_votes(q[::-1], k, 90, 6, 0.25)
    assert np.max(np.abs(v1 - v2)) < 1e-13


def test_indexed_draft_reduces_to_streamingllm():
    """idx = sink rows, tail from n - window: the SnapKV draft set is StreamingLLM's J (O3)."""
    case = AttnCase(3, 8, 4, 64, 300, [300, 200, 120], seed=5)
    sink, window = 4, 60
    idx = np.tile(np.arange(sink, dtype=np.int32), (3, 4, 1))
    cnt = np.full(3, sink, np.int32)
    tail = case.kv_len - window
    o, l = SK.draft_attn_indexed(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, idx, cnt, tail, case.scale)
    ro, rl = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, sink, window, case.scale)
    assert np.array_equal(o, ro) and np.array_equal(l, rl)


def test_indexed_draft_with_full_prefix_is_full_attention():
    case = AttnCase(2, 8, 2, 64, 150, [150, 99], seed=6)
    tail = np.array([100, 50], np.int32)
    idx = np.full((2, 2, 100), -1, np.int32)
    for b in range(2):
        idx[b, :, :tail[b]] = np.arange(tail[b])
    o, l = SK.draft_attn_indexed(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, idx, tail, tail, case.scale)
    ro, rl = OA.verify_attn_full(case.qd_bits[:, None], case.k_bits, case.v_bits, case.kv_len, case.scale)
    assert np.array_equal(o, ro[:, 0]) and np.array_equal(l, rl[:, 0])


def test_per_sequence_budgets():
    """Heterogeneous batches: sequence b keeps min(clamp(budgets[b], w, budget) - w,
    L - w) positions.  Pinned by the needle case (exact set), by clamping at both ends, and by
    equality with the uniform-budget selection at each sequence's own budget."""
    B, Hq, Hkv, d, L, w = 3, 4, 2, 16, 200, 8
    rng = np.random.default_rng(1)
    qk = rng.integers(-2, 3, size=(B, w, Hq, d))
    kk = rng.integers(-2, 3, size=(B, Hkv, L, d))
    direction = np.sign(rng.standard_normal(d)).astype(int)
    qk = qk + 20 * direction
    kk[:, :, 77] = 40 * direction
    qb, kb = k_to_bf16_bits(qk), k_to_bf16_bits(kk)
    budget = w + 40
    idx, cnt, _ = SK.snapkv_select(qb, kb, np.full(B, L), w, budget, 0.25, budgets=np.array([w + 5, 3, 10 ** 6]))
    assert cnt.tolist() == [5, 0, 40]
    for h in range(Hkv):
        assert idx[0, h, :5].tolist() == [75, 76, 77, 78, 79]
        assert (idx[1, h] == -1).all()
    for b, bud in ((0, w + 5), (2, budget)):
        ref, rc, _ = SK.snapkv_select(qb[b:b + 1], kb[b:b + 1], np.array([L]), w, bud, 0.25)
        assert rc[0] == cnt[b]
        assert np.array_equal(ref[0, :, :rc[0]], idx[b, :, :cnt[b]])
