"""GPU parity of md_draft_attn_indexed (SnapKV index-list drafting) against
the fp64 oracle (oracle/snapkv.py).  Index lists are seeded inputs (sorted random subsets of
the prefix), and, for a small case, the oracle's own SnapKV selection."""
import numpy as np
import pytest
import torch

import paper_2408_11049_b200 as md
from oracle import snapkv as SK
from synth import k_to_bf16_bits
from tests.helpers import AttnCase, bits_to_torch_bf16

pytestmark = pytest.mark.gpu
ATOL_O, ATOL_LSE = 2e-3, 1e-3


def _random_lists(rng, B, Hkv, stride, counts, tails):
    idx = np.full((B, Hkv, stride), -1, np.int32)
    for b in range(B):
        for h in range(Hkv):
            c = int(counts[b])
            idx[b, h, :c] = np.sort(rng.choice(int(tails[b]), size=c, replace=False))
    return idx


def _run(case, idx, counts, tails):
    B, Hq, d = case.B, case.Hq, case.d
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, Hq), float("nan"), device="cuda")
    ws = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, case.Hkv, d, 1, case.cap)), dtype=torch.uint8,
                     device="cuda")
    md.draft_attn_indexed(case.qd, case.k, case.v, case.kv_len_t, torch.from_numpy(idx).cuda(),
                          torch.from_numpy(counts).cuda(), torch.from_numpy(tails).cuda(), case.scale, out, lse, ws)
    torch.cuda.synchronize()
    return out.cpu().numpy(), lse.cpu().numpy()


@pytest.mark.parametrize("B,Hq,Hkv,d,lens,counts,stride,win", [
    (3, 32, 8, 128, [3000, 2000, 700], [500, 130, 0], 512, 32),
    (2, 28, 4, 128, [5000, 4100], [2017, 2017], 2020, 32),
    (4, 8, 8, 64, [300, 200, 150, 90], [61, 64, 65, 3], 68, 7),
    (2, 4, 1, 128, [9000, 40], [1000, 8], 1000, 40),          # tail empty for b=1 (n == tail_start)
])
def test_indexed_draft_parity(B, Hq, Hkv, d, lens, counts, stride, win):
    rng = np.random.default_rng(sum(lens))
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, seed=B * 7 + Hq).to_cuda()
    tails = (np.asarray(lens) - win).astype(np.int32)
    counts = np.minimum(np.asarray(counts), tails).astype(np.int32)
    idx = _random_lists(rng, B, Hkv, stride, counts, tails)
    o, l = _run(case, idx, counts, tails)
    ro, rl = SK.draft_attn_indexed(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, idx, counts, tails, case.scale)
    assert np.all(np.isfinite(o)) and np.max(np.abs(o - ro)) <= ATOL_O and np.max(np.abs(l - rl)) <= ATOL_LSE


def test_indexed_draft_with_oracle_snapkv_selection():
    """End to end on a small prompt: the oracle selects (S1-S4), the GPU drafts over it."""
    B, Hq, Hkv, d, L, w, budget = 2, 8, 2, 64, 700, 32, 160
    case = AttnCase(B, Hq, Hkv, d, L + 8, [L + 3, L + 1], seed=11).to_cuda()
    rng = np.random.default_rng(12)
    q_obs = k_to_bf16_bits(rng.integers(-32, 32, size=(B, w, Hq, d)))
    idx, cnt, _ = SK.snapkv_select(q_obs, case.k_bits, np.array([L, L]), w, budget, case.scale)
    idx = np.ascontiguousarray(np.pad(idx, ((0, 0), (0, 0), (0, (-idx.shape[2]) % 4)), constant_values=-1))
    tails = np.array([L - w, L - w], np.int32)
    o, l = _run(case, idx, cnt, tails)
    ro, rl = SK.draft_attn_indexed(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, idx, cnt, tails, case.scale)
    assert np.max(np.abs(o - ro)) <= ATOL_O and np.max(np.abs(l - rl)) <= ATOL_LSE


def test_indexed_equals_streaming_draft_on_gpu():
    """idx = sink rows, tail = n - window: the two draft calls walk the same logical keys in the
    same tiles, so their outputs agree bit for bit."""
    case = AttnCase(4, 32, 8, 128, 3100, [3000, 2000, 1500, 1100], seed=13).to_cuda()
    sink, window = 4, 1020
    idx = np.tile(np.arange(4, dtype=np.int32), (4, 8, 1))
    cnt = np.full(4, sink, np.int32)
    tails = (case.kv_len - window).astype(np.int32)
    o, l = _run(case, idx, cnt, tails)
    out = torch.empty((4, 32, 128), device="cuda")
    lse = torch.empty((4, 32), device="cuda")
    ws = torch.zeros(max(1, md.attn_workspace_bytes(4, 32, 8, 128, 1, 1024)), dtype=torch.uint8, device="cuda")
    md.draft_attn_sparse(case.qd, case.k, case.v, case.kv_len_t, sink, window, case.scale, out, lse, ws)
    torch.cuda.synchronize()
    assert np.array_equal(o, out.cpu().numpy()) and np.array_equal(l, lse.cpu().numpy())


def _check_selection(idx_gpu, cnt_gpu, idx_ref, cnt_ref, pooled_ref, rel_tol=1e-4):
    """Same count; the selected sets are identical except for positions whose fp64 pooled
    scores tie the selection threshold within rel_tol (fp32 vs fp64 order near ties)."""
    assert np.array_equal(cnt_gpu, cnt_ref)
    B, Hkv = idx_ref.shape[:2]
    ndiff = 0
    for b in range(B):
        c = int(cnt_ref[b])
        for h in range(Hkv):
            g = idx_gpu[b, h, :c]
            r = idx_ref[b, h, :c]
            assert np.all(np.diff(g) > 0), "GPU selection must be strictly ascending"
            pooled = pooled_ref[b][h]
            if c == len(pooled):
                assert np.array_equal(g, r)
                continue
            thr = np.sort(pooled)[::-1][c - 1]
            diff = set(g.tolist()) ^ set(r.tolist())
            ndiff += len(diff)
            for x in diff:
                assert abs(pooled[x] - thr) <= rel_tol * pooled.max(), (b, h, x, pooled[x], thr)
    return ndiff


@pytest.mark.parametrize("B,Hq,Hkv,d,L,w,budget,regime", [
    (2, 8, 2, 128, [3000, 2100], 32, 256, "peaky"),
    (3, 32, 8, 128, [1500, 1400, 700], 32, 512, "flat"),
    (2, 28, 4, 128, [2500, 300], 32, 1024, "peaky"),          # short prompt: keep everything
    (2, 4, 4, 64, [900, 1000], 8, 100, "peaky"),
    (1, 32, 8, 128, [9100], 32, 512, "peaky"),                 # several 4096-key tcgen05 chunks
])
def test_snapkv_select_matches_oracle(B, Hq, Hkv, d, L, w, budget, regime):
    import synth as S
    reg = S.Regime(regime, sink=4, needle_period=97) if regime == "peaky" else S.FLAT
    cap = max(L) + 8
    case = AttnCase(B, Hq, Hkv, d, cap, L, seed=B * 100 + Hq, regime=reg).to_cuda()
    q_obs_bits = k_to_bf16_bits(S.q_rows_k(B + 5, S.T_QVERIFY, B, w, Hq, Hkv, d, regime=reg))
    stride = ((budget - w) + 3) // 4 * 4
    idx = torch.full((B, Hkv, stride), -1, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(B, dtype=torch.int32, device="cuda")
    md.snapkv_select(case.k, case.v, bits_to_torch_bf16(q_obs_bits), torch.tensor(L, dtype=torch.int32).cuda(),
                     max(L), w, budget, case.scale, idx, cnt)
    torch.cuda.synchronize()
    ref_idx, ref_cnt, pooled = SK.snapkv_select(q_obs_bits, case.k_bits, np.array(L), w, budget, case.scale)
    _check_selection(idx.cpu().numpy(), cnt.cpu().numpy(), ref_idx, ref_cnt, pooled)


def test_snapkv_select_per_sequence_budgets():
    """Per-sequence budgets (heterogeneous batches): budgets below w keep nothing,
    above `budget` are clamped to it; each sequence's list matches the oracle's."""
    import synth as S
    B, Hq, Hkv, d, w, budget = 4, 32, 8, 128, 32, 512
    L = [3000, 2100, 1500, 900]
    budgets = [100, 10, 4096, 2048]
    reg = S.Regime("peaky", sink=4, needle_period=97)
    case = AttnCase(B, Hq, Hkv, d, max(L) + 8, L, seed=77, regime=reg).to_cuda()
    q_obs_bits = k_to_bf16_bits(S.q_rows_k(81, S.T_QVERIFY, B, w, Hq, Hkv, d, regime=reg))
    idx = torch.full((B, Hkv, budget - w), -1, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(B, dtype=torch.int32, device="cuda")
    md.snapkv_select(case.k, case.v, bits_to_torch_bf16(q_obs_bits), torch.tensor(L, dtype=torch.int32).cuda(),
                     max(L), w, budget, case.scale, idx, cnt, budgets=torch.tensor(budgets, dtype=torch.int32).cuda())
    torch.cuda.synchronize()
    ref_idx, ref_cnt, pooled = SK.snapkv_select(q_obs_bits, case.k_bits, np.array(L), w, budget, case.scale,
                                                budgets=np.array(budgets))
    assert cnt.cpu().tolist() == ref_cnt.tolist() == [100 - w, 0, budget - w, budget - w]
    _check_selection(idx.cpu().numpy(), cnt.cpu().numpy(), ref_idx, ref_cnt, pooled)
