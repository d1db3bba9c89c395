"""Pins for the oracle's attention (O1-O3, O6, kv_append): each check ties the oracle to
something other than itself — a closed form, a library routine (torch SDPA in fp64),
an invariant, a special case that reduces to another definition, or brute force.
Citations: PAPER.md P:204/P:281 (verify), P:453/P:720/P:1081 (StreamingLLM draft)."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import attention as A
from synth import bf16_bits_to_f32, k_to_bf16_bits

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _bits(rng, shape, lim=32):
    return k_to_bf16_bits(rng.integers(-lim, lim, size=shape))


def test_worked_example_closed_form():
    g = json.load(open(os.path.join(GOLD, "attn_worked_example.json")))
    o, lse = A.softmax_attention(np.array(g["q"]), np.array(g["k"]), np.array(g["v"]), g["scale"])
    assert np.allclose(o, g["o"], rtol=0, atol=1e-15)
    assert abs(lse - g["lse"]) < 1e-15


def test_bf16_decode_exact():
    bits = np.arange(0, 1 << 16, 257, dtype=np.uint16)
    ref = torch.tensor(bits.astype(np.int16)).view(torch.bfloat16).to(torch.float64).numpy()
    got = A.bf16_to_f64(bits)
    fin = np.isfinite(ref)
    assert np.array_equal(got[fin], ref[fin])


def test_equal_keys_give_mean_of_values():
    rng = np.random.default_rng(1)
    n, d = 37, 16
    q = rng.standard_normal(d)
    k = np.tile(rng.standard_normal(d), (n, 1))
    v = rng.standard_normal((n, d))
    o, lse = A.softmax_attention(q, k, v, 0.25)
    s = 0.25 * float(q @ k[0])
    assert np.allclose(o, v.mean(0), atol=1e-13)
    assert abs(lse - (s + np.log(n))) < 1e-12


def _sdpa_verify(qb, kb, vb, kv_len, scale):
    """torch SDPA (math backend, fp64) with an explicit boolean causal mask and
    KV repeated per query head (HF repeat_kv convention)."""
    q = torch.tensor(bf16_bits_to_f32(qb).astype(np.float64))       # [B,T,Hq,d]
    k = torch.tensor(bf16_bits_to_f32(kb).astype(np.float64))       # [B,Hkv,cap,d]
    v = torch.tensor(bf16_bits_to_f32(vb).astype(np.float64))
    B, T, Hq, d = q.shape
    g = Hq // k.shape[1]
    out = torch.zeros(B, T, Hq, d, dtype=torch.float64)
    for b in range(B):
        n = int(kv_len[b])
        kk = k[b, :, :n].repeat_interleave(g, dim=0)                  # [Hq, n, d]
        vv = v[b, :, :n].repeat_interleave(g, dim=0)
        qq = q[b].transpose(0, 1)                                     # [Hq, T, d]
        mask = torch.arange(n)[None, :] <= (n - T + torch.arange(T))[:, None]
        with torch.nn.attention.sdpa_kernel(torch.nn.attention.SDPBackend.MATH):
            o = torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, attn_mask=mask, scale=scale)
        out[b] = o.transpose(0, 1)
    return out.numpy()


@pytest.mark.parametrize("B,T,Hq,Hkv,d,cap", [(2, 5, 8, 2, 64, 70), (3, 4, 4, 4, 32, 41), (1, 1, 6, 1, 128, 33)])
def test_verify_matches_torch_sdpa_fp64(B, T, Hq, Hkv, d, cap):
    rng = np.random.default_rng(B * 100 + T)
    qb = _bits(rng, (B, T, Hq, d))
    kb = _bits(rng, (B, Hkv, cap, d))
    vb = _bits(rng, (B, Hkv, cap, d))
    kv_len = rng.integers(T, cap + 1, size=B)
    scale = 1.0 / np.sqrt(d)
    o, _ = A.verify_attn_full(qb, kb, vb, kv_len, scale)
    ref = _sdpa_verify(qb, kb, vb, kv_len, scale)
    assert np.max(np.abs(o - ref)) < 1e-12


def test_causal_row_equals_single_token_decode():
    rng = np.random.default_rng(7)
    B, T, Hq, Hkv, d, cap = 2, 5, 4, 2, 32, 50
    qb, kb, vb = _bits(rng, (B, T, Hq, d)), _bits(rng, (B, Hkv, cap, d)), _bits(rng, (B, Hkv, cap, d))
    kv_len = np.array([50, 23])
    o, lse = A.verify_attn_full(qb, kb, vb, kv_len, 0.125)
    for t in range(T):
        o1, l1 = A.verify_attn_full(qb[:, t:t + 1], kb, vb, kv_len - (T - 1 - t), 0.125)
        assert np.array_equal(o1[:, 0], o[:, t]) and np.array_equal(l1[:, 0], lse[:, t])


def test_gqa_equals_mha_on_repeated_kv():
    rng = np.random.default_rng(8)
    B, T, Hq, Hkv, d, cap = 2, 3, 8, 2, 16, 40
    qb, kb, vb = _bits(rng, (B, T, Hq, d)), _bits(rng, (B, Hkv, cap, d)), _bits(rng, (B, Hkv, cap, d))
    kv_len = np.array([40, 17])
    o, lse = A.verify_attn_full(qb, kb, vb, kv_len, 0.25)
    g = Hq // Hkv
    o2, lse2 = A.verify_attn_full(qb, np.repeat(kb, g, axis=1), np.repeat(vb, g, axis=1), kv_len, 0.25)
    assert np.array_equal(o, o2) and np.array_equal(lse, lse2)


def test_permutation_and_shift_invariance():
    rng = np.random.default_rng(9)
    n, d = 200, 64
    q, k, v = rng.standard_normal(d), rng.standard_normal((n, d)), rng.standard_normal((n, d))
    o, lse = A.softmax_attention(q, k, v, 0.1)
    perm = rng.permutation(n)
    o2, lse2 = A.softmax_attention(q, k[perm], v[perm], 0.1)
    assert np.max(np.abs(o - o2)) < 1e-12 and abs(lse - lse2) < 1e-12
    # adding a constant c to every score (extra dim: q_c = c / scale, k_c = 1) leaves o unchanged
    c = 3.7
    o3, lse3 = A.softmax_attention(np.append(q, c / 0.1), np.hstack([k, np.ones((n, 1))]), v, 0.1)
    assert np.max(np.abs(o - o3)) < 1e-12 and abs((lse3 - c) - lse) < 1e-11


@pytest.mark.parametrize("n,sink,window", [(1, 4, 60), (30, 4, 60), (64, 4, 60), (65, 4, 60), (200, 4, 60),
                                           (260, 0, 17), (100, 100, 0), (7, 3, 4), (8, 3, 4), (9, 3, 4)])
def test_draft_index_set_brute_force(n, sink, window):
    expect = sorted({j for j in range(n) if j < sink or j >= n - window})
    assert A.draft_index_set(n, sink, window).tolist() == expect


def test_draft_with_covering_window_equals_full_attention():
    rng = np.random.default_rng(10)
    B, Hq, Hkv, d, cap = 3, 8, 4, 64, 90
    qb, kb, vb = _bits(rng, (B, Hq, d)), _bits(rng, (B, Hkv, cap, d)), _bits(rng, (B, Hkv, cap, d))
    kv_len = np.array([90, 45, 1])
    full, lfull = A.verify_attn_full(qb[:, None], kb, vb, kv_len, 0.125)
    for sink, window in [(4, 90), (0, 90), (90, 0), (30, 60), (4, 86)]:
        o, l = A.draft_attn_sparse(qb, kb, vb, kv_len, sink, window, 0.125)
        assert np.array_equal(o, full[:, 0]) and np.array_equal(l, lfull[:, 0]), (sink, window)


def test_draft_equals_attention_over_gathered_rows():
    rng = np.random.default_rng(11)
    B, Hq, Hkv, d, cap = 2, 4, 4, 64, 256
    qb, kb, vb = _bits(rng, (B, Hq, d)), _bits(rng, (B, Hkv, cap, d)), _bits(rng, (B, Hkv, cap, d))
    kv_len = np.array([256, 150])
    o, lse = A.draft_attn_sparse(qb, kb, vb, kv_len, 4, 60, 0.125)
    # explicit materialised compressed cache, then plain decode over it (SDPA, fp64)
    for b in range(B):
        J = [j for j in range(kv_len[b]) if j < 4 or j >= kv_len[b] - 60]
        kc, vc = kb[b:b + 1, :, J], vb[b:b + 1, :, J]
        ref = _sdpa_verify(qb[b:b + 1, None], kc, vc, np.array([len(J)]), 0.125)
        assert np.max(np.abs(o[b] - ref[0, 0])) < 1e-12


def test_draft_per_sequence_windows():
    """Per-sequence windows: a covering window gives full attention for that sequence
    only, and every sequence matches an SDPA over its own materialised sink + window rows."""
    rng = np.random.default_rng(13)
    B, Hq, Hkv, d, cap = 3, 4, 2, 64, 200
    qb, kb, vb = _bits(rng, (B, Hq, d)), _bits(rng, (B, Hkv, cap, d)), _bits(rng, (B, Hkv, cap, d))
    kv_len = np.array([200, 150, 120])
    windows = np.array([196, 10, 50])
    o, lse = A.draft_attn_sparse(qb, kb, vb, kv_len, 4, windows, 0.125)
    full, lfull = A.verify_attn_full(qb[:, None], kb, vb, kv_len, 0.125)
    assert np.array_equal(o[0], full[0, 0]) and np.array_equal(lse[0], lfull[0, 0])
    assert np.max(np.abs(o[1] - full[1, 0])) > 1e-3   # a short window really drops keys
    for b in range(B):
        J = [j for j in range(kv_len[b]) if j < 4 or j >= kv_len[b] - windows[b]]
        ref = _sdpa_verify(qb[b:b + 1, None], kb[b:b + 1, :, J], vb[b:b + 1, :, J], np.array([len(J)]), 0.125)
        assert np.max(np.abs(o[b] - ref[0, 0])) < 1e-12


def test_split_merge_identity():
    rng = np.random.default_rng(12)
    n, d = 300, 32
    q, k, v = rng.standard_normal(d), rng.standard_normal((n, d)), rng.standard_normal((n, d))
    o, lse = A.softmax_attention(q, k, v, 0.3)
    for _ in range(5):
        cuts = np.sort(rng.choice(np.arange(1, n), size=3, replace=False))
        parts = np.split(np.arange(n), cuts)
        res = [A.softmax_attention(q, k[p], v[p], 0.3) for p in parts]
        om, lm = A.merge_partials([r[0] for r in res], [r[1] for r in res])
        assert np.max(np.abs(om - o)) < 1e-12 and abs(lm - lse) < 1e-12


def test_kv_append_writes_only_target_rows():
    rng = np.random.default_rng(13)
    B, Hkv, cap, d, T = 2, 3, 20, 8, 4
    kc, vc = _bits(rng, (B, Hkv, cap, d)), _bits(rng, (B, Hkv, cap, d))
    k0, v0 = kc.copy(), vc.copy()
    kn, vn = _bits(rng, (B, T, Hkv, d)), _bits(rng, (B, T, Hkv, d))
    start = np.array([3, 16])
    A.kv_append(kc, vc, kn, vn, start)
    for b in range(B):
        for h in range(Hkv):
            for s in range(cap):
                if start[b] <= s < start[b] + T:
                    assert np.array_equal(kc[b, h, s], kn[b, s - start[b], h])
                    assert np.array_equal(vc[b, h, s], vn[b, s - start[b], h])
                else:
                    assert np.array_equal(kc[b, h, s], k0[b, h, s]) and np.array_equal(vc[b, h, s], v0[b, h, s])
