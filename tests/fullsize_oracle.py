"""Oracle side of the full-size sampled parity test (tests/test_gpu_parity_fullsize.py), run in
worker processes: for one sampled sequence b and a few of its KV heads, regenerate from the
seeded generators the cache rows, the queries and the new K/V rows the GPU call consumed, apply
the step's appends exactly as md_kv_append would (oracle.attention.kv_append), and compute the
draft (O3) and verify (O2) outputs of those heads in fp64.  Inputs only come from synth/; no
value comes from the CUDA path."""
from __future__ import annotations

import numpy as np

import synth as S
from oracle import attention as OA

SEED = 4321


def inputs(kind, B, Hq, Hkv, d, T, b, heads, n_rows):
    """Host bits for sequence b: cache rows [0, n_rows) of `heads`, verify / draft queries of the
    heads' query groups, and the new rows (draft [1][Hkv][d], verify [T][Hkv][d])."""
    g = Hq // Hkv
    reg = S.Regime("peaky", sink=4)
    if kind == "offgrid":
        kb = S.kv_cache_bits_offgrid(SEED, S.T_KCACHE, B, Hkv, d, 0, n_rows, b_sel=[b], h_sel=heads)
        vb = S.kv_cache_bits_offgrid(SEED, S.T_VCACHE, B, Hkv, d, 0, n_rows, b_sel=[b], h_sel=heads)
        qv = S.flat_bits_offgrid(SEED, S.T_QVERIFY, (B, T, Hq, d), b_sel=[b])
        qd = S.flat_bits_offgrid(SEED, S.T_QDRAFT, (B, Hq, d), b_sel=[b])
        knd = S.flat_bits_offgrid(SEED + 1, S.T_KNEW, (B, 1, Hkv, d), b_sel=[b])
        vnd = S.flat_bits_offgrid(SEED + 1, S.T_VNEW, (B, 1, Hkv, d), b_sel=[b])
        knv = S.flat_bits_offgrid(SEED, S.T_KNEW, (B, T, Hkv, d), b_sel=[b])
        vnv = S.flat_bits_offgrid(SEED, S.T_VNEW, (B, T, Hkv, d), b_sel=[b])
    else:
        kb = S.k_to_bf16_bits(S.kv_cache_k(SEED, S.T_KCACHE, B, Hkv, d, 0, n_rows, b_sel=[b], h_sel=heads, regime=reg))
        vb = S.k_to_bf16_bits(S.kv_cache_k(SEED, S.T_VCACHE, B, Hkv, d, 0, n_rows, b_sel=[b], h_sel=heads, regime=reg))
        qv = S.k_to_bf16_bits(S.q_rows_k(SEED, S.T_QVERIFY, B, T, Hq, Hkv, d, b_sel=[b], regime=reg))
        qd = S.k_to_bf16_bits(S.q_rows_k(SEED, S.T_QDRAFT, B, 1, Hq, Hkv, d, b_sel=[b], regime=reg))[:, 0]
        knd = S.k_to_bf16_bits(S.new_kv_k(SEED + 1, S.T_KNEW, B, 1, Hkv, d))[b:b + 1]
        vnd = S.k_to_bf16_bits(S.new_kv_k(SEED + 1, S.T_VNEW, B, 1, Hkv, d))[b:b + 1]
        knv = S.k_to_bf16_bits(S.new_kv_k(SEED, S.T_KNEW, B, T, Hkv, d))[b:b + 1]
        vnv = S.k_to_bf16_bits(S.new_kv_k(SEED, S.T_VNEW, B, T, Hkv, d))[b:b + 1]
    qh = np.concatenate([np.arange(h * g, (h + 1) * g) for h in heads])
    return kb, vb, qv[:, :, qh], qd[:, qh], knd[:, :, heads], vnd[:, :, heads], knv[:, :, heads], vnv[:, :, heads]


def oracle_one(args):
    """(b, heads, draft out/lse, verify out/lse, the appended rows [L, L+T) of K and V) in fp64."""
    kind, B, Hq, Hkv, d, T, sink, window, scale, b, heads, L = args
    heads = list(heads)
    kb, vb, qv, qd, knd, vnd, knv, vnv = inputs(kind, B, Hq, Hkv, d, T, b, heads, L + T)
    # the step: draft j = 0 appends its row at L and attends with kv_len = L + 1 ...
    OA.kv_append(kb, vb, knd, vnd, np.array([L]))
    od, ld = OA.draft_attn_sparse(qd, kb, vb, np.array([L + 1]), sink, window, scale)
    # ... then the verify appends the T target rows at L (overwriting the draft row), kv_len = L + T
    OA.kv_append(kb, vb, knv, vnv, np.array([L]))
    ov, lv = OA.verify_attn_full(qv, kb, vb, np.array([L + T]), scale)
    return b, heads, od[0], ld[0], ov[0], lv[0], kb[0, :, L:L + T].copy(), vb[0, :, L:L + T].copy()
