"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(same md_* calls, same split plan): the caches are generated in HBM by the CUDA twin of
the synth generator; for a seeded sample of sequences the oracle regenerates that
sequence's K/V/Q on the host and computes its outputs one by one (fp64)."""
import numpy as np
import pytest
import torch

import paper_2408_11049_b200 as md
import synth as S
import synth.cuda as SC
from oracle import attention as OA

pytestmark = pytest.mark.gpu

ATOL_O, ATOL_LSE = 2e-3, 1e-3

# name, B, Hq, Hkv, d, ctx, gamma, sink, window   (BASELINE.json configs)
FULL = [
    ("llama2_8k", 64, 32, 32, 128, 8192, 3, 4, 508),
    ("llama3_b64_32k", 64, 32, 8, 128, 32768, 4, 4, 1020),
    ("qwen_100k", 64, 28, 4, 128, 100000, 4, 4, 2044),
    ("llama3_32k", 128, 32, 8, 128, 32768, 4, 4, 1020),
    ("llama3_scaling", 256, 32, 8, 128, 32768, 4, 4, 1020),
]


@pytest.mark.parametrize("name,B,Hq,Hkv,d,ctx,gamma,sink,window", FULL)
def test_fullsize_sampled_parity(name, B, Hq, Hkv, d, ctx, gamma, sink, window):
    seed, T = 1234, gamma + 1
    L = S.committed_lengths(seed, B, ctx, gamma, ragged=True)
    cap = ctx + T + 8
    reg = S.Regime("peaky", sink=sink)
    k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    SC.fill_cache(k, seed, S.T_KCACHE, 0, cap, reg)
    SC.fill_cache(v, seed, S.T_VCACHE, 0, cap, reg)
    qv = torch.empty((B, T, Hq, d), dtype=torch.bfloat16, device="cuda")
    qd = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_q(qv, seed, S.T_QVERIFY, Hkv, reg)
    SC.fill_q(qd, seed, S.T_QDRAFT, Hkv, reg)
    kv_v = (L + T).astype(np.int32)        # verify: committed + the T new tokens
    kv_d = (L + 1).astype(np.int32)        # first draft step
    scale = float(np.float32(1 / np.sqrt(d)))
    out_v = torch.empty((B, T, Hq, d), device="cuda")
    lse_v = torch.empty((B, T, Hq), device="cuda")
    mkl = int(kv_v.max())
    ws = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, T, mkl)), dtype=torch.uint8, device="cuda")
    md.verify_attn_full(qv, k, v, torch.from_numpy(kv_v).cuda(), mkl, scale, out_v, lse_v, ws)
    out_d = torch.empty((B, Hq, d), device="cuda")
    lse_d = torch.empty((B, Hq), device="cuda")
    wsd = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, 1, min(sink + window, cap))),
                      dtype=torch.uint8, device="cuda")
    md.draft_attn_sparse(qd, k, v, torch.from_numpy(kv_d).cuda(), sink, window, scale, out_d, lse_d, wsd)
    torch.cuda.synchronize()
    ov, lv, od, ld = (x.cpu().numpy() for x in (out_v, lse_v, out_d, lse_d))
    assert np.all(np.isfinite(ov)) and np.all(np.isfinite(od))
    for b in (0, B // 2 + 1, B - 1):
        n = int(kv_v[b])
        kb = S.k_to_bf16_bits(S.kv_cache_k(seed, S.T_KCACHE, B, Hkv, d, 0, n, b_sel=[b], regime=reg))
        vb = S.k_to_bf16_bits(S.kv_cache_k(seed, S.T_VCACHE, B, Hkv, d, 0, n, b_sel=[b], regime=reg))
        qvb = S.k_to_bf16_bits(S.q_rows_k(seed, S.T_QVERIFY, B, T, Hq, Hkv, d, b_sel=[b], regime=reg))
        qdb = S.k_to_bf16_bits(S.q_rows_k(seed, S.T_QDRAFT, B, 1, Hq, Hkv, d, b_sel=[b], regime=reg))[:, 0]
        ro, rl = OA.verify_attn_full(qvb, kb, vb, kv_v[b:b + 1], scale)
        assert np.max(np.abs(ov[b] - ro[0])) <= ATOL_O and np.max(np.abs(lv[b] - rl[0])) <= ATOL_LSE
        ro, rl = OA.draft_attn_sparse(qdb, kb, vb, kv_d[b:b + 1], sink, window, scale)
        assert np.max(np.abs(od[b] - ro[0])) <= ATOL_O and np.max(np.abs(ld[b] - rl[0])) <= ATOL_LSE
    del k, v
    torch.cuda.empty_cache()
