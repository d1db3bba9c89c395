"""Small launches of every attention-path kernel family for compute-sanitizer (racecheck /
synccheck / memcheck): tcgen05 verify (one and two row groups, fused append, split units),
the mma.sync keys kernel (draft, fused append, indexed draft), the rows kernel (head_dim 64),
and the SnapKV tcgen05 scoring passes.  usage: python tools/sanitize_cases.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402
import synth as S  # noqa: E402
from tests.helpers import AttnCase, bits_to_torch_bf16  # noqa: E402


def verify(case, T, fused=False):
    B, Hq, d = case.B, case.Hq, case.d
    out = torch.empty((B, T, Hq, d), device="cuda")
    lse = torch.empty((B, T, Hq), device="cuda")
    mkl = int(case.kv_len.max())
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, case.Hkv, d, T, mkl), dtype=torch.uint8, device="cuda")
    if fused:
        kn = bits_to_torch_bf16(S.k_to_bf16_bits(S.new_kv_k(3, S.T_KNEW, B, T, case.Hkv, d)))
        md.verify_attn_full_append(case.qv, case.k, case.v, kn, kn, case.kv_len_t, mkl, case.scale, out, lse, ws)
    else:
        md.verify_attn_full(case.qv, case.k, case.v, case.kv_len_t, mkl, case.scale, out, lse, ws)


def draft(case, sink, window, fused=False):
    B, Hq, d = case.B, case.Hq, case.d
    out = torch.empty((B, Hq, d), device="cuda")
    lse = torch.empty((B, Hq), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, case.Hkv, d, 1, sink + window), dtype=torch.uint8, device="cuda")
    if fused:
        kn = bits_to_torch_bf16(S.k_to_bf16_bits(S.new_kv_k(4, S.T_KNEW, B, 1, case.Hkv, d)))
        md.draft_attn_sparse_append(case.qd, case.k, case.v, kn, kn, case.kv_len_t, sink, window, case.scale, out, lse,
                                    ws)
    else:
        md.draft_attn_sparse(case.qd, case.k, case.v, case.kv_len_t, sink, window, case.scale, out, lse, ws)


def main():
    md.load_library()
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "tc"):
        verify(AttnCase(2, 32, 8, 128, 2100, [2100, 700], T=5, seed=1).to_cuda(), 5)             # R = 20
        verify(AttnCase(2, 32, 8, 128, 2100, [2100, 700], T=5, seed=1).to_cuda(), 5, fused=True)
        verify(AttnCase(1, 4, 1, 128, 9000, [9000], T=5, seed=2).to_cuda(), 5)                   # split unit
        verify(AttnCase(2, 28, 4, 128, 1500, [1500, 300], T=8, seed=3).to_cuda(), 8)             # R = 56: 2 groups
        verify(AttnCase(2, 28, 4, 128, 900, [900, 20], T=16, seed=4).to_cuda(), 16)              # R = 112
    if which in ("all", "keys"):
        c = AttnCase(3, 32, 8, 128, 3000, [3000, 1030, 64], T=1, seed=5).to_cuda()
        draft(c, 4, 1020)
        draft(c, 4, 1020, fused=True)
        verify(AttnCase(2, 32, 32, 128, 1200, [1200, 333], T=4, seed=6).to_cuda(), 4)            # MHA verify
    if which in ("all", "rows"):
        verify(AttnCase(2, 16, 2, 64, 800, [800, 129], T=8, seed=7).to_cuda(), 8)                # d = 64, R = 64
    if which in ("all", "snap"):
        B, Hq, Hkv, d, w, budget = 2, 32, 8, 128, 32, 256
        L = [1500, 900]
        case = AttnCase(B, Hq, Hkv, d, 1600, L, seed=8).to_cuda()
        q_obs = bits_to_torch_bf16(S.k_to_bf16_bits(S.q_rows_k(8, S.T_QVERIFY, B, w, Hq, Hkv, d)))
        idx = torch.zeros((B, Hkv, budget), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(B, dtype=torch.int32, device="cuda")
        md.snapkv_select(case.k, case.v, q_obs, torch.tensor(L, dtype=torch.int32).cuda(), max(L), w, budget,
                         case.scale, idx, cnt)
    if which in ("all", "tc_ct"):  # compile-time row counts (round 2): R = 24 / 36 / 42 / 48
        verify(AttnCase(2, 32, 8, 128, 1400, [1400, 300], T=6, seed=9).to_cuda(), 6)
        verify(AttnCase(2, 32, 8, 128, 1400, [1400, 300], T=9, seed=10).to_cuda(), 9)
        verify(AttnCase(2, 28, 4, 128, 1400, [1400, 300], T=6, seed=11).to_cuda(), 6)
        verify(AttnCase(2, 32, 8, 128, 1400, [1400, 300], T=12, seed=12).to_cuda(), 12, fused=True)
    if which in ("all", "indexed"):  # listed-row copies (8 rows x 64 B per instruction), plain and fused
        B, Hq, Hkv, d, K = 3, 32, 8, 128, 200
        L = [1800, 1100, 300]
        case = AttnCase(B, Hq, Hkv, d, 1850, L, T=1, seed=13).to_cuda()
        rng = np.random.default_rng(13)
        idx = np.zeros((B, Hkv, 200), np.int32)
        for b in range(B):
            for u in range(Hkv):
                idx[b, u, :K] = np.sort(rng.choice(L[b] - 64, size=K, replace=False))
        idx_t = torch.from_numpy(idx).cuda()
        cnt = torch.full((B,), K, dtype=torch.int32, device="cuda")
        tail = torch.tensor([n - 40 for n in L], dtype=torch.int32, device="cuda")
        out = torch.empty((B, Hq, d), device="cuda")
        ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, 1850), dtype=torch.uint8, device="cuda")
        md.draft_attn_indexed(case.qd, case.k, case.v, case.kv_len_t, idx_t, cnt, tail, case.scale, out, None, ws)
        kn = bits_to_torch_bf16(S.k_to_bf16_bits(S.new_kv_k(14, S.T_KNEW, B, 1, Hkv, d)))
        md.draft_attn_indexed(case.qd, case.k, case.v, case.kv_len_t, idx_t, cnt, tail, case.scale, out, None, ws,
                              k_new=kn, v_new=kn)
    if which in ("all", "pq"):  # PQ encode / LUT / score / select
        B, Hq, Hkv, d = 2, 32, 8, 128
        L = [3000, 1700]
        case = AttnCase(B, Hq, Hkv, d, 3000, L, T=1, seed=15).to_cuda()
        pos = S.pq_codebook_positions(15, B, Hkv, L)
        cb = bits_to_torch_bf16(S.pq_codebook_bits(case.k_bits, pos))
        codes = torch.zeros((B, Hkv, 3000, 16), dtype=torch.uint8, device="cuda")
        md.pq_encode(case.k, case.v, cb, torch.zeros(B, dtype=torch.int32, device="cuda"), 3000, codes)
        idx = torch.zeros((B, Hkv, 4 + 256), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(B, dtype=torch.int32, device="cuda")
        tail = torch.zeros(B, dtype=torch.int32, device="cuda")
        ws = torch.zeros(md.pq_workspace_bytes(B, Hkv, 3000), dtype=torch.uint8, device="cuda")
        md.pq_select(case.qd, cb, codes, case.kv_len_t, 3000, 4, 128, 256, idx, cnt, tail, ws)
    if which in ("all", "packed"):  # unit packing (R = 4: pack 2, R = 1: pack 8), fused append, early KV + stash
        for (B, Hq, Hkv, L0) in ((40, 32, 8, 200), (80, 32, 32, 90)):
            lens = [L0 - (b % 7) for b in range(B)]
            c = AttnCase(B, Hq, Hkv, 128, L0, lens, T=1, seed=18).to_cuda()
            draft(c, 4, 60)
            draft(c, 4, 60, fused=True)
            out = torch.empty((B, Hq, 128), device="cuda")
            ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, 128, 1, 64), dtype=torch.uint8, device="cuda")
            kn = bits_to_torch_bf16(S.k_to_bf16_bits(S.new_kv_k(19, S.T_KNEW, B, 1, Hkv, 128)))
            for _ in range(2):  # back to back: the second call's prologue overlaps the first call's tail
                md.draft_attn_sparse_append(c.qd, c.k, c.v, kn, kn, c.kv_len_t, 4, 60, c.scale, out, None, ws,
                                            early_kv=True)
    if which in ("all", "misc"):  # acceptance (sample / greedy), tree acceptance, compaction, append, philox
        B, gamma, V, T = 4, 4, 1000, 5
        rng = np.random.default_rng(16)
        p = rng.random((B, gamma + 1, V)) ** 4
        p /= p.sum(-1, keepdims=True)
        q = rng.random((B, gamma, V)) ** 4
        q /= q.sum(-1, keepdims=True)
        pt = torch.from_numpy(p.astype(np.float32)).cuda()
        qt = torch.from_numpy(q.astype(np.float32)).cuda()
        dt = torch.from_numpy(rng.integers(0, V, (B, gamma)).astype(np.int32)).cuda()
        rnd = torch.zeros((B, T + 1), dtype=torch.int32, device="cuda")
        md.philox_u32(17, 3, rnd)
        ot = torch.zeros((B, gamma + 1), dtype=torch.int32, device="cuda")
        na = torch.zeros(B, dtype=torch.int32, device="cuda")
        md.spec_accept(pt, qt, dt, rnd[:, :gamma + 2].contiguous(), ot, na)
        md.spec_accept(pt, qt, dt, rnd[:, :gamma + 2].contiguous(), ot, na, mode="greedy")
        ptr_ = torch.from_numpy((rng.random((B, T, V)) ** 4).astype(np.float32)).cuda()
        ptr_ /= ptr_.sum(-1, keepdim=True)
        qtr = torch.from_numpy((rng.random((B, T, V)) ** 4).astype(np.float32)).cuda()
        qtr /= qtr.sum(-1, keepdim=True)
        parent = torch.tensor([[-1, 0, 0, 1, 1]] * B, dtype=torch.int32, device="cuda")
        tok = torch.from_numpy(rng.integers(0, V, (B, T)).astype(np.int32)).cuda()
        otr = torch.zeros((B, T), dtype=torch.int32, device="cuda")
        nodes = torch.zeros((B, T), dtype=torch.int32, device="cuda")
        md.spec_accept_tree(ptr_, qtr, tok, parent, rnd, otr, na, accepted_nodes=nodes)
        case = AttnCase(B, 8, 2, 128, 300, [290, 200, 100, 50], T=T, seed=18).to_cuda()
        md.kv_compact(case.k, case.v, torch.tensor([280, 190, 90, 40], dtype=torch.int32, device="cuda"), nodes, na)
        kn = bits_to_torch_bf16(S.k_to_bf16_bits(S.new_kv_k(19, S.T_KNEW, B, T, 2, 128)))
        md.kv_append(case.k, case.v, kn, kn, torch.tensor([5, 100, 60, 0], dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    print("sanitize cases done:", which)


if __name__ == "__main__":
    main()
