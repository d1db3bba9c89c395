"""The deterministic fixed-split plan (md_verify_attn_full_det / md_draft_attn_sparse_det; SURVEY
§8(e) "bitwise-equal to single-GPU when the split plan is pinned (MD_FIXED_SPLIT)"): a
KV-head-sharded (tensor-parallel) or batch-sharded run reproduces the unsharded call BIT FOR BIT,
and the results match the fp64 oracle within the usual tolerance."""
import numpy as np
import pytest
import torch

import paper_2408_11049_b200 as md
from oracle import attention as OA
from tests.helpers import AttnCase

pytestmark = pytest.mark.gpu


def _verify_det(case, k, v, q, kv_len, T, split, mkl):
    B, _, Hq, d = q.shape
    out = torch.full((B, T, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, T, Hq), float("nan"), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes_det(B, Hq, k.shape[1], d, T, mkl, split), dtype=torch.uint8,
                     device="cuda")
    md.verify_attn_full_det(q, k, v, kv_len, mkl, split, case.scale, out, lse, ws)
    return out, lse


def _draft_det(case, k, v, q, kv_len, sink, window, split):
    B, Hq, d = q.shape
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, Hq), float("nan"), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes_det(B, Hq, k.shape[1], d, 1, min(sink + window, k.shape[2]), split),
                     dtype=torch.uint8, device="cuda")
    md.draft_attn_sparse_det(q, k, v, kv_len, sink, window, split, case.scale, out, lse, ws)
    return out, lse


@pytest.mark.parametrize("B,Hq,Hkv,d,T,lens,split", [
    (4, 32, 8, 128, 5, [3000, 2999, 1100, 64], 1024),   # tcgen05 kernel, R = 20
    (3, 28, 4, 128, 8, [2500, 700, 8], 512),            # tcgen05 row groups, R = 56
    (2, 32, 32, 128, 4, [2000, 333], 640),              # keys kernel (MHA verify)
    (3, 16, 4, 64, 4, [900, 129, 4], 256),              # rows kernel (head_dim 64, R = 16)
])
def test_verify_det_is_shard_invariant(B, Hq, Hkv, d, T, lens, split):
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, T=T, seed=B * 7 + Hq).to_cuda()
    mkl = max(lens)
    full_o, full_l = _verify_det(case, case.k, case.v, case.qv, case.kv_len_t, T, split, mkl)
    torch.cuda.synchronize()
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    assert np.max(np.abs(full_o.cpu().numpy() - ro)) <= 2e-3 and np.max(np.abs(full_l.cpu().numpy() - rl)) <= 1e-3
    g = Hq // Hkv
    for P in (2, 4):
        if Hkv % P:
            continue
        for r in range(P):              # KV-head tensor parallelism: rank r's heads, strided cache views
            ks = slice(r * Hkv // P, (r + 1) * Hkv // P)
            qs = slice(ks.start * g, ks.stop * g)
            o, l = _verify_det(case, case.k[:, ks], case.v[:, ks], case.qv[:, :, qs].contiguous(), case.kv_len_t, T,
                               split, mkl)
            assert torch.equal(o, full_o[:, :, qs]) and torch.equal(l, full_l[:, :, qs]), (P, r)
    for b0, b1 in ((0, 1), (1, B)):    # batch data parallelism
        o, l = _verify_det(case, case.k[b0:b1], case.v[b0:b1], case.qv[b0:b1].contiguous(),
                           case.kv_len_t[b0:b1].contiguous(), T, split, mkl)
        assert torch.equal(o, full_o[b0:b1]) and torch.equal(l, full_l[b0:b1]), (b0, b1)
    o2, l2 = _verify_det(case, case.k, case.v, case.qv, case.kv_len_t, T, split, mkl)   # repeatable
    assert torch.equal(o2, full_o) and torch.equal(l2, full_l)


def test_draft_det_is_shard_invariant():
    B, Hq, Hkv, d, sink, window, split = 4, 32, 8, 128, 4, 1020, 256
    lens = [3000, 1025, 700, 2]
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, seed=77).to_cuda()
    full_o, full_l = _draft_det(case, case.k, case.v, case.qd, case.kv_len_t, sink, window, split)
    torch.cuda.synchronize()
    ro, rl = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, sink, window, case.scale)
    assert np.max(np.abs(full_o.cpu().numpy() - ro)) <= 2e-3 and np.max(np.abs(full_l.cpu().numpy() - rl)) <= 1e-3
    g = Hq // Hkv
    for P in (2, 8):
        for r in range(P):
            ks = slice(r * Hkv // P, (r + 1) * Hkv // P)
            qs = slice(ks.start * g, ks.stop * g)
            o, l = _draft_det(case, case.k[:, ks], case.v[:, ks], case.qd[:, qs].contiguous(), case.kv_len_t, sink,
                              window, split)
            assert torch.equal(o, full_o[:, qs]) and torch.equal(l, full_l[:, qs]), (P, r)
    o, l = _draft_det(case, case.k[2:], case.v[2:], case.qd[2:].contiguous(), case.kv_len_t[2:].contiguous(), sink,
                      window, split)
    assert torch.equal(o, full_o[2:]) and torch.equal(l, full_l[2:])


def test_det_workspace_and_args():
    assert md.attn_workspace_bytes_det(4, 32, 8, 128, 5, 3000, 1024) > 0
    assert md.attn_workspace_bytes_det(4, 32, 8, 128, 5, 3000, 100) == 0      # not a multiple of 64
    case = AttnCase(1, 4, 1, 128, 200, [200], T=1, seed=3).to_cuda()
    out = torch.empty((1, 4, 128), device="cuda")
    with pytest.raises(md.MDError):
        md.draft_attn_sparse_det(case.qd, case.k, case.v, case.kv_len_t, 4, 60, 96, case.scale, out)
