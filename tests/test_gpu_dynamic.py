"""The keys kernel's dynamic tail (stream-K static shares + atomically claimed chunks, DESIGN.md
§7) engages only for long calls: >= DYN_MIN_TILES = 128 tiles of 64 keys per CTA of the
2 x 148-CTA grid (>= 37888 tiles).  These shapes cross that threshold with the library's
compile-time defaults (no environment knobs), so the claimed-chunk hand-off, the multi-partial
merge over dynamic chunks, and the fused *_append call falling back to a separate append launch
are all exercised against the fp64 oracle."""
import numpy as np
import pytest
import torch

import paper_2408_11049_b200 as md
from oracle import attention as OA
from tests.helpers import AttnCase, bits_to_torch_bf16
import synth as S

pytestmark = pytest.mark.gpu

DYN_TILES = 128 * 2 * 148


def _check(o, l, ro, rl):
    assert np.all(np.isfinite(o)) and np.all(np.isfinite(l))
    eo, el = float(np.max(np.abs(o - ro))), float(np.max(np.abs(l - rl)))
    assert eo <= 2e-3 and el <= 1e-3, (eo, el)


def test_mha_verify_dynamic_tail():
    lens = [20000, 19999, 18050, 21000]
    B, H, d, T = 4, 32, 128, 2
    assert sum((n + 63) // 64 for n in lens) * H >= DYN_TILES
    case = AttnCase(B, H, H, d, max(lens) + 8, lens, T=T, seed=1201).to_cuda()
    mkl = max(lens)
    ws = torch.zeros(md.attn_workspace_bytes(B, H, H, d, T, mkl), dtype=torch.uint8, device="cuda")
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    for rep in range(2):  # the counters are re-armed by the last CTA: a second call must agree
        out = torch.full((B, T, H, d), float("nan"), device="cuda")
        lse = torch.full((B, T, H), float("nan"), device="cuda")
        md.verify_attn_full(case.qv, case.k, case.v, case.kv_len_t, mkl, case.scale, out, lse, ws)
        torch.cuda.synchronize()
        _check(out.cpu().numpy(), lse.cpu().numpy(), ro, rl)
    # the fused form of a dynamic-tail call enqueues the append kernel ahead of the attention
    kn = S.k_to_bf16_bits(S.new_kv_k(1202, S.T_KNEW, B, T, H, d))
    vn = S.k_to_bf16_bits(S.new_kv_k(1202, S.T_VNEW, B, T, H, d))
    out = torch.full((B, T, H, d), float("nan"), device="cuda")
    lse = torch.full((B, T, H), float("nan"), device="cuda")
    md.verify_attn_full_append(case.qv, case.k, case.v, bits_to_torch_bf16(kn), bits_to_torch_bf16(vn), case.kv_len_t,
                               mkl, case.scale, out, lse, ws)
    torch.cuda.synchronize()
    OA.kv_append(case.k_bits, case.v_bits, kn, vn, case.kv_len - T)
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    _check(out.cpu().numpy(), lse.cpu().numpy(), ro, rl)
    assert np.array_equal(case.k.cpu().view(torch.int16).numpy().view(np.uint16), case.k_bits)
    assert np.array_equal(case.v.cpu().view(torch.int16).numpy().view(np.uint16), case.v_bits)


def test_mha_draft_dynamic_tail():
    rng = np.random.default_rng(1203)
    B, H, d, sink, window = 128, 32, 128, 4, 1020
    lens = rng.integers(1030, 1500, size=B)
    lens[:3] = [1024, 1025, 1499]
    assert sum((min(int(n), sink + window) + 63) // 64 for n in lens) * H >= DYN_TILES
    case = AttnCase(B, H, H, d, int(lens.max()) + 4, lens, seed=1203).to_cuda()
    ws = torch.zeros(md.attn_workspace_bytes(B, H, H, d, 1, sink + window), dtype=torch.uint8, device="cuda")
    out = torch.full((B, H, d), float("nan"), device="cuda")
    lse = torch.full((B, H), float("nan"), device="cuda")
    md.draft_attn_sparse(case.qd, case.k, case.v, case.kv_len_t, sink, window, case.scale, out, lse, ws)
    torch.cuda.synchronize()
    ro, rl = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, sink, window, case.scale)
    _check(out.cpu().numpy(), lse.cpu().numpy(), ro, rl)
