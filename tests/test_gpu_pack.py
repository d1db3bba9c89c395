"""GPU parity of unit packing in the draft calls (keys kernel, unit-aligned plan, R = g <= 4
query rows per KV head): a CTA's consecutive whole units share one pass, unit s on MMA rows
[sR, sR + R), and the group has one epilogue.  Only calls with more units than the grid's
resident CTAs (2 x 148) put several units on a CTA, so these shapes have hundreds to thousands
of (b, kv head) units: R = 4 (pack 2), R = 3 (pack 2, a thread's two rows in different units),
R = 2 (pack 4), R = 1 (MHA, pack 8); groups that cross sequence boundaries, CTAs with fewer
units than the pack, sequences shorter than the sink.  Each output against the fp64 oracle
(DESIGN.md §5 tolerances), the cache of the fused-append form bit-exact, and the per-CTA trace
(md_debug_trace slot 11: groups processed) shows the packing engaged.
"""
import zlib

import numpy as np
import pytest
import torch

import paper_2408_11049_b200 as md
import synth as S
from oracle import attention as OA
from oracle import snapkv as SK
from tests.helpers import AttnCase, bits_to_torch_bf16

pytestmark = pytest.mark.gpu

ATOL_O, ATOL_LSE = 2e-3, 1e-3
SLOTS = 16  # md_debug_trace slots per CTA

CASES = [
    # name,           B, Hq, Hkv, d, length range, sink, window
    ("llama3_pack2",  64, 32, 8, 128, (1000, 1300), 4, 1020),   # 512 units: 256 CTAs x one group of 2
    ("cross_seq",     111, 12, 3, 128, (200, 600), 4, 252),     # 333 units on 167 CTAs: groups of 1 and 2
    ("mha_pack8",     80, 32, 32, 64, (60, 400), 4, 124),       # 2560 units, 9 per CTA: groups of 8 + 1
    ("g2_pack4",      90, 16, 8, 128, (300, 700), 4, 252),      # 720 units, 3 per CTA: one group of 3
    ("g3_pack2",      60, 24, 8, 64, (100, 500), 0, 200),       # R = 3: rows 2 and 3 of a thread differ
    ("tiny_lengths",  64, 32, 8, 128, (1, 9), 4, 60),           # n <= sink + window, several n <= sink
]


def _lengths(name, B, lo, hi):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    return rng.integers(lo, hi + 1, size=B).astype(np.int32)


def _bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def _cmp(o, l, ro, rl):
    assert np.all(np.isfinite(o)) and np.all(np.isfinite(l))
    eo, el = np.max(np.abs(o - ro)), np.max(np.abs(l - rl))
    assert eo <= ATOL_O and el <= ATOL_LSE, (eo, el)


def _expected_groups(units, R):
    grid = 2 * torch.cuda.get_device_properties(0).multi_processor_count
    per = -(-units // grid)
    pack = 8 // R if R <= 4 else 1
    return -(-per // pack)


@pytest.mark.parametrize("name,B,Hq,Hkv,d,lr,sink,window", CASES)
def test_packed_draft_parity(name, B, Hq, Hkv, d, lr, sink, window):
    lens = _lengths(name, B, *lr)
    case = AttnCase(B, Hq, Hkv, d, int(lens.max()) + 3, lens, seed=zlib.crc32(name.encode()) & 0xFFFF).to_cuda()
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, Hq), float("nan"), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, sink + window), dtype=torch.uint8, device="cuda")
    tr = torch.zeros((4096, SLOTS), dtype=torch.int64, device="cuda")
    md.debug_trace(tr)
    md.draft_attn_sparse(case.qd, case.k, case.v, case.kv_len_t, sink, window, case.scale, out, lse, ws)
    torch.cuda.synchronize()
    md.debug_trace(None)
    ro, rl = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, sink, window, case.scale)
    _cmp(out.cpu().numpy(), lse.cpu().numpy(), ro, rl)
    t = tr.cpu().numpy()
    groups = t[t[:, 0] > 0][:, 11]
    assert groups.max() == _expected_groups(B * Hkv, Hq // Hkv), groups.max()


@pytest.mark.parametrize("name,B,Hq,Hkv,d,lr,sink,window", [c for c in CASES if c[0] != "tiny_lengths"])
@pytest.mark.parametrize("early_kv", [False, True])
def test_packed_draft_append_parity(name, B, Hq, Hkv, d, lr, sink, window, early_kv):
    """md_draft_attn_sparse_append(_ex) at packed shapes: equals kv_append + the plain call."""
    lens = _lengths(name, B, *lr)
    seed = zlib.crc32(name.encode()) & 0xFFFF
    case = AttnCase(B, Hq, Hkv, d, int(lens.max()) + 3, lens, seed=seed).to_cuda()
    kn = S.k_to_bf16_bits(S.new_kv_k(seed + 2, S.T_KNEW, B, 1, Hkv, d))
    vn = S.k_to_bf16_bits(S.new_kv_k(seed + 2, S.T_VNEW, B, 1, Hkv, d))
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, Hq), float("nan"), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, sink + window), dtype=torch.uint8, device="cuda")
    md.draft_attn_sparse_append(case.qd, case.k, case.v, bits_to_torch_bf16(kn), bits_to_torch_bf16(vn),
                                case.kv_len_t, sink, window, case.scale, out, lse, ws, early_kv=early_kv)
    torch.cuda.synchronize()
    kc, vc = case.k_bits.copy(), case.v_bits.copy()
    OA.kv_append(kc, vc, kn, vn, case.kv_len - 1)
    ro, rl = OA.draft_attn_sparse(case.qd_bits, kc, vc, case.kv_len, sink, window, case.scale)
    _cmp(out.cpu().numpy(), lse.cpu().numpy(), ro, rl)
    assert np.array_equal(_bits(case.k), kc) and np.array_equal(_bits(case.v), vc)


@pytest.mark.parametrize("B,Hq,Hkv,d,lr,stride,win", [
    (64, 32, 8, 128, (700, 1500), 512, 32),    # R = 4: pack 2
    (100, 32, 32, 64, (100, 300), 64, 7),      # MHA: pack 8
])
def test_packed_indexed_draft_parity(B, Hq, Hkv, d, lr, stride, win):
    """md_draft_attn_indexed (SnapKV / PQ index lists) at packed shapes."""
    rng = np.random.default_rng(B * 31 + Hkv)
    lens = rng.integers(lr[0], lr[1] + 1, size=B).astype(np.int32)
    case = AttnCase(B, Hq, Hkv, d, int(lens.max()) + 8, lens, seed=B + Hq).to_cuda()
    tails = (lens - win).astype(np.int32)
    counts = np.minimum(rng.integers(0, stride + 1, size=B), tails).astype(np.int32)
    idx = np.full((B, Hkv, stride), -1, np.int32)
    for b in range(B):
        for h in range(Hkv):
            idx[b, h, :counts[b]] = np.sort(rng.choice(int(tails[b]), size=int(counts[b]), replace=False))
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, Hq), float("nan"), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, case.cap), dtype=torch.uint8, device="cuda")
    md.draft_attn_indexed(case.qd, case.k, case.v, case.kv_len_t, torch.from_numpy(idx).cuda(),
                          torch.from_numpy(counts).cuda(), torch.from_numpy(tails).cuda(), case.scale, out, lse, ws)
    torch.cuda.synchronize()
    ro, rl = SK.draft_attn_indexed(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, idx, counts, tails, case.scale)
    _cmp(out.cpu().numpy(), lse.cpu().numpy(), ro, rl)
