"""GPU parity: every md_* call through the C ABI vs the fp64 oracle on identical seeded inputs.

Tolerances (north_star): attention outputs max-abs <= 2e-3, lse <= 1e-3
(bf16 KV and Q exact, fp32 accumulation, bf16 P in the PV product: worst case
2^-9 max|v| = 1.95e-3 with |v| <= 1); kv_append, Philox and spec_accept bit-exact.
Shapes: shrunken variants of every BASELINE.json config (same head geometry, smaller
B / ctx) that span several 64-key tiles, several splits and a ragged tail.
"""
import ctypes
import zlib

import numpy as np
import pytest
import torch

import paper_2408_11049_b200 as md
import synth as S
from oracle import accept as OACC
from oracle import attention as OA
from oracle import philox as OPH
from tests.helpers import AttnCase, bits_to_torch_bf16

pytestmark = pytest.mark.gpu

ATOL_O = 2e-3
ATOL_LSE = 1e-3


def _run_verify(case: AttnCase, max_kv_len=None):
    B, T, Hq, d = case.B, case.T, case.Hq, case.d
    mkl = int(case.kv_len.max()) if max_kv_len is None else max_kv_len
    out = torch.full((B, T, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, T, Hq), float("nan"), device="cuda")
    wsb = md.attn_workspace_bytes(B, Hq, case.Hkv, d, T, mkl)
    ws = torch.zeros(max(wsb, 1), dtype=torch.uint8, device="cuda")
    md.verify_attn_full(case.qv, case.k, case.v, case.kv_len_t, mkl, case.scale, out, lse, ws)
    torch.cuda.synchronize()
    return out.cpu().numpy(), lse.cpu().numpy()


def _run_draft(case: AttnCase, sink, window):
    B, Hq, d = case.B, case.Hq, case.d
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, Hq), float("nan"), device="cuda")
    wsb = md.attn_workspace_bytes(B, Hq, case.Hkv, d, 1, min(sink + window, case.cap))
    ws = torch.zeros(max(wsb, 1), dtype=torch.uint8, device="cuda")
    md.draft_attn_sparse(case.qd, case.k, case.v, case.kv_len_t, sink, window, case.scale, out, lse, ws)
    torch.cuda.synchronize()
    return out.cpu().numpy(), lse.cpu().numpy()


def _cmp(got_o, got_l, ref_o, ref_l):
    assert np.all(np.isfinite(got_o)) and np.all(np.isfinite(got_l))
    eo = np.max(np.abs(got_o - ref_o))
    el = np.max(np.abs(got_l - ref_l))
    assert eo <= ATOL_O and el <= ATOL_LSE, (eo, el)
    return eo, el


VERIFY_CASES = [
    # name,            B, Hq, Hkv,  d,  T, lengths
    ("tiny",           2, 4, 4, 64, 4, [256, 256]),
    ("llama2_mha",     2, 32, 32, 128, 4, [1000, 517]),
    ("llama3_gqa",     3, 32, 8, 128, 5, [1500, 1497, 64]),
    ("qwen_gqa",       2, 28, 4, 128, 5, [2100, 777]),
    ("decode_T1",      2, 32, 8, 128, 1, [300, 1]),
    ("gqa_g8_T8",      2, 16, 2, 64, 8, [130, 8]),       # 64 rows = 4 m-tiles
    ("d64_ragged",     4, 8, 2, 64, 3, [3, 65, 128, 129]),
    ("tc_generic_26",  2, 16, 8, 128, 13, [2000, 133]),      # tcgen05 kernel, NP=32, runtime R=26
    # compile-time row counts of the paper's operating points (Llama-3.1 gamma 5/6/7/8/11, Qwen2.5 gamma 5)
    ("tc_ct_24",       2, 32, 8, 128, 6, [1900, 411]),
    ("tc_ct_28",       2, 32, 8, 128, 7, [1300, 129]),
    ("tc_ct_32",       2, 32, 8, 128, 8, [2222, 64]),
    ("tc_ct_36",       2, 32, 8, 128, 9, [1700, 900]),
    ("tc_ct_42",       2, 28, 4, 128, 6, [2600, 150]),
    ("tc_ct_48",       3, 32, 8, 128, 12, [1500, 700, 12]),
    ("tc_generic_40",  2, 16, 2, 128, 5, [1500, 700]),       # tcgen05 kernel, NP=48, runtime R=40
    ("tc_np16_16",     2, 8, 2, 128, 4, [900, 260]),         # tcgen05 kernel, NP=16, R=16
    # R > 48: the tcgen05 kernel's row groups (NG = NP / 32 groups of 32 rows, SURVEY §8(b) g*T <= 128)
    ("tc_np64_56",     2, 28, 4, 128, 8, [3000, 190]),       # Qwen2.5 g=7, gamma=7: NP=64, 2 groups
    ("tc_np96_77",     2, 28, 4, 128, 11, [2500, 133]),      # Qwen2.5, gamma=10: NP=96, 3 groups
    ("tc_np128_112",   3, 28, 4, 128, 16, [2100, 300, 16]),  # Qwen2.5, gamma=15: NP=128, n = T edge
    ("tc_np128_128",   2, 32, 4, 128, 16, [1800, 1000]),     # g=8 x T=16 = 128 rows, the ABI maximum
]


@pytest.mark.parametrize("name,B,Hq,Hkv,d,T,lens", VERIFY_CASES)
def test_verify_parity(name, B, Hq, Hkv, d, T, lens):
    cap = max(lens) + 7
    case = AttnCase(B, Hq, Hkv, d, cap, lens, T=T, seed=zlib.crc32(name.encode()) & 0xFFFF).to_cuda()
    o, l = _run_verify(case)
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    _cmp(o, l, ro, rl)


def test_verify_peaky_sinks_and_many_splits():
    """Attention-sink regime (large score range, max rescaling) with a long context that
    the planner splits several ways, plus a max_kv_len hint larger than any kv_len."""
    reg = S.Regime("peaky", sink=4, needle_period=509)
    case = AttnCase(2, 32, 8, 128, 6000, [5990, 4100], T=5, seed=77, regime=reg).to_cuda()
    o, l = _run_verify(case, max_kv_len=6000)
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    _cmp(o, l, ro, rl)


def test_verify_ignores_nonfinite_garbage_beyond_kv_len():
    """Rows >= kv_len may hold anything (NaN / Inf bit patterns): they must not leak."""
    case = AttnCase(2, 8, 2, 128, 200, [70, 133], T=3, seed=5)
    for b, n in enumerate(case.kv_len):
        case.k_bits[b, :, n:] = 0x7FC0     # NaN
        case.v_bits[b, :, n:] = 0x7F80     # +Inf
    case.to_cuda()
    o, l = _run_verify(case, max_kv_len=200)
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    _cmp(o, l, ro, rl)


def test_verify_nhd_strided_cache():
    """A [B, cap, Hkv, d] (NHD) cache passed through the strides of md_kv_cache."""
    case = AttnCase(2, 16, 4, 128, 300, [300, 211], T=5, seed=9)
    case.to_cuda()
    k_nhd = case.k.permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3)
    v_nhd = case.v.permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3)
    assert k_nhd.stride(2) == 4 * 128
    case.k, case.v = k_nhd, v_nhd
    o, l = _run_verify(case)
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    _cmp(o, l, ro, rl)


DRAFT_CASES = [
    # name,           B, Hq, Hkv, d, lengths, sink, window
    ("tiny",          2, 4, 4, 64, [256, 256], 4, 60),
    ("llama2",        2, 32, 32, 128, [2000, 600], 4, 508),
    ("llama3",        3, 32, 8, 128, [3000, 1025, 1024], 4, 1020),
    ("qwen",          2, 28, 4, 128, [4100, 2049], 4, 2044),
    ("short_seq",     3, 8, 2, 64, [1, 5, 63], 4, 60),      # n <= sink + window: all keys
    ("no_sink",       2, 8, 8, 64, [500, 90], 0, 77),
    ("sink_only",     2, 8, 8, 64, [500, 3], 10, 0),
    ("big_sink",      2, 8, 2, 128, [700, 300], 130, 200),
]


@pytest.mark.parametrize("name,B,Hq,Hkv,d,lens,sink,window", DRAFT_CASES)
def test_draft_parity(name, B, Hq, Hkv, d, lens, sink, window):
    cap = max(lens) + 3
    case = AttnCase(B, Hq, Hkv, d, cap, lens, seed=zlib.crc32(name.encode()) & 0xFFFF).to_cuda()
    o, l = _run_draft(case, sink, window)
    ro, rl = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, sink, window, case.scale)
    _cmp(o, l, ro, rl)


def test_draft_peaky():
    reg = S.Regime("peaky", sink=4, needle_period=97)
    case = AttnCase(2, 32, 8, 128, 4000, [4000, 1500], seed=3, regime=reg).to_cuda()
    o, l = _run_draft(case, 4, 1020)
    ro, rl = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, 4, 1020, case.scale)
    _cmp(o, l, ro, rl)


@pytest.mark.parametrize("sink", [4, 0])
def test_draft_per_sequence_windows(sink):
    """md_draft_attn_sparse_windows: per-sequence windows, clamped to [max(0, 1 - sink),
    window]; covers window 0, a window covering the sequence, one above the bound and ragged
    lengths spanning several tiles."""
    lens = [4000, 1500, 700, 90, 3000, 2]
    windows = [1020, 0, 64, 500, 5000, 1]
    B, Hq, Hkv, d, window = len(lens), 32, 8, 128, 1020
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 3, lens, seed=41 + sink).to_cuda()
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, Hq), float("nan"), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, sink + window), dtype=torch.uint8, device="cuda")
    wt = torch.tensor(windows, dtype=torch.int32, device="cuda")
    md.draft_attn_sparse(case.qd, case.k, case.v, case.kv_len_t, sink, window, case.scale, out, lse, ws, windows=wt)
    torch.cuda.synchronize()
    eff = np.minimum(window, np.maximum(np.array(windows), max(0, 1 - sink)))
    ro, rl = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, sink, eff, case.scale)
    _cmp(out.cpu().numpy(), lse.cpu().numpy(), ro, rl)
    # a NULL windows pointer is rejected on the host
    lib = md.load_library()
    c = md.make_cache(case.k, case.v)
    st = lib.md_draft_attn_sparse_windows(ctypes.byref(c), case.qd.data_ptr(), Hq, case.kv_len_t.data_ptr(), sink,
                                          window, None, 0.1, out.data_ptr(), None, ws.data_ptr(), ws.numel(), None)
    assert st != 0 and b"windows" in lib.md_last_error()


def test_kv_append_bit_exact():
    rng = np.random.default_rng(0)
    B, T, Hkv, d, cap = 3, 5, 8, 128, 64
    kc = S.k_to_bf16_bits(rng.integers(-32, 32, size=(B, Hkv, cap, d)))
    vc = S.k_to_bf16_bits(rng.integers(-32, 32, size=(B, Hkv, cap, d)))
    kn = S.k_to_bf16_bits(S.new_kv_k(1, S.T_KNEW, B, T, Hkv, d))
    vn = S.k_to_bf16_bits(S.new_kv_k(1, S.T_VNEW, B, T, Hkv, d))
    start = np.array([0, 17, cap - T], dtype=np.int32)
    kg, vg = bits_to_torch_bf16(kc), bits_to_torch_bf16(vc)
    md.kv_append(kg, vg, bits_to_torch_bf16(kn), bits_to_torch_bf16(vn), torch.from_numpy(start).cuda())
    OA.kv_append(kc, vc, kn, vn, start)
    torch.cuda.synchronize()
    assert np.array_equal(kg.cpu().view(torch.int16).numpy().view(np.uint16), kc)
    assert np.array_equal(vg.cpu().view(torch.int16).numpy().view(np.uint16), vc)


def test_philox_bit_exact():
    out = torch.empty((37, 7), dtype=torch.int32, device="cuda")
    md.philox_u32(0xDEADBEEF12345678, 3, out)
    ref = OPH.philox_words(0xDEADBEEF12345678, 3, 37, 7)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref)


def _accept_inputs(B, gamma, V, sigma, seed):
    p, q, d = S.spec_probs(seed, B, gamma, V, sigma)
    rnd = OPH.philox_words(seed, 1, B, gamma + 2)
    return p, q, d, rnd


def _run_accept(p, q, d, rnd, mode, committed=None):
    B, G1, V = p.shape
    pt, qt = torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda()
    dt = torch.from_numpy(d).cuda()
    rt = torch.from_numpy(rnd.view(np.int32)).cuda()
    out = torch.empty((B, G1), dtype=torch.int32, device="cuda")
    n = torch.empty(B, dtype=torch.int32, device="cuda")
    cl = None if committed is None else torch.from_numpy(committed.copy()).cuda()
    md.spec_accept(pt, qt, dt, rt, out, n, cl, mode=mode)
    torch.cuda.synchronize()
    return out.cpu().numpy(), n.cpu().numpy(), None if cl is None else cl.cpu().numpy()


@pytest.mark.parametrize("B,gamma,V,sigma", [(64, 3, 32, 0.8), (64, 4, 1000, 1.0), (16, 4, 128256, 0.9),
                                             (8, 15, 5000, 0.3), (32, 0, 777, 0.0), (12, 1, 152064, 2.5)])
def test_spec_accept_sample_bit_exact(B, gamma, V, sigma):
    p, q, d, rnd = _accept_inputs(B, gamma, V, sigma, seed=B * 31 + V)
    committed = np.arange(B, dtype=np.int32) + 1000
    got = _run_accept(p, q, d, rnd, "sample", committed)
    ref = OACC.spec_accept(p, q, d, rnd, "sample", committed)
    for g_, r_ in zip(got, ref):
        assert np.array_equal(g_, r_)


@pytest.mark.parametrize("B,gamma,V", [(16, 4, 32000), (8, 3, 50)])
def test_spec_accept_greedy_bit_exact(B, gamma, V):
    p, q, d, rnd = _accept_inputs(B, gamma, V, 0.7, seed=5)
    # make some drafts match the argmax so acceptance runs past position 0
    am = p[:, :gamma].argmax(-1)
    d = np.where(np.random.default_rng(0).random((B, gamma)) < 0.6, am, d).astype(np.int32)
    got = _run_accept(p, q, d, rnd, "greedy")
    ref = OACC.spec_accept(p, q, d, None, "greedy")
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])


def test_spec_accept_degenerate_rows():
    """p == q (all accept), disjoint supports (reject at 0), all-tiny final row (argmax)."""
    B, gamma, V = 6, 3, 40
    p = np.zeros((B, gamma + 1, V), np.float32)
    q = np.zeros((B, gamma, V), np.float32)
    p[:2] = 1.0 / V
    q[:2] = 1.0 / V
    p[2:4, :, :20] = 0.05
    q[2:4, :, 20:] = 0.05
    p[4:, :, 7] = 1e-13
    p[4:, :, 9] = 3e-13
    q[4:, :, 3] = 1.0
    d = np.full((B, gamma), 3, np.int32)
    d[2:4] = 25
    rnd = OPH.philox_words(9, 0, B, gamma + 2)
    got = _run_accept(p, q, d, rnd, "sample")
    ref = OACC.spec_accept(p, q, d, rnd, "sample")
    assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    assert np.all(ref[1][:2] == gamma) and np.all(ref[1][2:4] == 0) and np.all(ref[0][4:, 0] == 9)


def test_determinism_bitwise():
    case = AttnCase(3, 32, 8, 128, 3000, [3000, 2500, 999], T=5, seed=21).to_cuda()
    a = _run_verify(case)
    b = _run_verify(case)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    c = _run_draft(case, 4, 1020)
    d = _run_draft(case, 4, 1020)
    assert np.array_equal(c[0], d[0]) and np.array_equal(c[1], d[1])


def test_calls_are_graph_capturable():
    """Every md_* call only enqueues work (no sync / alloc): a whole step captured in a CUDA
    graph and replayed gives bit-identical results to eager execution (P:722 uses graphs)."""
    case = AttnCase(4, 32, 8, 128, 2100, [2000, 1999, 1500, 700], T=5, seed=31).to_cuda()
    B, T, Hq, d = 4, 5, 32, 128
    mkl = 2090
    out_v = torch.zeros((B, T, Hq, d), device="cuda")
    out_d = torch.zeros((B, Hq, d), device="cuda")
    ws_v = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, 8, d, T, mkl)), dtype=torch.uint8, device="cuda")
    ws_d = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, 8, d, 1, 1024)), dtype=torch.uint8, device="cuda")
    kn = torch.zeros((B, T, 8, d), dtype=torch.bfloat16, device="cuda")
    start = torch.tensor([1995, 1994, 1495, 695], dtype=torch.int32, device="cuda")
    p, q, dt, rnd = _accept_inputs(B, 4, 500, 1.0, seed=2)
    pt, qt, dtt = torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda(), torch.from_numpy(dt).cuda()
    rt = torch.empty((B, 6), dtype=torch.int32, device="cuda")
    ot = torch.empty((B, 5), dtype=torch.int32, device="cuda")
    nt = torch.empty(B, dtype=torch.int32, device="cuda")

    def step():
        md.kv_append(case.k, case.v, kn, kn, start)
        md.draft_attn_sparse(case.qd, case.k, case.v, case.kv_len_t, 4, 1020, case.scale, out_d, None, ws_d)
        md.verify_attn_full(case.qv, case.k, case.v, case.kv_len_t, mkl, case.scale, out_v, None, ws_v)
        md.philox_u32(5, 1, rt)
        md.spec_accept(pt, qt, dtt, rt, ot, nt)

    step()
    torch.cuda.synchronize()
    ref = [x.clone() for x in (out_v, out_d, ot, nt)]
    for x in (out_v, out_d):
        x.zero_()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            step()
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(ref, (out_v, out_d, ot, nt)):
        assert torch.equal(a, b)


def test_verify_max_gamma_and_rows():
    """gamma = 15 (T = 16, the ABI maximum) with g = 4 -> 64 rows per KV head."""
    case = AttnCase(2, 16, 4, 128, 400, [400, 77], T=16, seed=41).to_cuda()
    o, l = _run_verify(case)
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    _cmp(o, l, ro, rl)


def test_stream_k_single_unit_spans_every_cta():
    """B=1, one KV head: the single unit's tiles are spread over the whole persistent grid,
    so its output is the merge of ~G partials (O6 across CTAs)."""
    case = AttnCase(1, 4, 1, 128, 40000, [39999], T=5, seed=51).to_cuda()
    o, l = _run_verify(case)
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    _cmp(o, l, ro, rl)
    o, l = _run_draft(case, 4, 30000)
    ro, rl = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, 4, 30000, case.scale)
    _cmp(o, l, ro, rl)


def test_stream_k_many_ragged_units():
    """Many short ragged units: CTA ranges cut units at arbitrary tiles and a CTA spans
    several units; lengths straddle tile boundaries (63/64/65) and equal T."""
    rng = np.random.default_rng(61)
    lens = rng.integers(5, 700, size=40)
    lens[:6] = [5, 63, 64, 65, 128, 129]
    case = AttnCase(40, 16, 2, 64, 704, lens, T=5, seed=61).to_cuda()
    o, l = _run_verify(case)
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    _cmp(o, l, ro, rl)
    o, l = _run_draft(case, 4, 100)
    ro, rl = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, 4, 100, case.scale)
    _cmp(o, l, ro, rl)


def test_workspace_reuse_across_calls():
    """The arrival counters are left at zero: back-to-back calls of different shapes on one
    zero-initialised workspace stay correct."""
    a = AttnCase(3, 32, 8, 128, 3000, [3000, 1700, 900], T=5, seed=71).to_cuda()
    b = AttnCase(2, 8, 8, 128, 5000, [5000, 4999], T=4, seed=72).to_cuda()
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    for case, T in ((a, 5), (b, 4), (a, 5), (b, 4)):
        out = torch.empty((case.B, T, case.Hq, case.d), device="cuda")
        lse = torch.empty((case.B, T, case.Hq), device="cuda")
        md.verify_attn_full(case.qv, case.k, case.v, case.kv_len_t, int(case.kv_len.max()), case.scale, out, lse, ws)
        od = torch.empty((case.B, case.Hq, case.d), device="cuda")
        md.draft_attn_sparse(case.qd, case.k, case.v, case.kv_len_t, 4, 1020, case.scale, od, None, ws)
        torch.cuda.synchronize()
        ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
        _cmp(out.cpu().numpy(), lse.cpu().numpy(), ro, rl)


def test_large_batch_uses_global_walk():
    """B > 1024 sequences (the in-CTA prefix table's limit): the CTA-range lookup falls back
    to walking kv_len in global memory."""
    rng = np.random.default_rng(81)
    lens = rng.integers(4, 150, size=1030)
    case = AttnCase(1030, 4, 1, 64, 152, lens, T=3, seed=81).to_cuda()
    o, l = _run_verify(case)
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    _cmp(o, l, ro, rl)
    o, l = _run_draft(case, 4, 60)
    ro, rl = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, 4, 60, case.scale)
    _cmp(o, l, ro, rl)


@pytest.mark.parametrize("Hq,Hkv,T", [(32, 8, 5), (28, 4, 16), (16, 2, 8)])
def test_verify_rising_scores_exercise_max_raises(Hq, Hkv, T):
    """Scores that climb by ~4 (log2 units) every 128 keys force the tcgen05 kernel's lazy
    max raise (threshold 2^8) again and again inside a segment, so the thread-local row sums
    and the O^T accumulator in TMEM are rescaled many times; also a falling sequence (the max
    is set by the first stage and never raised)."""
    B, d = 2, 128
    lens = [1500, 1100]
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, T=T, seed=97)
    one = S.k_to_bf16_bits(np.array([32]))[0]              # 1.0
    case.qv_bits[:] = one
    for b in range(B):
        for j in range(case.cap):
            level = min(j // 128, 63) * 8                    # 0.25 * (j // 128) on the k/32 grid
            val = S.k_to_bf16_bits(np.array([level]))[0]
            case.k_bits[b, :, j, :] = val if b == 0 else S.k_to_bf16_bits(np.array([max(0, 96 - level)]))[0]
    case.to_cuda()
    o, l = _run_verify(case)
    ro, rl = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    _cmp(o, l, ro, rl)
