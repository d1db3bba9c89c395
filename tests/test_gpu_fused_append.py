"""GPU parity of the fused append calls (md_verify_attn_full_append, md_draft_attn_sparse_append):
each must equal md_kv_append(start = kv_len - T) followed by the plain call, so the oracle is
oracle.attention.kv_append then oracle.attention.verify_attn_full / draft_attn_sparse on the
updated cache.  Outputs within the attention tolerance, the whole cache after the
call bit-exact.  The cache rows [n - T, n) hold other data before the call (the synth cache), so
a tile loaded before its new rows landed shows up as an output mismatch.
"""
import zlib

import numpy as np
import pytest
import torch

import paper_2408_11049_b200 as md
import synth as S
from oracle import attention as OA
from tests.helpers import AttnCase, bits_to_torch_bf16

pytestmark = pytest.mark.gpu

ATOL_O = 2e-3
ATOL_LSE = 1e-3


def _bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def _new_rows(seed, B, T, Hkv, d):
    kn = S.k_to_bf16_bits(S.new_kv_k(seed, S.T_KNEW, B, T, Hkv, d))
    vn = S.k_to_bf16_bits(S.new_kv_k(seed, S.T_VNEW, B, T, Hkv, d))
    return kn, vn


def _cmp(o, l, ro, rl):
    assert np.all(np.isfinite(o)) and np.all(np.isfinite(l))
    eo, el = np.max(np.abs(o - ro)), np.max(np.abs(l - rl))
    assert eo <= ATOL_O and el <= ATOL_LSE, (eo, el)


VERIFY_CASES = [
    # name,            B, Hq, Hkv,  d,  T, lengths                  kernel
    ("llama3_gqa",     3, 32, 8, 128, 5, [1500, 1497, 64]),      # tcgen05, R = 20
    ("qwen_gqa",       2, 28, 4, 128, 5, [2100, 777]),           # tcgen05, R = 35
    ("tc_generic_24",  2, 16, 4, 128, 6, [2000, 133]),           # tcgen05, runtime R = 24
    ("tile_straddle",  2, 32, 8, 128, 5, [130, 66]),             # new rows across a 64/128-key tile edge
    ("llama2_mha",     2, 32, 32, 128, 4, [1000, 517]),          # keys kernel (R = 4)
    ("decode_T1",      2, 32, 8, 128, 1, [300, 1]),              # keys kernel, n = T
    ("d64_rows",       4, 8, 2, 64, 3, [3, 65, 128, 129]),       # rows kernel: kv_append launch ahead
    ("mha_long",       4, 32, 32, 128, 4, [19000, 18000, 19005, 300]),  # keys kernel, long: append launch ahead
    ("tiny",           2, 4, 4, 64, 4, [256, 256]),
]


@pytest.mark.parametrize("name,B,Hq,Hkv,d,T,lens", VERIFY_CASES)
def test_verify_append_parity(name, B, Hq, Hkv, d, T, lens):
    seed = zlib.crc32(name.encode()) & 0xFFFF
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 7, lens, T=T, seed=seed).to_cuda()
    kn, vn = _new_rows(seed + 1, B, T, Hkv, d)
    mkl = int(case.kv_len.max())
    out = torch.full((B, T, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, T, Hq), float("nan"), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, mkl), dtype=torch.uint8, device="cuda")
    md.verify_attn_full_append(case.qv, case.k, case.v, bits_to_torch_bf16(kn), bits_to_torch_bf16(vn),
                               case.kv_len_t, mkl, case.scale, out, lse, ws)
    torch.cuda.synchronize()
    kc, vc = case.k_bits.copy(), case.v_bits.copy()
    OA.kv_append(kc, vc, kn, vn, case.kv_len - T)
    ro, rl = OA.verify_attn_full(case.qv_bits, kc, vc, case.kv_len, case.scale)
    _cmp(out.cpu().numpy(), lse.cpu().numpy(), ro, rl)
    assert np.array_equal(_bits(case.k), kc) and np.array_equal(_bits(case.v), vc)


DRAFT_CASES = [
    # name,           B, Hq, Hkv, d, lengths, sink, window
    ("llama3",        3, 32, 8, 128, [3000, 1025, 1024], 4, 1020),
    ("qwen",          2, 28, 4, 128, [4100, 2049], 4, 2044),
    ("llama2",        2, 32, 32, 128, [2000, 600], 4, 508),
    ("short_seq",     3, 8, 2, 64, [1, 5, 63], 4, 60),      # new row inside the sink rows (n <= sink)
    ("no_sink",       2, 8, 8, 64, [500, 90], 0, 77),
    ("window_1",      2, 8, 2, 128, [700, 3], 4, 1),        # the window is the new row alone
]


@pytest.mark.parametrize("name,B,Hq,Hkv,d,lens,sink,window", DRAFT_CASES)
def test_draft_append_parity(name, B, Hq, Hkv, d, lens, sink, window):
    seed = zlib.crc32(name.encode()) & 0xFFFF
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 3, lens, seed=seed).to_cuda()
    kn, vn = _new_rows(seed + 2, B, 1, Hkv, d)
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, Hq), float("nan"), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, sink + window), dtype=torch.uint8, device="cuda")
    md.draft_attn_sparse_append(case.qd, case.k, case.v, bits_to_torch_bf16(kn), bits_to_torch_bf16(vn),
                                case.kv_len_t, sink, window, case.scale, out, lse, ws)
    torch.cuda.synchronize()
    kc, vc = case.k_bits.copy(), case.v_bits.copy()
    OA.kv_append(kc, vc, kn, vn, case.kv_len - 1)
    ro, rl = OA.draft_attn_sparse(case.qd_bits, kc, vc, case.kv_len, sink, window, case.scale)
    _cmp(out.cpu().numpy(), lse.cpu().numpy(), ro, rl)
    assert np.array_equal(_bits(case.k), kc) and np.array_equal(_bits(case.v), vc)


def test_fused_step_sequence():
    """One speculation step of one layer through the fused calls, back to back on one stream
    (gamma draft calls, each appending its row, then the verify call overwriting those rows):
    every call's output and the final cache against the oracle's kv_append + attention chain."""
    B, Hq, Hkv, d, gamma, sink, window = 3, 32, 8, 128, 4, 4, 1020
    T = gamma + 1
    L = np.array([3000, 1100, 1021], dtype=np.int32)
    case = AttnCase(B, Hq, Hkv, d, int(L.max()) + T + 3, L + T, T=T, seed=77).to_cuda()
    kc, vc = case.k_bits.copy(), case.v_bits.copy()
    wsd = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, sink + window), dtype=torch.uint8, device="cuda")
    wsv = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, int(L.max()) + T), dtype=torch.uint8, device="cuda")
    outs, refs = [], []
    for j in range(gamma):
        kn, vn = _new_rows(100 + j, B, 1, Hkv, d)
        n = (L + j + 1).astype(np.int32)
        out = torch.empty((B, Hq, d), device="cuda")
        lse = torch.empty((B, Hq), device="cuda")
        md.draft_attn_sparse_append(case.qd, case.k, case.v, bits_to_torch_bf16(kn), bits_to_torch_bf16(vn),
                                    torch.from_numpy(n).cuda(), sink, window, case.scale, out, lse, wsd)
        outs.append((out, lse))
        OA.kv_append(kc, vc, kn, vn, n - 1)
        refs.append(OA.draft_attn_sparse(case.qd_bits, kc, vc, n, sink, window, case.scale))
    kn, vn = _new_rows(200, B, T, Hkv, d)
    n = (L + T).astype(np.int32)
    out = torch.empty((B, T, Hq, d), device="cuda")
    lse = torch.empty((B, T, Hq), device="cuda")
    md.verify_attn_full_append(case.qv, case.k, case.v, bits_to_torch_bf16(kn), bits_to_torch_bf16(vn),
                               torch.from_numpy(n).cuda(), int(n.max()), case.scale, out, lse, wsv)
    outs.append((out, lse))
    OA.kv_append(kc, vc, kn, vn, n - T)
    refs.append(OA.verify_attn_full(case.qv_bits, kc, vc, n, case.scale))
    torch.cuda.synchronize()
    for (o, l), (ro, rl) in zip(outs, refs):
        _cmp(o.cpu().numpy(), l.cpu().numpy(), ro, rl)
    assert np.array_equal(_bits(case.k), kc) and np.array_equal(_bits(case.v), vc)


def test_fused_append_rejects_bad_args():
    case = AttnCase(2, 8, 2, 128, 300, [200, 100]).to_cuda()
    kn = torch.zeros((2, 1, 2, 128), dtype=torch.bfloat16, device="cuda")
    kn_wide = torch.zeros((2, 1, 2, 256), dtype=torch.bfloat16, device="cuda")  # a non-contiguous view
    out = torch.empty((2, 8, 128), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(2, 8, 2, 128, 1, 64), dtype=torch.uint8, device="cuda")
    with pytest.raises(md.MDError, match="window >= 1"):
        md.draft_attn_sparse_append(case.qd, case.k, case.v, kn, kn, case.kv_len_t, 4, 0, case.scale, out, None, ws)
    with pytest.raises(ValueError):
        md.draft_attn_sparse_append(case.qd, case.k, case.v, kn_wide[..., :128], kn, case.kv_len_t, 4, 60,
                                    case.scale, out, None, ws)


def test_fused_calls_in_a_cuda_graph():
    """The fused calls only enqueue work: gamma draft calls + the verify call captured in one
    CUDA graph and replayed give bit-identical outputs and cache to eager execution."""
    B, Hq, Hkv, d, gamma, sink, window = 3, 32, 8, 128, 4, 4, 1020
    T = gamma + 1
    L = np.array([2500, 1300, 900], dtype=np.int32)
    case = AttnCase(B, Hq, Hkv, d, int(L.max()) + T + 3, L + T, T=T, seed=5).to_cuda()
    k0, v0 = case.k.clone(), case.v.clone()
    news = [tuple(bits_to_torch_bf16(x) for x in _new_rows(300 + j, B, 1, Hkv, d)) for j in range(gamma)]
    newv = tuple(bits_to_torch_bf16(x) for x in _new_rows(400, B, T, Hkv, d))
    lens = [torch.from_numpy((L + j + 1).astype(np.int32)).cuda() for j in range(gamma)]
    lenv = torch.from_numpy((L + T).astype(np.int32)).cuda()
    wsd = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, sink + window), dtype=torch.uint8, device="cuda")
    wsv = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, int(L.max()) + T), dtype=torch.uint8, device="cuda")
    outs = [torch.zeros((B, Hq, d), device="cuda") for _ in range(gamma)]
    outv = torch.zeros((B, T, Hq, d), device="cuda")

    def step():
        for j in range(gamma):
            md.draft_attn_sparse_append(case.qd, case.k, case.v, news[j][0], news[j][1], lens[j], sink, window,
                                        case.scale, outs[j], None, wsd)
        md.verify_attn_full_append(case.qv, case.k, case.v, newv[0], newv[1], lenv, int(L.max()) + T, case.scale,
                                   outv, None, wsv)

    step()
    torch.cuda.synchronize()
    ref = [x.clone() for x in outs + [outv, case.k, case.v]]
    for x in outs + [outv]:
        x.zero_()
    case.k.copy_(k0)
    case.v.copy_(v0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            step()
    torch.cuda.synchronize()
    case.k.copy_(k0)  # capture does not execute; reset anyway so the replay starts from the same cache
    case.v.copy_(v0)
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(ref, outs + [outv, case.k, case.v]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("B,Hq,Hkv,d,lens,counts,stride,win", [
    (3, 32, 8, 128, [3000, 2000, 700], [500, 130, 0], 512, 32),
    (2, 28, 4, 128, [5000, 4100], [2017, 2017], 2020, 32),
    (4, 8, 8, 64, [300, 200, 150, 90], [61, 64, 65, 3], 68, 7),
    (2, 4, 1, 128, [9000, 40], [1000, 8], 1000, 1),           # the tail is the new row alone
    (3, 32, 8, 128, [3000, 700, 64], [100, 700, 64], 704, 0),  # no tail: the new row is a LISTED row
])
def test_indexed_draft_append_parity(B, Hq, Hkv, d, lens, counts, stride, win):
    """md_draft_attn_indexed_append (SnapKV drafting, f2) = kv_append(kv_len - 1) + the indexed draft."""
    from oracle import snapkv as SK
    rng = np.random.default_rng(sum(lens) + 1)
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, seed=B * 11 + Hq).to_cuda()
    tails = (np.asarray(lens) - win).astype(np.int32)
    counts = np.minimum(np.asarray(counts), tails).astype(np.int32)
    idx = np.full((B, Hkv, stride), -1, np.int32)
    for b in range(B):
        for h in range(Hkv):
            if win == 0:  # tail_start = kv_len: list the new row n - 1 itself (PQ select with window 0)
                pick = rng.choice(int(tails[b]) - 1, size=int(counts[b]) - 1, replace=False)
                idx[b, h, :counts[b]] = np.sort(np.append(pick, tails[b] - 1))
            else:
                idx[b, h, :counts[b]] = np.sort(rng.choice(int(tails[b]), size=int(counts[b]), replace=False))
    kn, vn = _new_rows(B + 9, B, 1, Hkv, d)
    out = torch.full((B, Hq, d), float("nan"), device="cuda")
    lse = torch.full((B, Hq), float("nan"), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, case.cap), dtype=torch.uint8, device="cuda")
    md.draft_attn_indexed(case.qd, case.k, case.v, case.kv_len_t, torch.from_numpy(idx).cuda(),
                          torch.from_numpy(counts).cuda(), torch.from_numpy(tails).cuda(), case.scale, out, lse, ws,
                          k_new=bits_to_torch_bf16(kn), v_new=bits_to_torch_bf16(vn))
    torch.cuda.synchronize()
    kc, vc = case.k_bits.copy(), case.v_bits.copy()
    OA.kv_append(kc, vc, kn, vn, case.kv_len - 1)
    ro, rl = SK.draft_attn_indexed(case.qd_bits, kc, vc, case.kv_len, idx, counts, tails, case.scale)
    _cmp(out.cpu().numpy(), lse.cpu().numpy(), ro, rl)
    assert np.array_equal(_bits(case.k), kc) and np.array_equal(_bits(case.v), vc)


@pytest.mark.parametrize("B,Hq,Hkv,d,lens,sink,window", [
    (3, 32, 8, 128, [3000, 1100, 70], 4, 1020),     # long, medium, a unit of 2 tiles (new row in the 2nd)
    (2, 28, 4, 128, [2500, 40], 4, 2044),           # Qwen2.5 group of 7; a single-tile unit
    (4, 32, 32, 128, [900, 800, 513, 2], 4, 508),   # MHA (Llama-2); n = 2
    (2, 4, 4, 64, [256, 255], 4, 60),               # head_dim 64
])
def test_draft_append_early_kv_bit_identical(B, Hq, Hkv, d, lens, sink, window):
    """MD_ATTN_EARLY_KV (md_draft_attn_sparse_append_ex): the producer streams a unit's first tiles
    before the grid-dependency wait.  A chain of draft steps over 4 layer caches, back to back on
    one stream as in bench.py (each call's predecessor appends into another cache), with and
    without the flag: every output and both caches bit-identical, and the last call against the
    oracle."""
    R, steps = 4, 3
    L = np.array(lens, dtype=np.int32)
    cap = int(L.max()) + steps + 3

    def run(early):
        cases = [AttnCase(B, Hq, Hkv, d, cap, L + steps, seed=300 + r).to_cuda() for r in range(R)]
        ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, sink + window), dtype=torch.uint8, device="cuda")
        outs = []
        for j in range(steps):
            kn, vn = _new_rows(400 + j, B, 1, Hkv, d)
            kn_t, vn_t = bits_to_torch_bf16(kn), bits_to_torch_bf16(vn)
            n_t = torch.from_numpy((L + j + 1).astype(np.int32)).cuda()
            for r in range(R):
                out = torch.empty((B, Hq, d), device="cuda")
                lse = torch.empty((B, Hq), device="cuda")
                md.draft_attn_sparse_append(cases[r].qd, cases[r].k, cases[r].v, kn_t, vn_t, n_t, sink, window,
                                            cases[r].scale, out, lse, ws, early_kv=early)
                outs.append((out, lse))
        torch.cuda.synchronize()
        return cases, [(o.cpu().numpy(), l.cpu().numpy()) for o, l in outs]

    ce, oe = run(True)
    cp, op = run(False)
    for (a, b), (c, e) in zip(oe, op):
        assert np.array_equal(a.view(np.uint32), c.view(np.uint32)) and np.array_equal(b.view(np.uint32),
                                                                                     e.view(np.uint32))
    for x, y in zip(ce, cp):
        assert np.array_equal(_bits(x.k), _bits(y.k)) and np.array_equal(_bits(x.v), _bits(y.v))
    # the last call (step steps-1, cache R-1) against the oracle chain of that cache
    c = AttnCase(B, Hq, Hkv, d, cap, L + steps, seed=300 + R - 1)
    kc, vc = c.k_bits.copy(), c.v_bits.copy()
    for j in range(steps):
        kn, vn = _new_rows(400 + j, B, 1, Hkv, d)
        OA.kv_append(kc, vc, kn, vn, (L + j).astype(np.int32))
    ro, rl = OA.draft_attn_sparse(c.qd_bits, kc, vc, (L + steps).astype(np.int32), sink, window, c.scale)
    _cmp(oe[-1][0], oe[-1][1], ro, rl)
    assert np.array_equal(_bits(ce[-1].k), kc) and np.array_equal(_bits(ce[-1].v), vc)


def test_draft_append_ex_rejects_unknown_flags():
    B, Hq, Hkv, d = 2, 8, 2, 128
    case = AttnCase(B, Hq, Hkv, d, 300, [300, 200], seed=5).to_cuda()
    kn = bits_to_torch_bf16(_new_rows(1, B, 1, Hkv, d)[0])
    lib = md.load_library()
    c = md.make_cache(case.k, case.v)
    out = torch.empty((B, Hq, d), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, 64), dtype=torch.uint8, device="cuda")
    import ctypes
    st = lib.md_draft_attn_sparse_append_ex(ctypes.byref(c), case.qd.data_ptr(), Hq, kn.data_ptr(), kn.data_ptr(),
                                            case.kv_len_t.data_ptr(), 4, 60, 0.1, out.data_ptr(), None,
                                            ws.data_ptr(), ws.numel(), 6, None)
    assert st == md.MD_ERR_INVALID_ARG and b"unknown flags" in lib.md_last_error()
