"""GPU parity of PQCache dynamic selection (md_pq_encode / md_pq_select)
against the oracle (oracle/pqcache.py P1-P5): codes, index lists, counts and tail starts are
integers decided in the same fp32 / integer arithmetic on both sides, so they must match
bit for bit; the draft over the selected set must match the fp64 draft within 2e-3."""
import numpy as np
import pytest
import torch

import paper_2408_11049_b200 as md
import synth as S
from oracle import pqcache as PQ
from oracle import snapkv as SK
from tests.helpers import AttnCase, bits_to_torch_bf16

pytestmark = pytest.mark.gpu
ATOL_O, ATOL_LSE = 2e-3, 1e-3


def _rand_bf16(rng, shape, scale=0.5):
    """Random bf16 bit patterns off the k/32 grid (fp32 rounding matters for these)."""
    f = (rng.standard_normal(shape) * scale).astype(np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def _codebook(case, L, rng=None):
    if rng is None:
        return S.pq_codebook_bits(case.k_bits, S.pq_codebook_positions(case.seed, case.B, case.Hkv, L))
    return _rand_bf16(rng, (case.B, case.Hkv, 16, 256, case.d // 16), 0.3)


def _encode_gpu(case, cb, start, count, code_cap):
    codes = torch.zeros((case.B, case.Hkv, code_cap, 16), dtype=torch.uint8, device="cuda")
    md.pq_encode(case.k, case.v, bits_to_torch_bf16(cb), torch.from_numpy(np.asarray(start, np.int32)).cuda(),
                 count, codes)
    torch.cuda.synchronize()
    return codes


@pytest.mark.parametrize("B,Hkv,d,n,grid_cb", [(2, 3, 128, 700, True), (2, 2, 128, 600, False),
                                               (3, 2, 64, 530, False)])
def test_encode_bit_exact(B, Hkv, d, n, grid_cb):
    rng = np.random.default_rng(n)
    case = AttnCase(B, 2 * Hkv, Hkv, d, n + 40, [n] * B, seed=n, regime=S.Regime("peaky", sink=4)).to_cuda()
    if not grid_cb:  # off-grid keys too: every fp32 rounding step must agree
        case.k_bits = _rand_bf16(rng, case.k_bits.shape, 0.4)
        case.k = bits_to_torch_bf16(case.k_bits)
    cb = _codebook(case, [n] * B, None if grid_cb else rng)
    start = np.array([0, 13, 5][:B], np.int32)
    count = n - 20
    codes = _encode_gpu(case, cb, start, count, n + 40).cpu().numpy()
    ref = PQ.pq_encode_cache(case.k_bits, cb, start, count)
    for b in range(B):
        assert np.array_equal(codes[:, :, start[b]:start[b] + count][b], ref[b])
        # rows outside [start, start + count) untouched
        assert not codes[b, :, :start[b]].any() and not codes[b, :, start[b] + count:].any()


def _select_gpu(case, q_bits, cb, codes_t, sink, window, budget, max_kv):
    B, Hkv = case.B, case.Hkv
    K = (sink + budget + 3) // 4 * 4
    idx = torch.full((B, Hkv, K), -1, dtype=torch.int32, device="cuda")
    cnt = torch.full((B,), -7, dtype=torch.int32, device="cuda")
    tail = torch.full((B,), -7, dtype=torch.int32, device="cuda")
    md.pq_select(bits_to_torch_bf16(q_bits), bits_to_torch_bf16(cb), codes_t, case.kv_len_t, max_kv, sink, window,
                 budget, idx, cnt, tail)
    torch.cuda.synchronize()
    return idx, cnt, tail


def _check_select(case, q_bits, cb, codes_np, idx, cnt, tail, sink, window, budget):
    ridx, rcnt, rtail, _ = PQ.pq_select(q_bits, cb, codes_np, case.kv_len, sink, window, budget)
    idx, cnt, tail = idx.cpu().numpy(), cnt.cpu().numpy(), tail.cpu().numpy()
    assert np.array_equal(cnt, rcnt) and np.array_equal(tail, rtail)
    for b in range(case.B):
        assert np.array_equal(idx[b, :, :cnt[b]], ridx[b, :, :rcnt[b]])
        assert (idx[b, :, cnt[b]:] == -1).all()  # untouched


@pytest.mark.parametrize("B,Hq,Hkv,d,lens,sink,window,budget,offgrid", [
    (3, 32, 8, 128, [3000, 2000, 700], 4, 252, 256, False),
    (2, 28, 4, 128, [5000, 4100], 4, 512, 1530, True),       # g = 7
    (4, 8, 8, 64, [300, 200, 150, 9], 4, 60, 64, True),      # MHA d=64; b=3: n <= sink + window
    (2, 4, 1, 128, [9000, 40], 0, 100, 5000, False),          # no sink; budget covers b=1
    (2, 16, 1, 128, [1500, 700], 4, 20, 100, True),           # g = 16
])
def test_select_bit_exact(B, Hq, Hkv, d, lens, sink, window, budget, offgrid):
    rng = np.random.default_rng(sum(lens))
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, seed=B * 5 + Hq, regime=S.Regime("peaky", sink=4)).to_cuda()
    cb = _codebook(case, lens, rng if offgrid else None)
    q_bits = _rand_bf16(rng, case.qd_bits.shape, 1.0) if offgrid else case.qd_bits
    codes_np = PQ.pq_encode_cache(case.k_bits, cb, np.zeros(B, np.int64), max(lens))
    codes_t = torch.from_numpy(np.pad(codes_np, ((0, 0), (0, 0), (0, 8), (0, 0)))).cuda()
    idx, cnt, tail = _select_gpu(case, q_bits, cb, codes_t, sink, window, budget, max(lens))
    _check_select(case, q_bits, cb, codes_np, idx, cnt, tail, sink, window, budget)


def test_select_ties_and_global_path():
    """All codes equal -> all scores tie -> the lowest candidate positions; n = 60000 > the
    shared-memory staging bound exercises the global-memory radix path."""
    B, Hq, Hkv, d, n = 1, 4, 2, 128, 60000
    case = AttnCase(B, Hq, Hkv, d, n + 8, [n], seed=3).to_cuda()
    rng = np.random.default_rng(3)
    cb = _rand_bf16(rng, (B, Hkv, 16, 256, 8))
    codes_np = np.zeros((B, Hkv, n + 8, 16), np.uint8)
    codes_np[:, :, 40000:40010] = 7                    # a few distinct keys, the rest tie
    codes_t = torch.from_numpy(codes_np).cuda()
    idx, cnt, tail = _select_gpu(case, case.qd_bits, cb, codes_t, 4, 1000, 2000, n)
    _check_select(case, case.qd_bits, cb, codes_np[:, :, :n], idx, cnt, tail, 4, 1000, 2000)
    codes_np = rng.integers(0, 256, size=(B, Hkv, n + 8, 16)).astype(np.uint8)
    idx, cnt, tail = _select_gpu(case, case.qd_bits, cb, torch.from_numpy(codes_np).cuda(), 4, 1000, 2000, n)
    _check_select(case, case.qd_bits, cb, codes_np[:, :, :n], idx, cnt, tail, 4, 1000, 2000)


def test_pq_draft_end_to_end():
    """encode + select + md_draft_attn_indexed on the GPU vs the oracle's encode + select + draft."""
    B, Hq, Hkv, d, lens = 3, 32, 8, 128, [4000, 3100, 2500]
    sink, window, budget = 4, 124, 380
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, seed=21, regime=S.Regime("peaky", sink=4)).to_cuda()
    cb = _codebook(case, lens)
    codes_t = _encode_gpu(case, cb, np.zeros(B, np.int32), max(lens), max(lens) + 8)
    idx, cnt, tail = _select_gpu(case, case.qd_bits, cb, codes_t, sink, window, budget, max(lens))
    out = torch.empty((B, Hq, d), device="cuda")
    lse = torch.empty((B, Hq), device="cuda")
    ws = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, 1, max(lens))), dtype=torch.uint8, device="cuda")
    md.draft_attn_indexed(case.qd, case.k, case.v, case.kv_len_t, idx, cnt, tail, case.scale, out, lse, ws)
    torch.cuda.synchronize()
    codes_np = PQ.pq_encode_cache(case.k_bits, cb, np.zeros(B, np.int64), max(lens))
    ridx, rcnt, rtail, _ = PQ.pq_select(case.qd_bits, cb, codes_np, case.kv_len, sink, window, budget)
    ro, rl = SK.draft_attn_indexed(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, ridx, rcnt, rtail, case.scale)
    assert np.max(np.abs(out.cpu().numpy() - ro)) <= ATOL_O
    assert np.max(np.abs(lse.cpu().numpy() - rl)) <= ATOL_LSE


def test_pq_fullsize_sampled_units():
    """BASELINE target shape (Llama-3.1-8B GQA, B=64, ctx 32k, budget 1024 = 4 sink + 508 top-k +
    512 window): the GPU encodes and selects for the whole batch; the oracle recomputes the codes
    and the selection of sampled (b, kv head) units from the seeded generator and must agree."""
    B, Hq, Hkv, d, ctx = 64, 32, 8, 128, 32768
    sink, window, budget = 4, 512, 508
    reg = S.Regime("peaky", sink=4)
    L = S.committed_lengths(7, B, ctx, 4, ragged=True)
    cap = ctx + 16
    k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda")
    import synth.cuda as SC
    SC.fill_cache(k, 7, S.T_KCACHE, 0, cap, reg)
    q = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_q(q, 7, S.T_QDRAFT, Hkv, reg)
    pos = torch.from_numpy(S.pq_codebook_positions(7, B, Hkv, L)).cuda()
    # codebook = key sub-vectors at hashed positions (input generation, gathered on the device)
    bi = torch.arange(B, device="cuda")[:, None, None, None]
    ui = torch.arange(Hkv, device="cuda")[None, :, None, None]
    rows = k[bi, ui, pos]                                          # [B, Hkv, 16, 256, d]
    cb = torch.stack([rows[:, :, m, :, m * 8:(m + 1) * 8] for m in range(16)], dim=2).contiguous()
    del rows
    codes = torch.zeros((B, Hkv, cap, 16), dtype=torch.uint8, device="cuda")
    md.pq_encode(k, k, cb, torch.zeros(B, dtype=torch.int32, device="cuda"), ctx, codes)
    kv_len = torch.from_numpy(L.astype(np.int32)).cuda()
    K = sink + budget
    idx = torch.full((B, Hkv, K), -1, dtype=torch.int32, device="cuda")
    cnt = torch.empty(B, dtype=torch.int32, device="cuda")
    tail = torch.empty(B, dtype=torch.int32, device="cuda")
    md.pq_select(q, cb, codes, kv_len, ctx, sink, window, budget, idx, cnt, tail)
    torch.cuda.synchronize()
    q_np = S.k_to_bf16_bits(S.q_rows_k(7, S.T_QDRAFT, B, 1, Hq, Hkv, d, regime=reg))[:, 0]
    g = Hq // Hkv
    for b, u in ((0, 0), (37, 5), (63, 7)):
        n = int(L[b])
        kb = S.k_to_bf16_bits(S.kv_cache_k(7, S.T_KCACHE, B, Hkv, d, 0, n, b_sel=[b], h_sel=[u], regime=reg))[0, 0]
        p = S.pq_codebook_positions(7, B, Hkv, L)[b, u]
        cb_np = np.stack([kb[p[m], m * 8:(m + 1) * 8] for m in range(16)])    # [16, 256, 8]
        assert np.array_equal(cb[b, u].cpu().view(torch.int16).numpy().view(np.uint16), cb_np)
        codes_np = PQ.pq_encode(kb, cb_np)
        assert np.array_equal(codes[b, u, :n].cpu().numpy(), codes_np)
        lutq = PQ.pq_lut_fixed(PQ.pq_lut(q_np[b, u * g:(u + 1) * g], cb_np))
        sc = PQ.pq_scores(lutq, codes_np)
        s0, t0, c = PQ.select_window(n, sink, window, budget)
        want = np.concatenate([np.arange(s0), PQ.select_topk(sc, s0, t0, c)])
        assert int(cnt[b]) == s0 + c and int(tail[b]) == t0
        assert np.array_equal(idx[b, u, :s0 + c].cpu().numpy(), want)


def test_gpu_pq_against_the_fp64_definition_offgrid():
    """The GPU path against the plain PQ definition, independently of the oracle's fixed-point
    arithmetic (16 sub-vectors x 8-bit codes; readings Z25-Z29): on off-grid bf16 keys,
    queries and codebooks, (1) every GPU code is the fp64 nearest centroid up to the fp32 rounding
    bound of the squared distance, (2) the GPU selection is the exact top-k of the fp64 PQ scores
    q . k_hat computed from the GPU's own codes, except positions whose score ties the k-th within
    twice the derived score bound (the check of test_oracle_pqcache, applied to the GPU)."""
    U = 2.0 ** -24
    rng = np.random.default_rng(31)
    B, Hq, Hkv, d, g = 2, 16, 4, 128, 4
    s = d // 16
    lens = [2500, 1800]
    sink, window, budget = 4, 128, 300
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, seed=31)
    case.k_bits = _rand_bf16(rng, case.k_bits.shape, 1.0)
    case.to_cuda()
    cb = _rand_bf16(rng, (B, Hkv, 16, 256, s), 1.0)
    q_bits = _rand_bf16(rng, case.qd_bits.shape, 1.0)
    codes = _encode_gpu(case, cb, np.zeros(B), max(lens), max(lens) + 8)
    idx, cnt, tail = _select_gpu(case, q_bits, cb, codes, sink, window, budget, max(lens))
    codes = codes.cpu().numpy()
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    f64 = lambda bits: S.bf16_bits_to_f32(bits).astype(np.float64)
    ncode_diff = nsel_diff = 0
    for b in range(B):
        nb = lens[b]
        s0, t0 = min(sink, nb), max(min(sink, nb), nb - window)
        c = min(budget, t0 - s0)
        assert int(cnt[b]) == s0 + c and idx[b, 0, :s0].tolist() == list(range(s0))
        for u in range(Hkv):
            X, C = f64(case.k_bits[b, u, :nb]), f64(cb[b, u])
            for m in range(16):
                diff = X[:, None, m * s:(m + 1) * s] - C[m][None]
                dist = (diff ** 2).sum(-1)
                best = np.argmin(dist, axis=1)
                bound = (s + 2) * U * dist
                gc = codes[b, u, :nb, m].astype(np.int64)
                bad = np.nonzero(gc != best)[0]
                ncode_diff += len(bad)
                for j in bad:
                    assert dist[j, gc[j]] - dist[j, best[j]] <= bound[j, gc[j]] + bound[j, best[j]], (b, u, m, j)
            Q = f64(q_bits[b, u * g:(u + 1) * g])
            khat = np.concatenate([C[m][codes[b, u, :nb, m]] for m in range(16)], axis=1)
            exact = khat @ Q.sum(0)
            absterm = np.stack([np.abs(C[m]) @ np.abs(Q[:, m * s:(m + 1) * s]).sum(0) for m in range(16)])
            lut_max = max(float(np.max(np.abs(C[m] @ Q[:, m * s:(m + 1) * s].sum(0)))) for m in range(16))
            e = 26 - int(np.frexp(lut_max)[1])
            ent = 2 * g * s * U * absterm + 2.0 ** -e  # rint to the 2^-e grid, e within 1 of the fp64 max's
            sbound = sum(ent[m][codes[b, u, :nb, m]] for m in range(16))
            cand = np.arange(s0, t0)
            ref = set(sorted(cand.tolist(), key=lambda j: (-exact[j], j))[:c])
            got = set(idx[b, u, s0:s0 + c].tolist())
            thr = np.sort(exact[s0:t0])[::-1][c - 1]
            for x in ref ^ got:
                nsel_diff += 1
                assert abs(exact[x] - thr) <= 2 * sbound.max(), (b, u, x)
    assert ncode_diff <= B * Hkv * 16 * max(lens) * 1e-3
    assert nsel_diff <= 8


@pytest.mark.parametrize("ties", [False, True])
def test_select_many_units_256_thread_variant(ties):
    """More units than one wave of 512-thread select CTAs (2 per SM): the 256-thread variant with
    the 1024-key tie list (4 CTAs per SM).  ties=True: every unit's scores tie except a few keys,
    so the cutoff bin overflows the tie list and the global-memory refinement runs."""
    B, Hq, Hkv, d = 40, 32, 8, 128
    units = B * Hkv
    assert units > 2 * torch.cuda.get_device_properties(0).multi_processor_count
    rng = np.random.default_rng(77 + ties)
    lens = list(rng.integers(900, 2600, size=B))
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, seed=78, regime=S.Regime("peaky", sink=4)).to_cuda()
    cb = _codebook(case, lens, rng)
    q_bits = _rand_bf16(rng, case.qd_bits.shape, 1.0)
    if ties:
        codes_np = np.zeros((B, Hkv, max(lens), 16), np.uint8)
        codes_np[:, :, 300:305] = 9
    else:
        codes_np = PQ.pq_encode_cache(case.k_bits, cb, np.zeros(B, np.int64), max(lens))
    codes_t = torch.from_numpy(np.pad(codes_np, ((0, 0), (0, 0), (0, 8), (0, 0)))).cuda()
    idx, cnt, tail = _select_gpu(case, q_bits, cb, codes_t, 4, 252, 508, max(lens))
    _check_select(case, q_bits, cb, codes_np, idx, cnt, tail, 4, 252, 508)
