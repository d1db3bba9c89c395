"""Pins for the PQCache dynamic-selection oracle (P:1141 footnote "PQCache
employs product quantization with 16 sub-vectors and 8-bit quantization per key vector";
P:1132-1137 dynamic selection searches for each query's nearest keys).

What fixes each step independently of the oracle's own code:
  P1 encode      brute-force nearest centroid in fp64 on exact-grid inputs (the fp32
                 procedure can only differ where fp32 rounds, which exact-grid inputs never
                 do), keys placed on centroids, duplicate centroids (ties -> lowest index);
  P2-P4 scores   on exact-grid inputs score * 2^-e equals the PQ inner product
                 sum_hh q_hh . khat_j computed in fp64 from the reconstructed keys khat;
  P5 selection   brute-force set logic; with keys that the codebook reconstructs exactly the
                 selection is exact top-k attention by the group's true logits; a budget that
                 covers the range reduces the draft to full attention (bit-identical).
"""
import numpy as np

import synth as S
from oracle import attention as OA
from oracle import pqcache as PQ
from oracle import snapkv as SK


def _grid_bits(rng, shape, lo=-32, hi=32):
    return S.k_to_bf16_bits(rng.integers(lo, hi, size=shape))


def _f64(bits):
    return S.bf16_bits_to_f32(bits).astype(np.float64)


def test_encode_matches_fp64_nearest_centroid():
    rng = np.random.default_rng(1)
    for d in (64, 128):
        s = d // 16
        k = _grid_bits(rng, (300, d))
        cb = _grid_bits(rng, (16, 256, s))
        codes = PQ.pq_encode(k, cb)
        x, C = _f64(k), _f64(cb)
        for m in range(16):
            dist = ((x[:, None, m * s:(m + 1) * s] - C[m][None]) ** 2).sum(-1)   # [n, 256] exact
            assert np.array_equal(codes[:, m], np.argmin(dist, axis=1))


def test_encode_keys_on_centroids_and_ties():
    rng = np.random.default_rng(2)
    d, s = 128, 8
    cb = _grid_bits(rng, (16, 256, s))
    cb[:, 200] = cb[:, 17]                          # duplicate centroid: 17 must win
    want = rng.integers(0, 256, size=(50, 16))
    want[0, :] = 200
    k = np.zeros((50, d), dtype=np.uint16)
    for j in range(50):
        for m in range(16):
            k[j, m * s:(m + 1) * s] = cb[m, want[j, m]]
    codes = PQ.pq_encode(k, cb)
    expect = np.where(want == 200, 17, want)
    # other accidental duplicates among random grid centroids resolve to their lowest index too
    for m in range(16):
        for j in range(50):
            same = np.nonzero((cb[m] == cb[m, expect[j, m]]).all(-1))[0]
            expect[j, m] = same.min()
    assert np.array_equal(codes, expect)


def test_scores_equal_pq_inner_product_on_grid():
    rng = np.random.default_rng(3)
    for d, g in ((128, 4), (64, 1), (128, 7)):
        s = d // 16
        q = _grid_bits(rng, (g, d))
        cb = _grid_bits(rng, (16, 256, s))
        codes = rng.integers(0, 256, size=(400, 16)).astype(np.uint8)
        lut = PQ.pq_lut(q, cb)
        e = PQ.lut_exponent(lut)
        sc = PQ.pq_scores(PQ.pq_lut_fixed(lut), codes)
        khat = np.concatenate([_f64(cb)[m][codes[:, m]] for m in range(16)], axis=1)   # [n, d]
        exact = khat @ _f64(q).sum(0)                                                 # sum_hh q_hh . khat
        assert np.array_equal(sc.astype(np.float64) * 2.0 ** -e, exact)


def test_fixed_point_table_range():
    rng = np.random.default_rng(4)
    for scale in (1e-3, 1.0, 37.5):
        lut = (rng.standard_normal((16, 256)) * scale).astype(np.float32)
        lq = PQ.pq_lut_fixed(lut)
        assert np.abs(lq).max() < 2 ** 26 and np.abs(lq).max() >= 2 ** 24
    assert PQ.lut_exponent(np.zeros((16, 256), np.float32)) == 0
    assert PQ.lut_exponent(np.full((16, 256), 1.0, np.float32)) == 25    # 1.0 = 0.5 * 2^1
    assert PQ.lut_exponent(np.full((16, 256), 0.75, np.float32)) == 26   # 0.75 = 0.75 * 2^0


def test_select_window_and_ties():
    assert PQ.select_window(100, 4, 20, 30) == (4, 80, 30)
    assert PQ.select_window(100, 4, 20, 500) == (4, 80, 76)
    assert PQ.select_window(3, 4, 20, 30) == (3, 3, 0)       # short sequence: all sink
    assert PQ.select_window(30, 4, 40, 8) == (4, 4, 0)       # window covers the rest
    sc = np.array([5, 1, 7, 7, 3, 7, 0, 7], dtype=np.int64)
    assert PQ.select_topk(sc, 1, 8, 3).tolist() == [2, 3, 5]  # the 7s, lowest positions first
    assert PQ.select_topk(sc, 0, 8, 8).tolist() == list(range(8))
    assert PQ.select_topk(np.zeros(10, np.int64), 2, 9, 4).tolist() == [2, 3, 4, 5]


def _exact_codebook_case(rng, B, Hkv, g, d, n):
    """Keys whose sub-vectors are all centroids (the codebook reconstructs them exactly)."""
    s = d // 16
    cb = _grid_bits(rng, (B, Hkv, 16, 256, s))
    codes = rng.integers(0, 256, size=(B, Hkv, n, 16)).astype(np.uint8)
    k = np.zeros((B, Hkv, n, d), dtype=np.uint16)
    for m in range(16):
        k[..., m * s:(m + 1) * s] = np.take_along_axis(cb[:, :, m], codes[..., m:m + 1].astype(np.int64), axis=2)
    q = _grid_bits(rng, (B, Hkv * g, d))
    return q, cb, codes, k


def test_exact_reconstruction_selects_true_topk_logits():
    """PQ with zero quantisation error is exact top-k attention (the paper's Top-K drafter,
    P:1132): the selected set equals the brute-force top-k of the group's true logit sums."""
    rng = np.random.default_rng(5)
    B, Hkv, g, d, n = 2, 2, 4, 128, 300
    sink, window, budget = 4, 40, 25
    q, cb, codes, k = _exact_codebook_case(rng, B, Hkv, g, d, n)
    enc = PQ.pq_encode_cache(k, cb, np.zeros(B, np.int64), n)
    assert np.array_equal(enc, codes) or all(
        np.array_equal(_f64(k[b, u]), np.concatenate([_f64(cb[b, u, m])[enc[b, u, :, m]] for m in range(16)], 1))
        for b in range(B) for u in range(Hkv))
    kv_len = np.array([n, n - 37], dtype=np.int32)
    idx, cnt, tail, _ = PQ.pq_select(q, cb, enc, kv_len, sink, window, budget)
    for b in range(B):
        nb = int(kv_len[b])
        s0, t0, c = PQ.select_window(nb, sink, window, budget)
        assert cnt[b] == s0 + c and tail[b] == t0
        for u in range(Hkv):
            logit = _f64(k[b, u, :nb]) @ _f64(q[b, u * g:(u + 1) * g]).sum(0)
            cand = sorted(range(s0, t0), key=lambda j: (-logit[j], j))[:c]
            assert idx[b, u, :cnt[b]].tolist() == list(range(s0)) + sorted(cand)
            assert (idx[b, u, cnt[b]:] == -1).all()


def test_full_budget_draft_is_full_attention():
    rng = np.random.default_rng(6)
    B, Hkv, g, d, n = 2, 2, 2, 64, 90
    q, cb, codes, k = _exact_codebook_case(rng, B, Hkv, g, d, n)
    v = _grid_bits(rng, (B, Hkv, n, d))
    kv_len = np.array([n, 61], dtype=np.int32)
    idx, cnt, tail, _ = PQ.pq_select(q, cb, codes, kv_len, 4, 10, 200)
    scale = 0.125
    out, lse = SK.draft_attn_indexed(q, k, v, kv_len, idx, cnt, tail, scale)
    ref, rlse = OA.verify_attn_full(q[:, None], k, v, kv_len, scale)
    assert np.array_equal(out, ref[:, 0]) and np.array_equal(lse, rlse[:, 0])


def test_synth_codebook_selects_needles():
    """Peaky regime: boosted (needle) keys align with the group's queries, so the PQ scores
    of their codes dominate and every needle outside the sink/window is selected."""
    B, Hkv, g, d, n = 1, 2, 4, 128, 2000
    reg = S.Regime("peaky", sink=4, needle_period=97)
    k = S.k_to_bf16_bits(S.kv_cache_k(9, S.T_KCACHE, B, Hkv, d, 0, n, regime=reg))
    q = S.k_to_bf16_bits(S.q_rows_k(9, S.T_QDRAFT, B, 1, Hkv * g, Hkv, d, regime=reg))[:, 0]
    cb = S.pq_codebook_bits(k, S.pq_codebook_positions(9, B, Hkv, [n]))
    codes = PQ.pq_encode_cache(k, cb, np.zeros(B, np.int64), n)
    idx, cnt, tail, _ = PQ.pq_select(q, cb, codes, np.array([n], np.int32), 4, 64, 64)
    for u in range(Hkv):
        boosted = [j for j in range(4, int(tail[0]))
                   if S._is_boosted_pos(9, 0, u, np.array([j]), Hkv, reg)[0]]
        assert 0 < len(boosted) <= 64
        assert set(boosted) <= set(idx[0, u, :cnt[0]].tolist())


# ------------------------------------------------------------ off-grid: fp64 plain definition
# On arbitrary bf16 inputs (Gaussian keys, queries and centroids, not on the k/32 grid) fp32
# rounding does occur.  These pins bound the oracle's fixed-point pipeline (P1-P5, readings
# Z26 / Z28) against the PLAIN fp64 product-quantisation definition: nearest centroid by the
# exact squared distance, the PQ inner product sum_hh q_hh . khat_j in fp64, exact top-k of it.
# A deviation is allowed only where fp32 rounding can decide it: a near-tie within an error
# bound derived from the arithmetic (n-term fp32 sums: |err| <= n 2^-24 sum |terms|).
U = 2.0 ** -24


def _offgrid_bits(rng, shape, sigma=1.0):
    x = (rng.standard_normal(shape) * sigma).astype(np.float32)
    b = x.view(np.uint32)
    return ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)     # round to nearest bf16


def test_offgrid_encode_is_fp64_nearest_centroid_up_to_rounding_ties():
    rng = np.random.default_rng(21)
    for d in (64, 128):
        s = d // 16
        k = _offgrid_bits(rng, (2000, d))
        cb = _offgrid_bits(rng, (16, 256, s))
        codes = PQ.pq_encode(k, cb)
        x, C = _f64(k), _f64(cb)
        ndiff = 0
        for m in range(16):
            diff = x[:, None, m * s:(m + 1) * s] - C[m][None]          # [n, 256, s], exact in fp64
            dist = (diff ** 2).sum(-1)
            best = np.argmin(dist, axis=1)
            # fp32 left-to-right sum of s squares: |err| <= (s + 2) 2^-24 * dist (sub, mul, adds)
            bound = (s + 2) * U * dist
            rows = np.nonzero(codes[:, m] != best)[0]
            ndiff += len(rows)
            for j in rows:
                c32, c64 = int(codes[j, m]), int(best[j])
                assert dist[j, c32] - dist[j, c64] <= bound[j, c32] + bound[j, c64], (d, m, j)
        assert ndiff <= 2000 * 16 * 1e-3      # near-ties are rare


def test_offgrid_scores_are_the_pq_inner_product_within_the_rounding_bound():
    rng = np.random.default_rng(22)
    for d, g in ((128, 4), (128, 7), (64, 1)):
        s = d // 16
        q = _offgrid_bits(rng, (g, d))
        cb = _offgrid_bits(rng, (16, 256, s))
        codes = rng.integers(0, 256, size=(3000, 16)).astype(np.uint8)
        lut = PQ.pq_lut(q, cb)
        e = PQ.lut_exponent(lut)
        sc = PQ.pq_scores(PQ.pq_lut_fixed(lut), codes).astype(np.float64) * 2.0 ** -e
        Q, C = _f64(q), _f64(cb)
        khat = np.concatenate([C[m][codes[:, m]] for m in range(16)], axis=1)      # [n, d]
        exact = khat @ Q.sum(0)                                                     # fp64 PQ score
        # per table entry: g*s products and sums in fp32 -> <= 2 g s 2^-24 sum |q c|; then rint
        # to the 2^-e grid: <= 2^-e / 2 per entry; 16 entries per score
        absterm = np.stack([np.abs(C[m]) @ np.abs(Q[:, m * s:(m + 1) * s]).sum(0) for m in range(16)])  # [16, 256]
        ent_bound = 2 * g * s * U * absterm + 0.5 * 2.0 ** -e
        bound = sum(ent_bound[m][codes[:, m]] for m in range(16))
        err = np.abs(sc - exact)
        assert np.all(err <= bound), float(np.max(err / bound))
        assert np.max(err) > 0          # off-grid: rounding really happens (the bound is exercised)


def test_offgrid_selection_is_exact_pq_topk_up_to_near_ties():
    """P5 on the oracle's fixed-point scores vs exact top-k of the fp64 PQ scores: identical sets
    except positions whose fp64 score ties the k-th largest within twice the score bound."""
    rng = np.random.default_rng(23)
    B, Hkv, g, d, n = 2, 2, 4, 128, 1500
    s = d // 16
    sink, window, budget = 4, 64, 200
    k = _offgrid_bits(rng, (B, Hkv, n, d))
    q = _offgrid_bits(rng, (B, Hkv * g, d))
    cb = _offgrid_bits(rng, (B, Hkv, 16, 256, s))
    codes = PQ.pq_encode_cache(k, cb, np.zeros(B, np.int64), n)
    kv_len = np.array([n, n - 333], dtype=np.int32)
    idx, cnt, tail, _ = PQ.pq_select(q, cb, codes, kv_len, sink, window, budget)
    ndiff = 0
    for b in range(B):
        nb = int(kv_len[b])
        s0, t0, c = PQ.select_window(nb, sink, window, budget)
        for u in range(Hkv):
            Q, C = _f64(q[b, u * g:(u + 1) * g]), _f64(cb[b, u])
            khat = np.concatenate([C[m][codes[b, u, :nb, m]] for m in range(16)], axis=1)
            exact = khat @ Q.sum(0)
            lut = PQ.pq_lut(q[b, u * g:(u + 1) * g], cb[b, u])
            e = PQ.lut_exponent(lut)
            absterm = np.stack([np.abs(C[m]) @ np.abs(Q[:, m * s:(m + 1) * s]).sum(0) for m in range(16)])
            ent = 2 * g * s * U * absterm + 0.5 * 2.0 ** -e
            bound = sum(ent[m][codes[b, u, :nb, m]] for m in range(16))
            cand = np.arange(s0, t0)
            ref = set(sorted(cand, key=lambda j: (-exact[j], j))[:c])
            got = idx[b, u, s0:s0 + c].tolist()
            assert idx[b, u, :s0].tolist() == list(range(s0))
            thr = np.sort(exact[s0:t0])[::-1][c - 1]
            for x in ref ^ set(got):
                ndiff += 1
                assert abs(exact[x] - thr) <= 2 * bound.max(), (b, u, x)
    assert ndiff <= 4
