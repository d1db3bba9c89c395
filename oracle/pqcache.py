"""PQCache-style dynamic KV selection for self-speculative drafting (TEST INFRASTRUCTURE
ONLY; see oracle/__init__.py).  SURVEY §8(f) row f4.

The paper compares static KV selection (StreamingLLM, SnapKV) with dynamic selection that
"dynamically searches the KV cache for each input query, attempting to find the top k
nearest neighbors", represented by PQCache: "product quantization with 16
sub-vectors and 8-bit quantization per key vector" (P:1141 footnote).  Its cost is the
T_select term of Eq.3: T_D,select = T_D(B, K) + T_select(B, S, K), "a
batch-size-dependent KV selection cost".  The paper gives no algorithmic detail
beyond the footnote; the readings below (Z25-Z29) are those of product
quantisation with asymmetric distance computation (the standard PQ search):

  P1  encode:  key k (head_dim d) is cut into M = 16 sub-vectors of s = d/16 elements; the
      code of sub-vector m is the index of the nearest of the 256 centroids C[m][0..255]
      (8-bit code), squared Euclidean distance, ties -> lowest index.  The distance is
      taken in fp32 exactly as dist = sum_{i<s} (x_i - c_i)^2 evaluated left to right with
      every subtraction, product and sum rounded to fp32 (no fused multiply-add), because
      an integer (the code) is decided by it (Z26).
  P2  table:   per (sequence, KV head), the group's g query heads fold into one lookup
      table  lut[m][c] = sum_{hh<g} sum_{i<s} q[hh][m*s+i] * C[m][c][i]  (fp32, hh outer,
      i inner, left to right, no FMA), i.e. the inner product of the query with each
      centroid (asymmetric distance: the query is not quantised).  Summing over the group
      scores a key by the sum of the group's logits (Z27, as SnapKV's votes, Z17).
  P3  fixed point: e = 26 - E where max|lut| = f * 2^E, f in [0.5, 1) (e = 0 if the table
      is all zero); lutq = rint(lut * 2^e) (round half to even) as int32 — the scaling is
      exact (a power of two), |lutq| < 2^26, so the 16-term score below is an exact
      integer whatever the summation order (Z28).
  P4  score:   score[j] = sum_m lutq[m][code[j][m]]  (= 2^e * the PQ approximation of
      sum_hh q_hh . k_j, up to the rounding in P3).
  P5  select:  with n = kv_len, s0 = min(sink, n), tail_start = max(s0, n - window): the
      c = min(budget, tail_start - s0) positions of [s0, tail_start) with the largest
      score (ties -> lower position), ascending, after the sink rows [0, s0):
      idx = [0 .. s0) ++ selected, idx_count = s0 + c.  The draft attends to
      idx U [tail_start, n) (the window stays exact, as in PQCache's local tokens) (Z29).

The draft attention over that set is oracle.snapkv.draft_attn_indexed (the O2 core).
Codebook training (k-means at prefill) is outside the decode hot path: the codebook is an
input (bf16 [B][Hkv][16][256][s]).
"""
from __future__ import annotations

import numpy as np

M_SUB = 16       # sub-vectors per key
N_CENT = 256     # 8-bit codes

F32 = np.float32


def _bf16_to_f32(bits) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(F32)


def pq_encode(k_bits_rows, codebook_bits_unit) -> np.ndarray:
    """P1 for the rows of one (b, kv head): k_bits_rows [n, d] bf16 bits, codebook
    [16, 256, s] bf16 bits -> codes [n, 16] uint8."""
    x = _bf16_to_f32(k_bits_rows)                       # [n, d]
    C = _bf16_to_f32(codebook_bits_unit)                # [16, 256, s]
    n, d = x.shape
    s = d // M_SUB
    codes = np.zeros((n, M_SUB), dtype=np.uint8)
    for m in range(M_SUB):
        xs = x[:, m * s:(m + 1) * s]                     # [n, s]
        acc = np.zeros((n, N_CENT), dtype=F32)
        for i in range(s):                               # left to right, fp32, no FMA
            t = (xs[:, i:i + 1] - C[m][None, :, i]).astype(F32)
            acc = (acc + (t * t).astype(F32)).astype(F32)
        codes[:, m] = np.argmin(acc, axis=1)             # first minimum = lowest index
    return codes


def pq_encode_cache(k_cache_bits, codebook_bits, start, count) -> np.ndarray:
    """P1 over rows [start_b, start_b + count) of every (b, kv head) -> codes
    [B, Hkv, count, 16] uint8."""
    B, Hkv = k_cache_bits.shape[:2]
    out = np.zeros((B, Hkv, count, M_SUB), dtype=np.uint8)
    for b in range(B):
        for u in range(Hkv):
            s0 = int(start[b])
            out[b, u] = pq_encode(k_cache_bits[b, u, s0:s0 + count], codebook_bits[b, u])
    return out


def pq_lut(q_group_bits, codebook_bits_unit) -> np.ndarray:
    """P2: q_group_bits [g, d] bf16 bits (the KV head's query heads), codebook [16, 256, s]
    -> lut [16, 256] fp32."""
    q = _bf16_to_f32(q_group_bits)
    C = _bf16_to_f32(codebook_bits_unit)
    g, d = q.shape
    s = d // M_SUB
    lut = np.zeros((M_SUB, N_CENT), dtype=F32)
    for m in range(M_SUB):
        acc = np.zeros(N_CENT, dtype=F32)
        for hh in range(g):
            for i in range(s):
                acc = (acc + (q[hh, m * s + i] * C[m, :, i]).astype(F32)).astype(F32)
        lut[m] = acc
    return lut


def lut_exponent(lut: np.ndarray) -> int:
    """P3's scale exponent e."""
    mx = float(np.max(np.abs(lut)))
    if mx == 0.0:
        return 0
    _, E = np.frexp(mx)
    return 26 - int(E)


def pq_lut_fixed(lut: np.ndarray) -> np.ndarray:
    """P3: int32 table rint(lut * 2^e) (exact power-of-two scaling, round half to even)."""
    e = lut_exponent(lut)
    return np.rint(np.ldexp(lut.astype(F32), e).astype(F32)).astype(np.int64).astype(np.int32)


def pq_scores(lutq: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """P4: codes [n, 16] -> int64 scores [n] (exact integer sums)."""
    return sum(lutq[m].astype(np.int64)[codes[:, m].astype(np.int64)] for m in range(M_SUB))


def select_topk(scores: np.ndarray, lo: int, hi: int, c: int) -> np.ndarray:
    """The c largest scores among positions [lo, hi) (ties -> lower position), ascending."""
    pos = np.arange(lo, hi)
    sc = scores[lo:hi]
    order = np.lexsort((pos, -sc))                       # by -score, then position
    return np.sort(pos[order[:c]]).astype(np.int32)


def select_window(n: int, sink: int, window: int, budget: int):
    """P5's ranges: (s0, tail_start, c)."""
    s0 = min(sink, n)
    tail = max(s0, n - window)
    return s0, tail, min(budget, tail - s0)


def pq_select(q_bits, codebook_bits, codes, kv_len, sink: int, window: int, budget: int):
    """P2-P5, batched.  q_bits [B, Hq, d] (the draft query), codebook [B, Hkv, 16, 256, s],
    codes [B, Hkv, >= n, 16] ->
    (idx [B, Hkv, sink + budget] int32 (-1 padded), idx_count [B], tail_start [B], scores list)."""
    B, Hq, d = q_bits.shape
    Hkv = codebook_bits.shape[1]
    g = Hq // Hkv
    K = sink + budget
    idx = np.full((B, Hkv, K), -1, dtype=np.int32)
    cnt = np.zeros(B, dtype=np.int32)
    tail_start = np.zeros(B, dtype=np.int32)
    all_scores = []
    for b in range(B):
        n = int(kv_len[b])
        s0, tail, c = select_window(n, sink, window, budget)
        cnt[b] = s0 + c
        tail_start[b] = tail
        row = []
        for u in range(Hkv):
            lutq = pq_lut_fixed(pq_lut(q_bits[b, u * g:(u + 1) * g], codebook_bits[b, u]))
            sc = pq_scores(lutq, codes[b, u, :n])
            row.append(sc)
            idx[b, u, :s0] = np.arange(s0)
            idx[b, u, s0:s0 + c] = select_topk(sc, s0, tail, c)
        all_scores.append(row)
    return idx, cnt, tail_start, all_scores
