"""SnapKV static KV selection and index-list draft attention (TEST INFRASTRUCTURE ONLY;
see oracle/__init__.py).  SURVEY §8(f) row f2.

The paper's best drafter is self-speculation over a SnapKV-compressed KV (P:514, P:538
headline 2.51x; P:1141 footnote: "SnapKV ... utilizing average pooling with a kernel size
of 5 and an observation window size of 32").  SnapKV (Li et al. 2024) selects, once at
prefill, the prefix positions the last `w` prompt queries attend to most:

  S1  for each query head h of the KV head's GQA group and each window query i (prompt
      position L-w+i):  a[h,i,j] = softmax_j(scale q[h,i] . k[j]),  j in [0, L-w+i]
      (causal softmax over the whole prompt, natural exp);
  S2  vote[j] = sum_{h,i} a[h,i,j]            for prefix positions j in [0, L-w);
  S3  pooled[j] = (1/5) sum_{t=-2..2} vote[j+t]   (zero padding outside [0, L-w));
  S4  keep the top (budget - w) prefix positions by pooled (ties -> lower position),
      reported in ascending order; the window [L-w, L) is always kept.

Readings (Z17-Z19): S2 sums over the g query heads of a GQA group (sum and
mean select the same set); ties in S4 go to the lower position; after prefill the draft
attends to the selected positions plus every position from L-w on (the window and all
tokens generated since), i.e. J = idx U [tail_start, n) with tail_start = L - w.

The draft attention over J is the O2 core on the gathered rows (as in attention.py O3).
"""
from __future__ import annotations

import numpy as np

from .attention import bf16_to_f64, softmax_attention


def snapkv_votes(q_obs_bits, k_bits_unit, L: int, w: int, scale: float) -> np.ndarray:
    """S1-S2 for one (b, kv head): q_obs_bits [g, w, d] (the group's window queries),
    k_bits_unit [>= L, d] -> vote [L - w] (fp64)."""
    q = bf16_to_f64(q_obs_bits)
    k = bf16_to_f64(k_bits_unit[:L])
    g = q.shape[0]
    vote = np.zeros(L - w)
    for h in range(g):
        for i in range(w):
            last = L - w + i                       # causal: keys [0, L-w+i]
            s = scale * (k[: last + 1] @ q[h, i])
            a = np.exp(s - s.max())
            a /= a.sum()
            vote += a[: L - w]
    return vote


def avg_pool5(vote: np.ndarray) -> np.ndarray:
    """S3: kernel 5, stride 1, zero padding 2, divisor 5."""
    padded = np.concatenate([np.zeros(2), vote, np.zeros(2)])
    return (padded[0:-4] + padded[1:-3] + padded[2:-2] + padded[3:-1] + padded[4:]) / 5.0


def topk_positions(pooled: np.ndarray, k: int) -> np.ndarray:
    """S4: the k largest (ties -> lower position), ascending."""
    if k >= len(pooled):
        return np.arange(len(pooled), dtype=np.int32)
    order = np.lexsort((np.arange(len(pooled)), -pooled))   # by -score, then position
    return np.sort(order[:k]).astype(np.int32)


def snapkv_select(q_obs_bits, k_cache_bits, prefill_len, w: int, budget: int, scale: float, budgets=None):
    """Batched S1-S4.  q_obs_bits [B, w, Hq, d] (queries of the last w prompt positions),
    k_cache_bits [B, Hkv, cap, d], prefill_len [B] ->
    (idx [B, Hkv, budget - w] int32 (ascending; -1 padded), count [B] int32, pooled list).
    budgets: optional per-sequence budgets [B] ("different sequences in the same batch can
    leverage different draft KV cache sizes"), each clamped to [w, budget]."""
    B, _, Hq, d = q_obs_bits.shape
    Hkv = k_cache_bits.shape[1]
    g = Hq // Hkv
    kmax = budget - w
    idx = np.full((B, Hkv, kmax), -1, dtype=np.int32)
    count = np.zeros(B, dtype=np.int32)
    pooled_all = []
    for b in range(B):
        L = int(prefill_len[b])
        kb = kmax if budgets is None else min(max(int(budgets[b]), w), budget) - w
        cnt = min(kb, L - w)
        count[b] = cnt
        row = []
        for h in range(Hkv):
            qg = np.transpose(q_obs_bits[b, :, h * g:(h + 1) * g], (1, 0, 2))    # [g, w, d]
            pooled = avg_pool5(snapkv_votes(qg, k_cache_bits[b, h], L, w, scale))
            idx[b, h, :cnt] = topk_positions(pooled, cnt)
            row.append(pooled)
        pooled_all.append(row)
    return idx, count, pooled_all


def draft_index_set_indexed(idx_row, count: int, tail_start: int, n: int) -> np.ndarray:
    """J = idx[:count] U [tail_start, n), ascending (idx < tail_start by construction)."""
    return np.concatenate([np.asarray(idx_row[:count], dtype=np.int64), np.arange(tail_start, n)])


def draft_attn_indexed(q_bits, k_cache_bits, v_cache_bits, kv_len, idx, count, tail_start, scale):
    """Draft attention over the SnapKV set.  q_bits [B, Hq, d]; idx [B, Hkv, K]; count [B];
    tail_start [B] -> out [B, Hq, d] fp64, lse [B, Hq] fp64."""
    q = bf16_to_f64(q_bits)
    B, Hq, d = q.shape
    Hkv = k_cache_bits.shape[1]
    g = Hq // Hkv
    out = np.zeros((B, Hq, d))
    lse = np.zeros((B, Hq))
    for b in range(B):
        for kvh in range(Hkv):
            J = draft_index_set_indexed(idx[b, kvh], int(count[b]), int(tail_start[b]), int(kv_len[b]))
            K = bf16_to_f64(k_cache_bits[b, kvh, J])
            V = bf16_to_f64(v_cache_bits[b, kvh, J])
            for h in range(kvh * g, (kvh + 1) * g):
                out[b, h], lse[b, h] = softmax_attention(q[b, h], K, V, scale)
    return out, lse
