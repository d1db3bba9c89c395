"""Oracle attention for the verify / draft calls (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Definitions (fp64, two-pass softmax, no online rescaling, no splits):

  O1  bf16 inputs are decoded exactly: bits << 16 -> fp32 -> fp64.
  O2  verify_attn_full ("the target model to verify gamma tokens", P:281
      "verification and decoding share the same KV budget"): for sequence b,
      query token t in [0, T) and query head h, with kv head kvh = floor(h / g)
      (g = Hq / Hkv, GQA) and n = kv_len[b] (which counts the T new tokens):
          J   = [0, n - T + t]                       (causal among the T new rows)
          s_j = scale * sum_c q[b,t,h,c] * k[b,kvh,j,c]
          o   = sum_j softmax(s)_j * v[b,kvh,j,:],   lse = log sum_j exp(s_j)  (natural log)
  O3  draft_attn_sparse (StreamingLLM sink + window drafting, P:453, P:460, P:720,
      Eq.3): one query token per sequence attends to
          J = {j < min(sink, n)}  U  {max(sink, n - window) <= j < n}
      (ascending, no index twice), gathered, then the O2 core with T = 1.
  kv_append: cache rows [start_b, start_b + T) of every kv head take the new rows.
  O6  merge of partials over a partition J = J1 u J2 (used only by the pins).
"""
from __future__ import annotations

import numpy as np


def bf16_to_f64(bits) -> np.ndarray:
    """O1: exact decode of bf16 bit patterns (uint16) to float64."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32).astype(np.float64)


def softmax_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float, vT=None):
    """The O2 core for one query row over an explicit key set.

    q [d], k [n, d], v [n, d] (fp64) -> (o [d], lse).  Two passes: the maximum, then the
    exp-sum and the weighted sum.  Every sum is taken sequentially in ascending index order
    (np.cumsum's last element: a left-to-right recurrence, not BLAS's blocked order): the dot
    products over c (each product of two bf16 values is exact in fp64), Z over j, o over j.
    vT: optionally v transposed ([d, n], any strides; only a faster memory layout, same sums)."""
    s = scale * np.cumsum(k * q[None, :], axis=1)[:, -1]   # s_j = scale * sum_c q_c k_jc, c ascending
    m = s.max()
    w = np.exp(s - m)
    z = np.cumsum(w)[-1]                                   # Z = sum_j w_j, j ascending
    vT = v.T if vT is None else vT
    o = np.cumsum(vT * w[None, :], axis=1)[:, -1] / z      # o_c = sum_j w_j v_jc / Z, j ascending
    return o, m + np.log(z)


def verify_attn_full(q_bits, k_cache_bits, v_cache_bits, kv_len, scale):
    """O2.  q_bits [B, T, Hq, d] uint16 (bf16), caches [B, Hkv, cap, d] uint16,
    kv_len [B] (includes the T new tokens) -> out [B, T, Hq, d] fp64, lse [B, T, Hq] fp64."""
    q = bf16_to_f64(q_bits)
    B, T, Hq, d = q.shape
    Hkv = k_cache_bits.shape[1]
    g = Hq // Hkv
    out = np.zeros((B, T, Hq, d))
    lse = np.zeros((B, T, Hq))
    for b in range(B):
        n = int(kv_len[b])
        for kvh in range(Hkv):
            K = bf16_to_f64(k_cache_bits[b, kvh, :n])
            V = bf16_to_f64(v_cache_bits[b, kvh, :n])
            VT = np.ascontiguousarray(V.T)
            for t in range(T):
                last = n - T + t                  # row t sees keys [0, n - T + t]
                for h in range(kvh * g, (kvh + 1) * g):
                    out[b, t, h], lse[b, t, h] = softmax_attention(q[b, t, h], K[: last + 1], V[: last + 1], scale,
                                                                   VT[:, : last + 1])
    return out, lse


def draft_index_set(n: int, sink: int, window: int) -> np.ndarray:
    """O3 index set J = {j < min(sink, n)} U {max(sink, n - window) <= j < n}, ascending."""
    head = np.arange(min(sink, n))
    tail = np.arange(max(sink, n - window), n)
    return np.concatenate([head, tail]).astype(np.int64)


def draft_attn_sparse(q_bits, k_cache_bits, v_cache_bits, kv_len, sink, window, scale):
    """O3.  q_bits [B, Hq, d] uint16 -> out [B, Hq, d] fp64, lse [B, Hq] fp64.  `window` may be a
    per-sequence array [B] (heterogeneous batches: "different sequences in the same batch can
    leverage different draft KV cache sizes")."""
    q = bf16_to_f64(q_bits)
    B, Hq, d = q.shape
    Hkv = k_cache_bits.shape[1]
    g = Hq // Hkv
    out = np.zeros((B, Hq, d))
    lse = np.zeros((B, Hq))
    for b in range(B):
        J = draft_index_set(int(kv_len[b]), sink, int(window[b]) if np.ndim(window) else window)
        for kvh in range(Hkv):
            K = bf16_to_f64(k_cache_bits[b, kvh, J])
            V = bf16_to_f64(v_cache_bits[b, kvh, J])
            for h in range(kvh * g, (kvh + 1) * g):
                out[b, h], lse[b, h] = softmax_attention(q[b, h], K, V, scale)
    return out, lse


def kv_append(k_cache_bits, v_cache_bits, k_new_bits, v_new_bits, start):
    """Cache update: rows [start_b, start_b + T) of every kv head <- the new rows.
    k_new / v_new are [B, T, Hkv, d] (as a QKV projection emits them).  In place."""
    B, T, Hkv, d = k_new_bits.shape
    for b in range(B):
        s = int(start[b])
        k_cache_bits[b, :, s:s + T] = np.transpose(k_new_bits[b], (1, 0, 2))
        v_cache_bits[b, :, s:s + T] = np.transpose(v_new_bits[b], (1, 0, 2))


def merge_partials(o_parts, lse_parts):
    """O6: combine attention results over disjoint key sets.
    o = sum_s e^{lse_s} o_s / sum_s e^{lse_s},  lse = log sum_s e^{lse_s}."""
    lse_parts = np.asarray(lse_parts, dtype=np.float64)
    m = lse_parts.max()
    w = np.exp(lse_parts - m)
    o = sum(wi * np.asarray(oi) for wi, oi in zip(w, o_parts)) / w.sum()
    return o, m + np.log(w.sum())
