"""Tree-based speculation: tree-masked verification attention, tree acceptance and KV
compaction (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).  SURVEY §8(f) row f3.

The paper lists tree-based speculation as compatible with its analysis without
details; the readings below (Z21-Z24) follow the standard token-tree
verification of SpecInfer / Sequoia with the integer decisions of oracle/accept.py.

Tree: T nodes per sequence, node 0 is the pending token (root), parent[t] < t for t >= 1.
The T nodes' K/V rows occupy cache positions [n - T, n) in node order.

  verify_attn_tree:  row (t, h) attends to the prefix [0, n - T) and to the new keys
      n - T + j for every j with bit j of mask[b][t] set (for a tree: the ancestors-or-self
      of t, mask[t] = mask[parent[t]] | 1 << t); otherwise as O2 (attention.py).

  spec_accept_tree (SAMPLE): walk from the root.  At node `cur` the children are tried in
      index order; the first child is tested exactly like the chain rule
      (m q(x) < p(x) 2^29, m = rnd >> 3); after a rejection the target is replaced by the
      residual on the 2^-40 grid, R_i = max(0, P_i - Q_i) with P = floor(p 2^40),
      Q = floor(q 2^40) (R = P if that sums to 0), and each later sibling x is accepted iff
      m Q_x S < R_x 2^69 (S = sum R; exact integers), a rejection updating
      R_i <- max(0, floor(R_i 2^40 / S) - Q_i) (kept if that sums to 0; with S = 0, only
      possible for an all-zero p row, the sibling is rejected and R kept).  When a child is
      accepted the walk moves to it; when none is (or there are none) the new token is
      drawn from R (or from P at a node whose children were not tried) with the 64-bit
      uniform (rnd[T-1] << 32 | rnd[T]) exactly as in accept.py.  Test words are consumed
      in order rnd[0], rnd[1], ...  For a chain this is exactly oracle/accept.py.
  spec_accept_tree (GREEDY): a = lowest-index argmax p[cur]; move to the lowest-index child
      whose token is a, else emit a.
  kv_compact: rows of the accepted path nodes move to consecutive slots after the root.
"""
from __future__ import annotations

import numpy as np

from .accept import TWO29, argmax_lowest, draw_from_weights, grid40
from .attention import bf16_to_f64, softmax_attention


def chain_mask(T: int) -> np.ndarray:
    return np.array([(1 << (t + 1)) - 1 for t in range(T)], dtype=np.uint32)


def tree_mask_from_parents(parent) -> np.ndarray:
    T = len(parent)
    mask = np.zeros(T, dtype=np.uint32)
    for t in range(T):
        mask[t] = (1 << t) | (0 if t == 0 else int(mask[parent[t]]))
    return mask


def verify_attn_tree(q_bits, k_cache_bits, v_cache_bits, kv_len, tree_mask, scale):
    """q_bits [B, T, Hq, d], tree_mask [B, T] uint32 -> out [B, T, Hq, d], lse [B, T, Hq] (fp64)."""
    q = bf16_to_f64(q_bits)
    B, T, Hq, d = q.shape
    Hkv = k_cache_bits.shape[1]
    g = Hq // Hkv
    out = np.zeros((B, T, Hq, d))
    lse = np.zeros((B, T, Hq))
    for b in range(B):
        n = int(kv_len[b])
        for t in range(T):
            J = list(range(n - T)) + [n - T + j for j in range(T) if (int(tree_mask[b, t]) >> j) & 1]
            for kvh in range(Hkv):
                K = bf16_to_f64(k_cache_bits[b, kvh, J])
                V = bf16_to_f64(v_cache_bits[b, kvh, J])
                for h in range(kvh * g, (kvh + 1) * g):
                    out[b, t, h], lse[b, t, h] = softmax_attention(q[b, t, h], K, V, scale)
    return out, lse


def _renorm40(R: np.ndarray) -> np.ndarray:
    """floor(R_i 2^40 / sum R) with exact integers."""
    S = int(R.sum(dtype=np.uint64))
    return np.array([(int(r) << 40) // S for r in R], dtype=np.uint64)


def _accept_sibling(m: int, Qx: int, S: int, Rx: int) -> bool:
    return m * Qx * S < Rx * (1 << 69)


def accept_tree_one(p, q, tokens, parent, rnd, mode="sample"):
    """One sequence.  p, q [T, V] fp32; tokens, parent [T]; rnd [T + 1] uint32.
    Returns (path node indices excluding the root, new token)."""
    T = len(tokens)
    children = [[c for c in range(1, T) if parent[c] == t] for t in range(T)]
    cur, path, k = 0, [], 0
    if mode == "greedy":
        while True:
            a = argmax_lowest(p[cur])
            nxt = [c for c in children[cur] if int(tokens[c]) == a]
            if not nxt:
                return path, a
            cur = nxt[0]
            path.append(cur)
    u64 = (int(rnd[T - 1]) << 32) | int(rnd[T])
    while True:
        kids = children[cur]
        if not kids:                                    # leaf: bonus draw from p
            P = grid40(p[cur])
            tok = draw_from_weights(P, u64) if int(P.sum(dtype=np.uint64)) else argmax_lowest(p[cur])
            return path, tok
        P = grid40(p[cur])
        Q = grid40(q[cur])
        R = None
        accepted = None
        for i, c in enumerate(kids):
            x = int(tokens[c])
            m = int(rnd[k]) >> 3
            k += 1
            if i == 0:
                ok = float(m) * float(q[cur][x]) < float(p[cur][x]) * TWO29
            else:
                S = int(R.sum(dtype=np.uint64))
                ok = S > 0 and _accept_sibling(m, int(Q[x]), S, int(R[x]))
            if ok:
                accepted = c
                break
            if i == 0:
                R = np.where(P > Q, P - Q, np.uint64(0))
                if int(R.sum(dtype=np.uint64)) == 0:
                    R = P.copy()
            elif int(R.sum(dtype=np.uint64)) == 0:      # degenerate (all-zero p row): keep R
                pass
            else:
                Rn = _renorm40(R)
                R2 = np.where(Rn > Q, Rn - Q, np.uint64(0))
                R = R2 if int(R2.sum(dtype=np.uint64)) else R
        if accepted is not None:
            cur = accepted
            path.append(cur)
            continue
        if int(R.sum(dtype=np.uint64)) == 0:
            return path, argmax_lowest(p[cur])
        return path, draw_from_weights(R, u64)


def spec_accept_tree(p, q, tokens, parent, rnd, mode="sample"):
    """Batched.  p, q [B, T, V]; tokens, parent [B, T] int32; rnd [B, T + 1] uint32 ->
    out_tokens [B, T] (accepted tokens then the new one, -1 padded), num_accepted [B],
    accepted_nodes [B, T] (path node indices, -1 padded)."""
    B, T = tokens.shape
    out = np.full((B, T), -1, np.int32)
    nodes = np.full((B, T), -1, np.int32)
    nacc = np.zeros(B, np.int32)
    for b in range(B):
        path, tok = accept_tree_one(p[b], q[b], tokens[b], parent[b], None if rnd is None else rnd[b], mode)
        for i, c in enumerate(path):
            out[b, i] = tokens[b, c]
            nodes[b, i] = c
        out[b, len(path)] = tok
        nacc[b] = len(path)
    return out, nacc, nodes


def kv_compact(k_cache_bits, v_cache_bits, base, nodes, count):
    """For each b: rows base[b] + nodes[b][i] -> base[b] + 1 + i for i < count[b] (in place,
    every kv head).  base[b] is the root's cache position (n - T)."""
    B = len(base)
    for b in range(B):
        for i in range(int(count[b])):
            src = int(base[b]) + int(nodes[b, i])
            dst = int(base[b]) + 1 + i
            k_cache_bits[b, :, dst] = k_cache_bits[b, :, src]
            v_cache_bits[b, :, dst] = v_cache_bits[b, :, src]
