"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no attention, no softmax of the
method, no acceptance rule).  It only produces inputs:

* bf16 Q / K / V values on the exact grid x = k/32 (k integer, |k| <= 256), so every
  value is exactly representable in bf16 and its fp64 decode is exact
  (SURVEY.md §8(d) "Synthetic inputs");
* per-sequence committed lengths (uniform or ragged, "misalignment of the
  sequence lengths");
* target / draft probability rows p, q (Zipf(1.1) logits, q = noisy p) and draft
  tokens d ~ q, which are what the (out-of-scope) model + LM head upstream of
  `spec_accept` would hand it;
* uniform words for `spec_accept` come from Philox, which both sides implement
  independently (oracle/philox.py and csrc/philox.cuh); see DESIGN.md.

Every value is a pure function of (seed, tensor id, coordinates) through a
splitmix64-style counter hash, so any slice can be regenerated anywhere without
generating the rest.  `synth/csrc/synth_gen.cu` implements the identical hash on
the GPU (bit-exact; tests/test_synth.py checks it) so that full-size (multi-GB)
caches can be produced in HBM and any sampled sequence regenerated on the host
for the oracle.
"""
from __future__ import annotations

import numpy as np

U64 = np.uint64
MASK64 = (1 << 64) - 1

# tensor ids (the counter-hash domain separator)
T_KCACHE = 1
T_VCACHE = 2
T_QVERIFY = 3
T_QDRAFT = 4
T_KNEW = 5
T_VNEW = 6
T_DIR = 7
T_NEEDLE = 8
T_LEN = 9
T_LOGIT = 10
T_NOISE = 11
T_DRAFTU = 12

POSMAX = 1 << 24          # position stride in the K/V hash index (independent of capacity)


def _mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = x.astype(U64, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> U64(30)
        x *= U64(0xBF58476D1CE4E5B9)
        x ^= x >> U64(27)
        x *= U64(0x94D049BB133111EB)
        x ^= x >> U64(31)
    return x


def _key(seed: int, tensor: int) -> np.uint64:
    k = ((seed * 0x9E3779B97F4A7C15) + (tensor << 56) + tensor * 0xD1B54A32D192ED03) & MASK64
    return _mix64(np.array([k], dtype=U64))[0]


def hash_u64(seed: int, tensor: int, idx) -> np.ndarray:
    """h = mix64(key(seed, tensor) + idx) for a uint64 index array."""
    idx = np.asarray(idx, dtype=U64)
    with np.errstate(over="ignore"):
        return _mix64(idx + _key(seed, tensor))


def grid_k(seed: int, tensor: int, idx) -> np.ndarray:
    """Integer k in [-32, 31]: the value is k/32 (exact in bf16)."""
    return (hash_u64(seed, tensor, idx) >> U64(58)).astype(np.int32) - 32


def k_to_bf16_bits(k: np.ndarray) -> np.ndarray:
    """bf16 bit pattern of k/32 for integer |k| <= 256 (exact: <= 8 significant bits)."""
    f = (np.asarray(k, dtype=np.float32) / np.float32(32.0)).astype(np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


# ----------------------------------------------------------------------------------------
# score regimes
# ----------------------------------------------------------------------------------------
class Regime:
    """'flat': plain hash values.  'peaky': a per-(b, kv head) +-1 direction r is added
    (x32) to keys at positions < sink and at hashed needle positions, and a_q * r is
    added to every query row of that group, so the sinks take a large share of the
    softmax mass (attention sinks, P:453 StreamingLLM)."""

    def __init__(self, kind: str = "flat", sink: int = 4, a_q: int = 24, a_k: int = 32,
                 needle_period: int = 4099):
        assert kind in ("flat", "peaky")
        self.kind, self.sink, self.a_q, self.a_k, self.needle_period = kind, sink, a_q, a_k, needle_period

    def code(self) -> int:
        return 0 if self.kind == "flat" else 1


FLAT = Regime("flat")


def _dir_sign(seed, b, kvh, c, Hkv, d):
    idx = (np.asarray(b, dtype=U64) * U64(Hkv) + np.asarray(kvh, dtype=U64)) * U64(d) + np.asarray(c, dtype=U64)
    return np.where((hash_u64(seed, T_DIR, idx) >> U64(63)) == U64(1), 1, -1).astype(np.int32)


def _is_boosted_pos(seed, b, kvh, pos, Hkv, reg: Regime):
    pos = np.asarray(pos, dtype=np.int64)
    idx = (np.asarray(b, dtype=U64) * U64(Hkv) + np.asarray(kvh, dtype=U64)) * U64(POSMAX) + pos.astype(U64)
    needle = (hash_u64(seed, T_NEEDLE, idx) % U64(reg.needle_period)) == U64(0)
    return (pos < reg.sink) | needle


def kv_cache_k(seed: int, tensor: int, B: int, Hkv: int, d: int, pos0: int, npos: int,
               b_sel=None, h_sel=None, regime: Regime = FLAT) -> np.ndarray:
    """Integer grid values k for cache rows pos0..pos0+npos-1 -> int32 [nb, nh, npos, d].

    b_sel / h_sel select a subset of sequences / KV heads (coordinates stay global)."""
    bs = np.arange(B) if b_sel is None else np.asarray(b_sel)
    hs = np.arange(Hkv) if h_sel is None else np.asarray(h_sel)
    b = bs[:, None, None, None].astype(U64)
    h = hs[None, :, None, None].astype(U64)
    p = (np.arange(npos, dtype=np.int64) + pos0)[None, None, :, None]
    c = np.arange(d, dtype=np.int64)[None, None, None, :]
    idx = ((b * U64(Hkv) + h) * U64(POSMAX) + p.astype(U64)) * U64(d) + c.astype(U64)
    k = grid_k(seed, tensor, idx)
    if regime.kind == "peaky" and tensor == T_KCACHE:
        boost = _is_boosted_pos(seed, b, h, p, Hkv, regime)
        k = k + np.where(boost, regime.a_k * _dir_sign(seed, b, h, c, Hkv, d), 0)
    return k.astype(np.int32)


def q_rows_k(seed: int, tensor: int, B: int, T: int, Hq: int, Hkv: int, d: int,
             b_sel=None, regime: Regime = FLAT) -> np.ndarray:
    """Integer grid values for queries [nb, T, Hq, d] (T=1 for draft queries)."""
    bs = np.arange(B) if b_sel is None else np.asarray(b_sel)
    b = bs[:, None, None, None].astype(U64)
    t = np.arange(T, dtype=np.int64)[None, :, None, None].astype(U64)
    h = np.arange(Hq, dtype=np.int64)[None, None, :, None].astype(U64)
    c = np.arange(d, dtype=np.int64)[None, None, None, :].astype(U64)
    idx = ((b * U64(T) + t) * U64(Hq) + h) * U64(d) + c
    k = grid_k(seed, tensor, idx)
    if regime.kind == "peaky":
        g = Hq // Hkv
        kvh = (np.arange(Hq) // g)[None, None, :, None]
        k = k + regime.a_q * _dir_sign(seed, b, kvh.astype(U64), c, Hkv, d)
    return k.astype(np.int32)


def new_kv_k(seed: int, tensor: int, B: int, T: int, Hkv: int, d: int) -> np.ndarray:
    """Integer grid values for freshly projected K/V rows [B, T, Hkv, d] (kv_append input)."""
    idx = np.arange(B * T * Hkv * d, dtype=np.int64).astype(U64)
    return grid_k(seed, tensor, idx).reshape(B, T, Hkv, d)


# ----------------------------------------------------------------------------------------
# off-grid values: arbitrary bf16 bit patterns (full 8-bit significand, 7 binades), |x| < 1
# ----------------------------------------------------------------------------------------
def offgrid_bits_from_hash(h: np.ndarray) -> np.ndarray:
    """bf16 bits from a uint64 hash: sign, biased exponent 120..126 (|x| in [2^-7, 1)), and a
    random 7-bit mantissa -- values OFF the k/32 grid (every bf16 in that range is reachable),
    so fp32 rounding in QK^T and the softmax really happens; |x| < 1 keeps the north_star
    tolerance derivation (bf16 P error <= 2^-9 max|v|) valid."""
    h = np.asarray(h, dtype=U64)
    sign = ((h >> U64(63)) & U64(1)).astype(np.uint16)
    ex = (((h >> U64(40)) & U64(0xFFFF)) % U64(7)).astype(np.uint16) + np.uint16(120)
    man = ((h >> U64(20)) & U64(0x7F)).astype(np.uint16)
    return (sign << np.uint16(15)) | (ex << np.uint16(7)) | man


def kv_cache_bits_offgrid(seed: int, tensor: int, B: int, Hkv: int, d: int, pos0: int, npos: int,
                          b_sel=None, h_sel=None) -> np.ndarray:
    """Off-grid cache rows pos0..pos0+npos-1 -> uint16 bf16 bits [nb, nh, npos, d] (the same
    hash index as kv_cache_k)."""
    bs = np.arange(B) if b_sel is None else np.asarray(b_sel)
    hs = np.arange(Hkv) if h_sel is None else np.asarray(h_sel)
    b = bs[:, None, None, None].astype(U64)
    h = hs[None, :, None, None].astype(U64)
    p = (np.arange(npos, dtype=np.int64) + pos0)[None, None, :, None]
    c = np.arange(d, dtype=np.int64)[None, None, None, :]
    idx = ((b * U64(Hkv) + h) * U64(POSMAX) + p.astype(U64)) * U64(d) + c.astype(U64)
    return offgrid_bits_from_hash(hash_u64(seed, tensor, idx))


def flat_bits_offgrid(seed: int, tensor: int, shape, b_sel=None) -> np.ndarray:
    """Off-grid values of a contiguous tensor (queries [B, T, Hq, d], new rows [B, T, Hkv, d]),
    element i hashed by its flat index; b_sel selects rows of the leading dimension."""
    shape = tuple(shape)
    per = int(np.prod(shape[1:]))
    bs = np.arange(shape[0]) if b_sel is None else np.asarray(b_sel)
    idx = (bs[:, None].astype(U64) * U64(per) + np.arange(per, dtype=np.int64)[None, :].astype(U64))
    return offgrid_bits_from_hash(hash_u64(seed, tensor, idx)).reshape((len(bs),) + shape[1:])


# ----------------------------------------------------------------------------------------
# lengths
# ----------------------------------------------------------------------------------------
def committed_lengths(seed: int, B: int, ctx: int, gamma: int, ragged: bool) -> np.ndarray:
    """L_b = ctx (uniform) or ctx - (h(b) mod (gamma+1)) (ragged)."""
    if not ragged:
        return np.full(B, ctx, dtype=np.int32)
    h = hash_u64(seed, T_LEN, np.arange(B))
    return (ctx - (h % U64(gamma + 1)).astype(np.int64)).astype(np.int32)


# ----------------------------------------------------------------------------------------
# probabilities for spec_accept
# ----------------------------------------------------------------------------------------
def _uniform01(seed, tensor, idx):
    """fp64 uniform in (0,1) from the top 53 bits."""
    h = hash_u64(seed, tensor, idx)
    return ((h >> U64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def zipf_logits(seed: int, row: int, V: int, s: float = 1.1) -> np.ndarray:
    """Zipf(s) log-weights over a hashed permutation of the vocabulary for one row."""
    keys = hash_u64(seed, T_LOGIT, np.arange(V, dtype=np.int64) + np.int64(row) * np.int64(1 << 32))
    rank = np.empty(V, dtype=np.int64)
    rank[np.argsort(keys, kind="stable")] = np.arange(V)
    return -s * np.log1p(rank.astype(np.float64))


def _softmax64(z):
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def normal_noise(seed: int, row: int, V: int) -> np.ndarray:
    i = np.arange(V, dtype=np.int64) + np.int64(row) * np.int64(1 << 32)
    u1 = _uniform01(seed, T_NOISE, 2 * i)
    u2 = _uniform01(seed, T_NOISE, 2 * i + 1)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def spec_probs(seed: int, B: int, gamma: int, V: int, sigma: float, zipf_s: float = 1.1):
    """p [B, gamma+1, V] fp32 (target rows), q [B, gamma, V] fp32 (draft rows), and
    draft tokens d [B, gamma] int32 sampled from q (the drafter's own sampler,
    upstream of spec_accept).  p = softmax(zipf), q = softmax(log p + sigma * xi);
    sigma controls the overlap beta = sum min(p, q) (the per-position acceptance
    rate).  Computed in fp64 and rounded to fp32."""
    p = np.empty((B, gamma + 1, V), dtype=np.float32)
    q = np.empty((B, gamma, V), dtype=np.float32)
    d = np.empty((B, gamma), dtype=np.int32)
    for b in range(B):
        for j in range(gamma + 1):
            row = b * (gamma + 1) + j
            z = zipf_logits(seed, row, V, zipf_s)
            p[b, j] = _softmax64(z).astype(np.float32)
            if j < gamma:
                qz = z + sigma * normal_noise(seed, row, V)
                q64 = _softmax64(qz)
                q[b, j] = q64.astype(np.float32)
                u = _uniform01(seed, T_DRAFTU, np.array([row]))[0]
                cdf = np.cumsum(q[b, j].astype(np.float64))
                d[b, j] = min(int(np.searchsorted(cdf, u * cdf[-1], side="right")), V - 1)
    return p, q, d


def overlap(p_row: np.ndarray, q_row: np.ndarray) -> float:
    """beta = sum_x min(p, q)(x), in fp64 (input recipe diagnostic only)."""
    return float(np.minimum(p_row.astype(np.float64), q_row.astype(np.float64)).sum())


def sigma_for_overlap(seed: int, V: int, target: float, rows: int = 4, zipf_s: float = 1.1) -> float:
    """Bisect sigma so the mean overlap of a few sample rows is ~target."""
    zs = [zipf_logits(seed ^ 0x5A5A, r, V, zipf_s) for r in range(rows)]
    ns = [normal_noise(seed ^ 0x5A5A, r, V) for r in range(rows)]
    lo, hi = 0.0, 8.0
    for _ in range(40):
        mid = 0.5 * (lo + hi)
        beta = np.mean([overlap(_softmax64(z), _softmax64(z + mid * n)) for z, n in zip(zs, ns)])
        if beta > target:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


# ----------------------------------------------------------------------------------------
# PQCache codebooks.  The codebook is trained at prefill (k-means,
# outside the decode hot path); the synthetic stand-in takes centroid c of sub-space m to be
# sub-vector m of the unit's own key at a hashed prompt position (the usual k-means
# initialisation), so it lies on the same exact bf16 grid as the keys.
# ----------------------------------------------------------------------------------------
T_PQCB = 13
PQ_M, PQ_C = 16, 256


def pq_codebook_positions(seed: int, B: int, Hkv: int, L) -> np.ndarray:
    """int64 [B, Hkv, 16, 256]: prompt position (in [0, L_b)) whose key sub-vector m seeds
    centroid c."""
    L = np.asarray(L, dtype=np.int64).reshape(B)
    b, u, m, c = np.meshgrid(np.arange(B), np.arange(Hkv), np.arange(PQ_M), np.arange(PQ_C), indexing="ij")
    idx = (((b * Hkv + u) * PQ_M + m) * PQ_C + c).astype(U64)
    return (hash_u64(seed, T_PQCB, idx) % L[b].astype(U64)).astype(np.int64)


def pq_codebook_bits(k_bits: np.ndarray, positions: np.ndarray) -> np.ndarray:
    """bf16 bits [B, Hkv, 16, 256, d/16]: gathered key sub-vectors (k_bits [B, Hkv, cap, d])."""
    B, Hkv, _, d = k_bits.shape
    s = d // PQ_M
    b, u, c = np.meshgrid(np.arange(B), np.arange(Hkv), np.arange(PQ_C), indexing="ij")
    out = np.empty((B, Hkv, PQ_M, PQ_C, s), dtype=np.uint16)
    for mm in range(PQ_M):
        out[:, :, mm] = k_bits[b, u, positions[:, :, mm], mm * s:(mm + 1) * s]
    return out
