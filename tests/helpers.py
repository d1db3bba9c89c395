"""Shared test helpers: build seeded inputs (synth) as numpy bit arrays for the oracle and
as CUDA tensors for the library.  No arithmetic of the method lives here."""
from __future__ import annotations

import numpy as np
import torch

import synth as S


def bits_to_torch_bf16(bits: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(device)


class AttnCase:
    """A KV cache + verify/draft queries built from the synth generators."""

    def __init__(self, B, Hq, Hkv, d, cap, kv_len, T=1, seed=1, regime=S.FLAT):
        self.B, self.Hq, self.Hkv, self.d, self.cap, self.T = B, Hq, Hkv, d, cap, T
        self.kv_len = np.asarray(kv_len, dtype=np.int32)
        self.seed, self.regime = seed, regime
        self.k_bits = S.k_to_bf16_bits(S.kv_cache_k(seed, S.T_KCACHE, B, Hkv, d, 0, cap, regime=regime))
        self.v_bits = S.k_to_bf16_bits(S.kv_cache_k(seed, S.T_VCACHE, B, Hkv, d, 0, cap, regime=regime))
        self.qv_bits = S.k_to_bf16_bits(S.q_rows_k(seed, S.T_QVERIFY, B, T, Hq, Hkv, d, regime=regime))
        self.qd_bits = S.k_to_bf16_bits(S.q_rows_k(seed, S.T_QDRAFT, B, 1, Hq, Hkv, d, regime=regime))[:, 0]
        self.scale = float(np.float32(1.0 / np.sqrt(d)))

    def to_cuda(self):
        self.k = bits_to_torch_bf16(self.k_bits)
        self.v = bits_to_torch_bf16(self.v_bits)
        self.qv = bits_to_torch_bf16(self.qv_bits)
        self.qd = bits_to_torch_bf16(self.qd_bits)
        self.kv_len_t = torch.from_numpy(self.kv_len).cuda()
        return self
