"""The CUDA input generator (synth/csrc) is bit-identical to the numpy one (synth/__init__.py)."""
import numpy as np
import pytest
import torch

import synth as S
import synth.cuda as SC

pytestmark = pytest.mark.gpu


def _bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("regime", [S.FLAT, S.Regime("peaky", sink=4, needle_period=37)])
def test_cache_generator_bit_exact(regime):
    B, H, cap, d = 3, 4, 300, 128
    k = torch.zeros((B, H, cap, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_cache(k, 11, S.T_KCACHE, 0, 250, regime)
    SC.fill_cache(k, 11, S.T_KCACHE, 250, 50, regime)
    ref = S.k_to_bf16_bits(S.kv_cache_k(11, S.T_KCACHE, B, H, d, 0, cap, regime=regime))
    assert np.array_equal(_bits(k), ref)
    # strided (NHD) destination
    v = torch.zeros((B, cap, H, d), dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3)
    SC.fill_cache(v, 11, S.T_VCACHE, 0, cap, regime)
    ref = S.k_to_bf16_bits(S.kv_cache_k(11, S.T_VCACHE, B, H, d, 0, cap, regime=regime))
    assert np.array_equal(_bits(v.contiguous()), ref)


@pytest.mark.parametrize("regime", [S.FLAT, S.Regime("peaky")])
def test_query_and_new_kv_generators_bit_exact(regime):
    q = torch.empty((3, 5, 32, 128), dtype=torch.bfloat16, device="cuda")
    SC.fill_q(q, 4, S.T_QVERIFY, 8, regime)
    assert np.array_equal(_bits(q), S.k_to_bf16_bits(S.q_rows_k(4, S.T_QVERIFY, 3, 5, 32, 8, 128, regime=regime)))
    qd = torch.empty((3, 28, 128), dtype=torch.bfloat16, device="cuda")
    SC.fill_q(qd, 4, S.T_QDRAFT, 4, regime)
    assert np.array_equal(_bits(qd), S.k_to_bf16_bits(S.q_rows_k(4, S.T_QDRAFT, 3, 1, 28, 4, 128, regime=regime))[:, 0])
    kn = torch.empty((3, 5, 8, 128), dtype=torch.bfloat16, device="cuda")
    SC.fill_new_kv(kn, 4, S.T_KNEW)
    assert np.array_equal(_bits(kn), S.k_to_bf16_bits(S.new_kv_k(4, S.T_KNEW, 3, 5, 8, 128)))


def test_cache_slice_generator_equals_the_full_cache_slice():
    """A tensor-parallel / batch shard (b0, h0 of a cache with Hkv_total heads) holds exactly the
    full cache's values, so sharded runs see the same inputs as the single-GPU run."""
    reg = S.Regime("peaky", sink=4, needle_period=37)
    B, H, cap, d = 4, 8, 200, 128
    full = S.k_to_bf16_bits(S.kv_cache_k(13, S.T_KCACHE, B, H, d, 0, cap, regime=reg))
    shard = torch.zeros((2, 2, cap, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_cache(shard, 13, S.T_KCACHE, 0, cap, reg, b0=2, h0=4, Hkv_total=H)
    assert np.array_equal(_bits(shard), full[2:4, 4:6])


def test_offgrid_generators_bit_exact():
    B, H, cap, d = 3, 4, 130, 128
    k = torch.zeros((B, H, cap, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_cache_offgrid(k, 17, S.T_KCACHE, 0, cap)
    assert np.array_equal(_bits(k), S.kv_cache_bits_offgrid(17, S.T_KCACHE, B, H, d, 0, cap))
    shard = torch.zeros((1, 2, cap, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_cache_offgrid(shard, 17, S.T_KCACHE, 0, cap, b0=2, h0=1, Hkv_total=H)
    assert np.array_equal(_bits(shard), S.kv_cache_bits_offgrid(17, S.T_KCACHE, B, H, d, 0, cap)[2:3, 1:3])
    q = torch.zeros((3, 5, 32, 128), dtype=torch.bfloat16, device="cuda")
    SC.fill_flat_offgrid(q, 17, S.T_QVERIFY)
    assert np.array_equal(_bits(q), S.flat_bits_offgrid(17, S.T_QVERIFY, (3, 5, 32, 128)))
    assert np.array_equal(_bits(q)[1:2], S.flat_bits_offgrid(17, S.T_QVERIFY, (3, 5, 32, 128), b_sel=[1]))
