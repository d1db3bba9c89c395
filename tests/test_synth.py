"""Input-generator checks (CPU): determinism, the exact bf16 grid, slice consistency,
length recipes and the probability recipe.  The CUDA generator's bit-exactness
against this module is checked in tests/test_gpu_synth.py."""
import numpy as np

import synth as S


def test_grid_values_exact_and_in_range():
    k = S.kv_cache_k(1, S.T_KCACHE, 2, 3, 64, 0, 50)
    assert k.min() >= -32 and k.max() <= 31
    bits = S.k_to_bf16_bits(k)
    assert np.array_equal(S.bf16_bits_to_f32(bits).astype(np.float64), k / 32.0)


def test_slices_are_consistent_and_deterministic():
    a = S.kv_cache_k(5, S.T_VCACHE, 4, 2, 16, 0, 100)
    b = S.kv_cache_k(5, S.T_VCACHE, 4, 2, 16, 40, 30, b_sel=[1, 3], h_sel=[1])
    assert np.array_equal(a[[1, 3]][:, [1], 40:70], b)
    assert np.array_equal(a, S.kv_cache_k(5, S.T_VCACHE, 4, 2, 16, 0, 100))
    assert not np.array_equal(a, S.kv_cache_k(6, S.T_VCACHE, 4, 2, 16, 0, 100))


def test_peaky_regime_stays_on_exact_bf16_grid():
    reg = S.Regime("peaky", sink=4)
    k = S.kv_cache_k(2, S.T_KCACHE, 2, 2, 128, 0, 5000, regime=reg)
    q = S.q_rows_k(2, S.T_QVERIFY, 2, 5, 8, 2, 128, regime=reg)
    assert np.abs(k).max() <= 256 and np.abs(q).max() <= 256
    assert np.array_equal(S.bf16_bits_to_f32(S.k_to_bf16_bits(k)).astype(np.float64), k / 32.0)
    # sinks are boosted: |k| > 31 occurs at positions < 4
    assert np.abs(k[:, :, :4]).max() > 31


def test_ragged_lengths():
    L = S.committed_lengths(3, 64, 1000, 4, ragged=True)
    assert L.min() >= 996 and L.max() <= 1000 and len(set(L.tolist())) > 1
    assert np.all(S.committed_lengths(3, 8, 1000, 4, ragged=False) == 1000)


def test_spec_probs_rows_are_distributions_and_overlap_tracks_sigma():
    p, q, d = S.spec_probs(11, 2, 3, 500, sigma=0.5)
    assert np.allclose(p.sum(-1), 1, atol=1e-5) and np.allclose(q.sum(-1), 1, atol=1e-5)
    assert d.min() >= 0 and d.max() < 500
    p2, q2, _ = S.spec_probs(11, 2, 3, 500, sigma=2.0)
    b1 = np.mean([S.overlap(p[b, j], q[b, j]) for b in range(2) for j in range(3)])
    b2 = np.mean([S.overlap(p2[b, j], q2[b, j]) for b in range(2) for j in range(3)])
    assert b1 > b2


def test_offgrid_values_are_off_grid_and_bounded():
    """Off-grid generator: every value is a finite bf16 with |x| in [2^-7, 1), most are not
    multiples of 1/32 (so fp32 rounding happens in the attention), signs are balanced."""
    bits = S.kv_cache_bits_offgrid(5, S.T_KCACHE, 2, 3, 128, 0, 200)
    x = S.bf16_bits_to_f32(bits).astype(np.float64)
    assert np.all(np.isfinite(x)) and np.all(np.abs(x) < 1.0) and np.all(np.abs(x) >= 2.0 ** -7)
    assert np.mean(np.abs(x * 32 - np.round(x * 32)) > 0) > 0.5
    assert abs(np.mean(np.sign(x))) < 0.05
    q = S.flat_bits_offgrid(5, S.T_QVERIFY, (2, 5, 8, 64))
    assert q.shape == (2, 5, 8, 64) and np.array_equal(q[1:], S.flat_bits_offgrid(5, S.T_QVERIFY, (2, 5, 8, 64), [1]))
