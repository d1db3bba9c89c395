"""Statistical checks of md_spec_accept at scale (GPU, SAMPLE mode).

With the same (p, q) rows broadcast to B = 2^16 sequences, d_j ~ q_j drawn per sequence
and Philox uniforms, the emitted stream must follow the target law (SD is lossless):
the first emitted token ~ p_0, the accepted count ~ the truncated-geometric law
P(n = k) = prod_{i<k} beta_i (1 - beta_k), and E[n + 1] = Eq.1 when all
beta_i = alpha.  Chi-square p-values > 1e-3."""
import numpy as np
import pytest
import torch
from scipy import stats

import paper_2408_11049_b200 as md
from oracle.theory import accepted_count_pmf, omega

pytestmark = pytest.mark.gpu


def _rows(rng, n, V):
    w = rng.random((n, V)) ** 2
    return (w / w.sum(-1, keepdims=True)).astype(np.float32)


def _overlap(p, q):
    return float(np.minimum(p.astype(np.float64), q.astype(np.float64)).sum())


def test_accept_law_matches_target_at_scale():
    B, gamma, V = 1 << 16, 4, 32
    rng = np.random.default_rng(123)
    p1 = _rows(rng, gamma + 1, V)
    q1 = _rows(rng, gamma, V)
    p = torch.from_numpy(np.broadcast_to(p1, (B, gamma + 1, V)).copy()).cuda()
    q = torch.from_numpy(np.broadcast_to(q1, (B, gamma, V)).copy()).cuda()
    # draft tokens d_j ~ q_j per sequence: inverse CDF with host uniforms (input generation)
    u = rng.random((B, gamma))
    cdf = np.cumsum(q1.astype(np.float64), -1)
    d = np.stack([np.minimum(np.searchsorted(cdf[j] / cdf[j, -1], u[:, j], side="right"), V - 1)
                  for j in range(gamma)], 1).astype(np.int32)
    rnd = torch.empty((B, gamma + 2), dtype=torch.int32, device="cuda")
    md.philox_u32(99, 7, rnd)
    out = torch.empty((B, gamma + 1), dtype=torch.int32, device="cuda")
    n = torch.empty(B, dtype=torch.int32, device="cuda")
    md.spec_accept(p, q, torch.from_numpy(d).cuda(), rnd, out, n)
    torch.cuda.synchronize()
    out, n = out.cpu().numpy(), n.cpu().numpy()
    # first emitted token ~ p_0
    cnt = np.bincount(out[:, 0], minlength=V)
    exp = p1[0].astype(np.float64) * B
    keep = exp > 5
    chi = stats.chisquare(cnt[keep], exp[keep] * cnt[keep].sum() / exp[keep].sum())
    assert chi.pvalue > 1e-3, chi
    # accepted count ~ prod(beta) law
    betas = [_overlap(p1[j], q1[j]) for j in range(gamma)]
    pmf = np.array(accepted_count_pmf(betas))
    cn = np.bincount(n, minlength=gamma + 1)
    chi = stats.chisquare(cn, pmf * B)
    assert chi.pvalue > 1e-3, (cn, pmf * B)


def test_mean_emitted_tokens_matches_eq1():
    """beta_i = alpha for every position: E[n + 1] = Omega(gamma, alpha) (Eq.1)."""
    B, gamma, V, alpha = 1 << 16, 4, 16, 0.75
    # p = (alpha on 0 ..) construct q with overlap exactly alpha: p uniform on {0..7}, q uniform on {2..9}
    p1 = np.zeros((gamma + 1, V), np.float32)
    q1 = np.zeros((gamma, V), np.float32)
    p1[:, 0:8] = 1 / 8
    q1[:, 2:10] = 1 / 8                      # overlap 6/8 = 0.75
    rng = np.random.default_rng(5)
    d = rng.integers(2, 10, size=(B, gamma)).astype(np.int32)
    p = torch.from_numpy(np.broadcast_to(p1, (B, gamma + 1, V)).copy()).cuda()
    q = torch.from_numpy(np.broadcast_to(q1, (B, gamma, V)).copy()).cuda()
    rnd = torch.empty((B, gamma + 2), dtype=torch.int32, device="cuda")
    md.philox_u32(3, 1, rnd)
    out = torch.empty((B, gamma + 1), dtype=torch.int32, device="cuda")
    n = torch.empty(B, dtype=torch.int32, device="cuda")
    cl = torch.zeros(B, dtype=torch.int32, device="cuda")
    md.spec_accept(p, q, torch.from_numpy(d).cuda(), rnd, out, n, cl)
    torch.cuda.synchronize()
    emitted = cl.cpu().numpy().astype(np.float64)
    mean, se = emitted.mean(), emitted.std() / np.sqrt(B)
    assert abs(mean - omega(gamma, alpha)) < 4 * se, (mean, omega(gamma, alpha), se)
    # every emitted token lies in p's support (lossless: never a token p gives 0)
    o = out.cpu().numpy()
    assert np.all(o[o >= 0] < 10) and np.all((o[np.arange(B), n.cpu().numpy()] < 8))
