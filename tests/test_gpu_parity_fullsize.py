"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times: the SAME
fused calls (md_draft_attn_sparse_append, then md_verify_attn_full_append with the bench's
max_kv_len bound), the same shapes, ragged lengths and split plan.  The caches, queries and new
rows are generated in HBM by the CUDA twins of the synth generators; for >= 8 sampled sequences
(the shortest and longest ragged lengths, the first and last sequence and seeded others) and some
of their KV heads the oracle regenerates the inputs on the host, applies the step's appends and
computes those outputs one by one in fp64 (worker processes).  Two value regimes: the peaky
k/32-grid inputs the bench runs, and arbitrary (off-grid) bf16 inputs with |x| < 1, where fp32
rounding really occurs.  Tolerances (north_star): outputs 2e-3 max-abs, lse 1e-3; the appended
cache rows bit-exact.  The observed max and 99.99th-percentile errors are printed (and written to
$MD_PARITY_REPORT, one JSON line per case, when set)."""
import json
import os

import numpy as np
import pytest
import torch

import paper_2408_11049_b200 as md
import synth as S
import synth.cuda as SC
from tests import fullsize_oracle as FO

pytestmark = pytest.mark.gpu

ATOL_O, ATOL_LSE = 2e-3, 1e-3

# name, B, Hq, Hkv, d, ctx, gamma, sink, window   (BASELINE.json configs)
FULL = {
    "llama2_8k": (64, 32, 32, 128, 8192, 3, 4, 508),
    "llama3_b64_32k": (64, 32, 8, 128, 32768, 4, 4, 1020),
    "qwen_100k": (64, 28, 4, 128, 100000, 4, 4, 2044),
    "llama3_32k": (128, 32, 8, 128, 32768, 4, 4, 1020),
    "llama3_scaling": (256, 32, 8, 128, 32768, 4, 4, 1020),
}
CASES = [(n, "peaky") for n in FULL] + [("llama3_b64_32k", "offgrid"), ("qwen_100k", "offgrid")]


def _sampled(L, B, n=8):
    rng = np.random.default_rng(B)
    pick = {int(np.argmin(L)), int(np.argmax(L)), 0, B - 1}
    while len(pick) < n:
        pick.add(int(rng.integers(0, B)))
    return sorted(pick)


def _bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("name,kind", CASES)
def test_fullsize_sampled_parity_of_the_bench_calls(name, kind):
    B, Hq, Hkv, d, ctx, gamma, sink, window = FULL[name]
    T, seed = gamma + 1, FO.SEED
    L = S.committed_lengths(seed, B, ctx, gamma, ragged=True)
    cap = ctx + 40
    max_kv = int(L.max()) + 5 * T          # bench.py passes a bound above every kv_len
    reg = S.Regime("peaky", sink=4)
    k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    qv = torch.empty((B, T, Hq, d), dtype=torch.bfloat16, device="cuda")
    qd = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
    knd = torch.empty((B, 1, Hkv, d), dtype=torch.bfloat16, device="cuda")
    vnd, knv, vnv = torch.empty_like(knd), torch.empty((B, T, Hkv, d), dtype=torch.bfloat16, device="cuda"), None
    vnv = torch.empty_like(knv)
    if kind == "offgrid":
        SC.fill_cache_offgrid(k, seed, S.T_KCACHE, 0, cap)
        SC.fill_cache_offgrid(v, seed, S.T_VCACHE, 0, cap)
        SC.fill_flat_offgrid(qv, seed, S.T_QVERIFY)
        SC.fill_flat_offgrid(qd, seed, S.T_QDRAFT)
        SC.fill_flat_offgrid(knd, seed + 1, S.T_KNEW)
        SC.fill_flat_offgrid(vnd, seed + 1, S.T_VNEW)
        SC.fill_flat_offgrid(knv, seed, S.T_KNEW)
        SC.fill_flat_offgrid(vnv, seed, S.T_VNEW)
    else:
        SC.fill_cache(k, seed, S.T_KCACHE, 0, cap, reg)
        SC.fill_cache(v, seed, S.T_VCACHE, 0, cap, reg)
        SC.fill_q(qv, seed, S.T_QVERIFY, Hkv, reg)
        SC.fill_q(qd, seed, S.T_QDRAFT, Hkv, reg)
        SC.fill_new_kv(knd, seed + 1, S.T_KNEW)
        SC.fill_new_kv(vnd, seed + 1, S.T_VNEW)
        SC.fill_new_kv(knv, seed, S.T_KNEW)
        SC.fill_new_kv(vnv, seed, S.T_VNEW)
    scale = float(np.float32(1 / np.sqrt(d)))
    kv_d = torch.from_numpy((L + 1).astype(np.int32)).cuda()
    kv_v = torch.from_numpy((L + T).astype(np.int32)).cuda()
    out_d = torch.full((B, Hq, d), float("nan"), device="cuda")
    lse_d = torch.full((B, Hq), float("nan"), device="cuda")
    out_v = torch.full((B, T, Hq, d), float("nan"), device="cuda")
    lse_v = torch.full((B, T, Hq), float("nan"), device="cuda")
    ws_d = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, min(sink + window, cap)), dtype=torch.uint8,
                       device="cuda")
    ws_v = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, max_kv), dtype=torch.uint8, device="cuda")
    # one step of one layer, exactly as bench.py launches it
    md.draft_attn_sparse_append(qd, k, v, knd, vnd, kv_d, sink, window, scale, out_d, lse_d, ws_d)
    od, ldr = out_d.cpu().numpy(), lse_d.cpu().numpy()
    md.verify_attn_full_append(qv, k, v, knv, vnv, kv_v, max_kv, scale, out_v, lse_v, ws_v)
    torch.cuda.synchronize()
    ov, lv = out_v.cpu().numpy(), lse_v.cpu().numpy()
    assert np.all(np.isfinite(od)) and np.all(np.isfinite(ov)) and np.all(np.isfinite(lv))
    seqs = _sampled(L, B)
    nh = 1 if ctx > 50000 else 2
    jobs = [(kind, B, Hq, Hkv, d, T, sink, window, scale, b, [(b * 3 + i * (Hkv // nh + 1)) % Hkv for i in range(nh)],
             int(L[b])) for b in seqs]
    import concurrent.futures as cf
    import multiprocessing as mp
    with cf.ProcessPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1),
                                mp_context=mp.get_context("spawn")) as ex:
        results = list(ex.map(FO.oracle_one, jobs))
    g = Hq // Hkv
    errs = {"draft_o": [], "draft_lse": [], "verify_o": [], "verify_lse": []}
    for b, heads, rod, rld, rov, rlv, rk, rv in results:
        qh = np.concatenate([np.arange(h * g, (h + 1) * g) for h in heads])
        errs["draft_o"].append(np.abs(od[b, qh] - rod).ravel())
        errs["draft_lse"].append(np.abs(ldr[b, qh] - rld).ravel())
        errs["verify_o"].append(np.abs(ov[b][:, qh] - rov).ravel())
        errs["verify_lse"].append(np.abs(lv[b][:, qh] - rlv).ravel())
        n0 = int(L[b])
        assert np.array_equal(_bits(k[b, heads, n0:n0 + T]), rk), (b, "K rows")
        assert np.array_equal(_bits(v[b, heads, n0:n0 + T]), rv), (b, "V rows")
    rep = {"case": f"{name}/{kind}", "sequences": seqs, "kv_heads_per_sequence": nh,
           "outputs_checked": int(sum(len(e) for e in errs["verify_o"]) + sum(len(e) for e in errs["draft_o"]))}
    for key, lst in errs.items():
        e = np.concatenate(lst)
        rep[key] = {"max": float(e.max()), "p99.99": float(np.percentile(e, 99.99))}
    print(json.dumps(rep))
    if os.environ.get("MD_PARITY_REPORT"):
        with open(os.environ["MD_PARITY_REPORT"], "a") as f:
            f.write(json.dumps(rep) + "\n")
    assert rep["draft_o"]["max"] <= ATOL_O and rep["verify_o"]["max"] <= ATOL_O, rep
    assert rep["draft_lse"]["max"] <= ATOL_LSE and rep["verify_lse"]["max"] <= ATOL_LSE, rep
    del k, v
    torch.cuda.empty_cache()
