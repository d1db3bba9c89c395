"""Time md_verify_attn_full / md_draft_attn_sparse alone for BASELINE configs (CUDA events,
rotated layer caches so every call streams from HBM).  usage: python tools/attn_sweep.py [cfg ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402
import synth as S  # noqa: E402
import synth.cuda as SC  # noqa: E402
from bench import CONFIGS, SEED, draft_bytes, verify_bytes  # noqa: E402


def sweep(cfg, R=3, reps=12):
    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[cfg]
    T = gamma + 1
    cap = ctx + 64
    reg = S.Regime("peaky", sink=sink)
    L0 = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
    kc, vc = [], []
    for r in range(R):
        k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        SC.fill_cache(k, SEED + r, S.T_KCACHE, 0, cap, reg)
        SC.fill_cache(v, SEED + r, S.T_VCACHE, 0, cap, reg)
        kc.append(k)
        vc.append(v)
    qv = torch.empty((B, T, Hq, d), dtype=torch.bfloat16, device="cuda")
    qd = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_q(qv, SEED, S.T_QVERIFY, Hkv, reg)
    SC.fill_q(qd, SEED, S.T_QDRAFT, Hkv, reg)
    kvv = torch.from_numpy((L0 + T).astype(np.int32)).cuda()
    kvd = torch.from_numpy((L0 + 1).astype(np.int32)).cuda()
    mkl = int(L0.max()) + T
    scale = float(np.float32(1 / np.sqrt(d)))
    out_v = torch.empty((B, T, Hq, d), device="cuda")
    lse_v = torch.empty((B, T, Hq), device="cuda")
    out_d = torch.empty((B, Hq, d), device="cuda")
    lse_d = torch.empty((B, Hq), device="cuda")
    ws_v = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, T, mkl)), dtype=torch.uint8, device="cuda")
    ws_d = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, 1, cap)), dtype=torch.uint8, device="cuda")

    def t(fn):
        fn(0)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(reps):
            fn(i)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    vms = t(lambda i: md.verify_attn_full(qv, kc[i % R], vc[i % R], kvv, mkl, scale, out_v, lse_v, ws_v))
    dms = t(lambda i: md.draft_attn_sparse(qd, kc[i % R], vc[i % R], kvd, sink, window, scale, out_d, lse_d, ws_d))
    # SnapKV draft: 2048-token budget = 2016 listed prefix rows + the 32-token window tail,
    # selected by md_snapkv_select from window queries of the same synthetic regime (the
    # selection is clustered by the 5-wide pooling, as SnapKV's is)
    w_obs, budget = 32, 2048
    q_obs = torch.empty((B, w_obs, Hq, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_q(q_obs, SEED + 7, S.T_QVERIFY, Hkv, reg)
    plen = torch.from_numpy(L0.astype(np.int32)).cuda()
    idx_t = torch.zeros((B, Hkv, budget), dtype=torch.int32, device="cuda")
    cnt_t = torch.zeros(B, dtype=torch.int32, device="cuda")
    md.snapkv_select(kc[0], vc[0], q_obs, plen, int(L0.max()), w_obs, budget, scale, idx_t, cnt_t)
    torch.cuda.synchronize()
    idx_np = idx_t.cpu().numpy()[:, :, : budget - w_obs]
    runs = float(np.mean(np.diff(idx_np, axis=2) == 1))
    tail_t = torch.from_numpy((L0 - w_obs).astype(np.int32)).cuda()
    sms = t(lambda i: md.draft_attn_indexed(qd, kc[i % R], vc[i % R], kvd, idx_t, cnt_t, tail_t, scale, out_d, lse_d,
                                            ws_d))
    sb = int(B * Hkv * (budget + 1) * d * 4 + B * Hq * d * 6 + B * Hq * 4)
    vb = verify_bytes(L0 + T, Hkv, Hq, d, T)
    db = draft_bytes(L0 + 1, Hkv, Hq, d, sink, window)
    res = {"cfg": cfg, "verify_ms": round(vms, 4), "verify_gbs": round(vb / vms / 1e6, 1),
           "draft_us": round(dms * 1e3, 2), "draft_gbs": round(db / dms / 1e6, 1),
           "snapkv_draft_us": round(sms * 1e3, 2), "snapkv_draft_gbs": round(sb / sms / 1e6, 1),
           "snapkv_adjacent_fraction": round(runs, 3),
           "env": {k: v for k, v in os.environ.items() if k.startswith("MD_")}}
    print(json.dumps(res), flush=True)
    del kc, vc
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["llama3_b64_32k", "llama2_8k", "qwen_100k", "llama3_32k"]):
        sweep(c)
