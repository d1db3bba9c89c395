"""Time PQCache dynamic selection (md_pq_select = T_select of Eq.3) and the draft over
the selected set (md_draft_attn_indexed = T_D(B, K)) for BASELINE configs (CUDA events; two
code buffers and two layer caches rotated so every call streams from HBM).
Budget split: sink 4 + top-k + window, total = the config's StreamingLLM budget, window = half.
usage: python tools/pq_sweep.py [cfg ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402
import synth as S  # noqa: E402
import synth.cuda as SC  # noqa: E402
from bench import CONFIGS, SEED  # noqa: E402


def sweep(cfg, R=2, reps=10):
    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[cfg]
    budget_total = sink + window
    win = budget_total // 2
    topk = budget_total - sink - win
    cap = ctx + 64
    reg = S.Regime("peaky", sink=sink)
    L0 = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
    kc, vc, cbs, codes = [], [], [], []
    pos = torch.from_numpy(S.pq_codebook_positions(SEED, B, Hkv, L0)).cuda()
    bi = torch.arange(B, device="cuda")[:, None, None, None]
    ui = torch.arange(Hkv, device="cuda")[None, :, None, None]
    s = d // 16
    for r in range(R):
        k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        SC.fill_cache(k, SEED + r, S.T_KCACHE, 0, cap, reg)
        SC.fill_cache(v, SEED + r, S.T_VCACHE, 0, cap, reg)
        cb = torch.empty((B, Hkv, 16, 256, s), dtype=torch.bfloat16, device="cuda")
        for m in range(16):
            cb[:, :, m] = k[bi[..., 0], ui[..., 0], pos[:, :, m]][..., m * s:(m + 1) * s]
        c = torch.zeros((B, Hkv, cap, 16), dtype=torch.uint8, device="cuda")
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        md.pq_encode(k, v, cb, torch.zeros(B, dtype=torch.int32, device="cuda"), ctx, c)
        t1.record()
        torch.cuda.synchronize()
        enc_ms = t0.elapsed_time(t1)
        kc.append(k)
        vc.append(v)
        cbs.append(cb)
        codes.append(c)
    qd = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_q(qd, SEED, S.T_QDRAFT, Hkv, reg)
    kvl_np = (L0 + 1).astype(np.int32)
    kvl = torch.from_numpy(kvl_np).cuda()
    K = (sink + topk + 3) // 4 * 4
    idx = torch.zeros((B, Hkv, K), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(B, dtype=torch.int32, device="cuda")
    tail = torch.zeros(B, dtype=torch.int32, device="cuda")
    ws = torch.empty(md.pq_workspace_bytes(B, Hkv, cap), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, Hq, d), device="cuda")
    lse = torch.empty((B, Hq), device="cuda")
    wsd = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, cap), dtype=torch.uint8, device="cuda")
    scale = float(np.float32(1 / np.sqrt(d)))

    def sel(r):
        md.pq_select(qd, cbs[r % R], codes[r % R], kvl, cap, sink, win, topk, idx, cnt, tail, ws)

    def draft(r):
        md.draft_attn_indexed(qd, kc[r % R], vc[r % R], kvl, idx, cnt, tail, scale, out, lse, wsd)

    def timeit(fn):
        fn(0)
        torch.cuda.synchronize()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for r in range(reps):
            fn(r)
        b_.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b_) / reps

    sel_ms = timeit(sel)
    draft_ms = timeit(draft)
    both_ms = timeit(lambda r: (sel(r), draft(r)))
    cand = np.maximum(0, kvl_np - win - sink).astype(np.int64)
    scan_bytes = int(cand.sum()) * Hkv * 16 + B * Hkv * (16 * 256 * s * 2 + 16 * 256 * 4 * 2) + B * Hq * d * 2
    keys = np.minimum(kvl_np, sink + topk + win).astype(np.int64)
    draft_bytes = int(keys.sum()) * Hkv * d * 4 + B * Hq * d * 6
    return {"cfg": cfg, "sink": sink, "topk": topk, "window": win, "encode_prefill_ms": round(enc_ms, 2),
            "select_us": round(sel_ms * 1e3, 2), "select_code_scan_gbs": round(scan_bytes / sel_ms / 1e6, 1),
            "draft_us": round(draft_ms * 1e3, 2), "draft_gbs": round(draft_bytes / draft_ms / 1e6, 1),
            "select_plus_draft_us": round(both_ms * 1e3, 2)}


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["llama3_b64_32k", "llama2_8k", "qwen_100k"]
    for c in cfgs:
        print(json.dumps(sweep(c)), flush=True)
        torch.cuda.empty_cache()
