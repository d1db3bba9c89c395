"""Per-rank kernel time of the KV-head tensor-parallel split measured
on one B200: for P = 1, 2, 4, 8 the verify and draft calls run on the shard a rank owns (all B
sequences, Hkv / P KV heads with their g*Hkv/P query heads; the fused-append calls bench.py
times), graph-timed back to back over rotated layer caches, and
    E_kernel(P) = T(1) / (P * T_shard(P))
is the scaling efficiency of the attention kernels alone: each rank streams 1/P of the bytes on
its own GPU, so this is what the P-GPU call costs before the output exchange (the all-gather of
[B, T, Hq/P, d] fp32 per call, or the fused peer-store epilogue; volume printed, not timed: this
pool has one GPU per call).  Not a multi-GPU measurement: no NVLink traffic, no clock or power
interaction between GPUs.
usage: python tools/shard_scaling.py [config]      (default llama3_scaling: B=256, ctx 32k)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402
import synth as S  # noqa: E402
import synth.cuda as SC  # noqa: E402
from bench import CONFIGS, SEED, draft_bytes, graph_time_calls, verify_bytes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "llama3_scaling"
B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[cfg]
T, rot = gamma + 1, 2
reg = S.Regime("peaky", sink=sink)
L0 = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
cap = ctx + 2 * T + 8
kvl = (L0 + T).astype(np.int32)
scale = float(np.float32(1 / np.sqrt(d)))
md.load_library()
res = {"config": cfg, "batch": B, "ctx": ctx, "gamma": gamma, "P": {}}
t1 = None
for P in (1, 2, 4, 8):
    if Hkv % P:
        continue
    hk, hq = Hkv // P, Hq // P
    kc, vc = [], []
    for r in range(rot):
        k = torch.empty((B, hk, cap, d), dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        SC.fill_cache(k, SEED + r, S.T_KCACHE, 0, cap, reg, h0=0, Hkv_total=Hkv)
        SC.fill_cache(v, SEED + r, S.T_VCACHE, 0, cap, reg, h0=0, Hkv_total=Hkv)
        kc.append(k)
        vc.append(v)
    qv = torch.empty((B, T, hq, d), dtype=torch.bfloat16, device="cuda")
    qd = torch.empty((B, hq, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_q(qv, SEED, S.T_QVERIFY, hk, reg)
    SC.fill_q(qd, SEED, S.T_QDRAFT, hk, reg)
    kn = torch.zeros((B, T, hk, d), dtype=torch.bfloat16, device="cuda")
    kn1 = kn[:, :1].contiguous()
    kv_v = torch.from_numpy(kvl).cuda()
    kv_d = torch.from_numpy((L0 + 1).astype(np.int32)).cuda()
    ov, lv = torch.empty((B, T, hq, d), device="cuda"), torch.empty((B, T, hq), device="cuda")
    od, ld = torch.empty((B, hq, d), device="cuda"), torch.empty((B, hq), device="cuda")
    wsv = torch.zeros(md.attn_workspace_bytes(B, hq, hk, d, T, int(kvl.max())), dtype=torch.uint8, device="cuda")
    wsd = torch.zeros(md.attn_workspace_bytes(B, hq, hk, d, 1, sink + window), dtype=torch.uint8, device="cuda")
    tv = float(np.median([graph_time_calls(
        lambda r: md.verify_attn_full_append(qv, kc[r % rot], vc[r % rot], kn, kn, kv_v, int(kvl.max()), scale, ov, lv,
                                             wsv), 16, rot) for _ in range(3)]))
    td = float(np.median([graph_time_calls(
        lambda r: md.draft_attn_sparse_append(qd, kc[r % rot], vc[r % rot], kn1, kn1, kv_d, sink, window, scale, od,
                                              ld, wsd, early_kv=True), 64, rot) for _ in range(3)]))
    if P == 1:
        t1 = (tv, td)
    vb = verify_bytes(kvl, hk, hq, d, T)
    db = draft_bytes(L0 + 1, hk, hq, d, sink, window)
    res["P"][P] = {"kv_heads_per_rank": hk, "verify_ms": round(tv, 4), "verify_gbs": round(vb / tv / 1e6, 1),
                   "draft_us": round(td * 1e3, 2), "draft_gbs": round(db / td / 1e6, 1),
                   "E_kernel_verify": round(t1[0] / (P * tv), 4), "E_kernel_draft": round(t1[1] / (P * td), 4),
                   "exchange_bytes_per_verify_call_per_rank": (P - 1) * B * T * hq * d * 4 if P > 1 else 0,
                   "exchange_bytes_per_draft_call_per_rank": (P - 1) * B * hq * d * 4 if P > 1 else 0}
    print(json.dumps({"P": P, **res["P"][P]}), flush=True)
    del kc, vc
    torch.cuda.empty_cache()
print(json.dumps(res))
