"""Indexed-draft ceiling: md_draft_attn_indexed over 2016 listed rows + 32 tail rows with the
list (a) contiguous, (b) runs of 8, (c) uniform random; B=64, 8 KV heads, 32k cache."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa
import synth as S  # noqa
import synth.cuda as SC  # noqa
B, Hq, Hkv, d, ctx = 64, 32, 8, 128, 32768
cap = ctx + 64
k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda"); v = torch.empty_like(k)
SC.fill_cache(k, 1, S.T_KCACHE, 0, cap); SC.fill_cache(v, 1, S.T_VCACHE, 0, cap)
q = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda"); SC.fill_q(q, 1, S.T_QDRAFT, Hkv)
kv = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
out = torch.empty((B, Hq, d), device="cuda")
ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, cap), dtype=torch.uint8, device="cuda")
K = 2016
cnt = torch.full((B,), K, dtype=torch.int32, device="cuda")
tail = torch.full((B,), ctx - 32, dtype=torch.int32, device="cuda")
rng = np.random.default_rng(0)
res = {}
for name in ("contiguous", "runs8", "random"):
    if name == "contiguous":
        idx = np.tile(np.arange(1000, 1000 + K, dtype=np.int32), (B, Hkv, 1))
    elif name == "runs8":
        starts = np.sort(rng.choice((ctx - 64) // 8, size=K // 8, replace=False)) * 8
        idx = np.tile((starts[:, None] + np.arange(8)).reshape(-1).astype(np.int32), (B, Hkv, 1))
    else:
        idx = np.stack([np.sort(rng.choice(ctx - 64, size=K, replace=False)) for _ in range(B * Hkv)]).reshape(B, Hkv, K).astype(np.int32)
    it = torch.from_numpy(np.ascontiguousarray(idx)).cuda()
    f = lambda: md.draft_attn_indexed(q, k, v, kv, it, cnt, tail, 0.088, out, None, ws)
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) / 20 * 1e3
    res[name] = {"us": round(us, 1), "GBs": round(B * Hkv * (K + 32) * d * 4 / us / 1e3, 1)}
print(json.dumps(res))
