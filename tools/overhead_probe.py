"""Fixed per-call overhead of the attention kernels: time draft calls whose StreamingLLM
budget shrinks from 1024 to 64 keys (B=64, Llama-3.1 shape) back to back; the intercept of
time vs bytes is the per-call fixed cost."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402
import synth as S  # noqa: E402
import synth.cuda as SC  # noqa: E402

B, Hq, Hkv, d, ctx = 64, 32, 8, 128, 32768
cap = ctx + 64
k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda")
v = torch.empty_like(k)
SC.fill_cache(k, 1, S.T_KCACHE, 0, cap)
SC.fill_cache(v, 1, S.T_VCACHE, 0, cap)
qd = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
SC.fill_q(qd, 1, S.T_QDRAFT, Hkv)
kvd = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
out = torch.empty((B, Hq, d), device="cuda")
ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, cap), dtype=torch.uint8, device="cuda")
scale = float(np.float32(1 / np.sqrt(d)))
res = []
for window in (60, 124, 252, 508, 1020, 2044, 4092):
    f = lambda: md.draft_attn_sparse(qd, k, v, kvd, 4, window, scale, out, None, ws)
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        f()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 50 * 1e3
    mb = B * Hkv * (window + 4) * d * 4 / 1e6
    res.append({"window": window, "MB": round(mb, 1), "us": round(us, 2), "GBs": round(mb / us * 1e3, 1)})
print(json.dumps({"pdl": os.environ.get("MD_PDL", "1"), "probe": res}))
