"""Verify-call time for UNIFORM context lengths (every unit the same length, so all CTAs hit
segment boundaries together) vs the ragged lengths of the bench; rotated caches, CUDA events,
no trace.  usage: python tools/uniform_probe.py [config]"""
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

cfg = sys.argv[1] if len(sys.argv) > 1 else "llama3_b64_32k"
B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[cfg]
T = gamma + 1
cap = ctx + 64
R = 3
kc, vc = [], []
for r in range(R):
    k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    SC.fill_cache(k, SEED + r, S.T_KCACHE, 0, cap)
    SC.fill_cache(v, SEED + r, S.T_VCACHE, 0, cap)
    kc.append(k)
    vc.append(v)
q = torch.empty((B, T, Hq, d), dtype=torch.bfloat16, device="cuda")
SC.fill_q(q, SEED, S.T_QVERIFY, Hkv)
out = torch.empty((B, T, Hq, d), device="cuda")
scale = float(np.float32(1 / np.sqrt(d)))
res = {"cfg": cfg}
L0 = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
for name, lens in (("uniform", np.full(B, ctx, np.int32)), ("ragged", (L0 + T).astype(np.int32))):
    kv = torch.from_numpy(lens).cuda()
    mkl = int(lens.max())
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, mkl), dtype=torch.uint8, device="cuda")
    call = lambda i: md.verify_attn_full(q, kc[i % R], vc[i % R], kv, mkl, scale, out, None, ws)
    for i in range(3):
        call(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(12):
        call(i)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 12
    byts = int(lens.sum()) * Hkv * d * 4
    res[name + "_ms"] = round(ms, 4)
    res[name + "_kv_gbs"] = round(byts / ms / 1e6, 1)
print(json.dumps(res))
