"""Burst vs sustained: time N back-to-back md_verify_attn_full calls (rotating 4 layer caches)
for N = 4 .. 256 and, for comparison, a plain torch read stream (sum over a 8.6 GB bf16
tensor) the same way, sampling SM clocks / power with nvidia-smi during each run.
usage: python tools/sustain_probe.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402
import synth as S  # noqa: E402
import synth.cuda as SC  # noqa: E402
from bench import CONFIGS, SEED, ClockSampler  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "llama3_b64_32k"
B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[cfg]
T, R = gamma + 1, 4
cap = (ctx + 64 + 7) // 8 * 8
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
SC.fill_q(qv, SEED, S.T_QVERIFY, Hkv, reg)
kvv = torch.from_numpy((L0 + T).astype(np.int32)).cuda()
mkl = int(L0.max()) + T
scale = float(np.float32(1 / np.sqrt(d)))
out_v = torch.empty((B, T, Hq, d), device="cuda")
lse_v = torch.empty((B, T, Hq), device="cuda")
ws_v = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, T, mkl)), dtype=torch.uint8, device="cuda")
vbytes = int(np.sum(L0 + T)) * Hkv * d * 4


def run(fn, n):
    fn(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        a.record()
        for i in range(n):
            fn(i)
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    return {"n": n, "ms": round(ms, 4), "gbs": round(vbytes / ms / 1e6, 1), "clk": clk.summary()}


res = {"cfg": cfg, "verify": [], "torch_sum": []}
for n in (4, 16, 64, 256):
    res["verify"].append(run(lambda i: md.verify_attn_full(qv, kc[i % R], vc[i % R], kvv, mkl, scale, out_v, lse_v,
                                                            ws_v), n))
flat = [torch.cat([kc[r].view(-1)[: vbytes // 4], vc[r].view(-1)[: vbytes // 4]]) for r in range(2)]
acc = torch.empty((), dtype=torch.float32, device="cuda")
for n in (4, 16, 64, 256):
    res["torch_sum"].append(run(lambda i: acc.copy_(flat[i % 2].sum(dtype=torch.float32)), n))
print(json.dumps(res))
