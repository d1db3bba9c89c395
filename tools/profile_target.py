"""Run a few md_verify_attn_full / md_draft_attn_sparse calls of one bench config (for ncu).

usage: python tools/profile_target.py [config] [n_calls] [fused|plain] [gamma]
("fused": the md_*_append calls, with the new K/V rows written inside the kernel, as bench.py runs them;
gamma: override the config's gamma, e.g. to profile the verify kernel's larger row counts)"""
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
ncalls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
fused = len(sys.argv) > 3 and sys.argv[3] == "fused"
B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[cfg]
if len(sys.argv) > 4:
    gamma = int(sys.argv[4])
T, R = gamma + 1, 2
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
ws_d = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, 1, sink + window)), dtype=torch.uint8, device="cuda")
knv = torch.zeros((B, T, Hkv, d), dtype=torch.bfloat16, device="cuda")
knd = torch.zeros((B, 1, Hkv, d), dtype=torch.bfloat16, device="cuda")
for i in range(ncalls):
    if fused:
        md.verify_attn_full_append(qv, kc[i % R], vc[i % R], knv, knv, kvv, mkl, scale, out_v, lse_v, ws_v)
    else:
        md.verify_attn_full(qv, kc[i % R], vc[i % R], kvv, mkl, scale, out_v, lse_v, ws_v)
for i in range(ncalls):
    if fused:
        md.draft_attn_sparse_append(qd, kc[i % R], vc[i % R], knd, knd, kvd, sink, window, scale, out_d, lse_d, ws_d)
    else:
        md.draft_attn_sparse(qd, kc[i % R], vc[i % R], kvd, sink, window, scale, out_d, lse_d, ws_d)
torch.cuda.synchronize()
print("profile_target done", cfg)
