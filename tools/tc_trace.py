"""Wait-cycle breakdown of the tcgen05 verify kernel (md_debug_trace slots 8-15, per CTA):
MMA thread waiting for K/V (full), for S buffers (sempty), for P (pfull); softmax thread 0
waiting for S (sfull), for the previous PV (pempty), its total cycles; producer waiting for
free stages.  usage: python tools/tc_trace.py [config]"""
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
k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda")
v = torch.empty_like(k)
SC.fill_cache(k, 1, S.T_KCACHE, 0, cap)
SC.fill_cache(v, 1, S.T_VCACHE, 0, cap)
q = torch.empty((B, T, Hq, d), dtype=torch.bfloat16, device="cuda")
SC.fill_q(q, 1, S.T_QVERIFY, Hkv)
kv = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
out = torch.empty((B, T, Hq, d), device="cuda")
ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, ctx), dtype=torch.uint8, device="cuda")
scale = float(np.float32(1 / np.sqrt(d)))
trace = torch.zeros((1024, 16), dtype=torch.int64, device="cuda")
call = lambda: md.verify_attn_full(q, k, v, kv, ctx, scale, out, None, ws)
for _ in range(3):
    call()
torch.cuda.synchronize()
md.debug_trace(trace)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
call()
b.record()
torch.cuda.synchronize()
md.debug_trace(None)
t = trace.cpu().numpy().astype(np.float64)
t = t[t[:, 11] > 0]
names = {0: "sm_ld", 1: "sm_scale_need", 2: "sm_vote_rescale", 3: "sm_exp_pack", 4: "sm_pstore", 5: "sm_fence_arrive", 7: "sm_epilogue", 8: "mma_wait_full", 9: "mma_wait_sempty", 10: "mma_wait_pfull", 12: "sm_wait_sfull", 13: "sm_wait_pempty",
         14: "sm_total", 15: "prod_wait_empty"}
res = {"cfg": cfg, "ctas": int(len(t)), "call_us": round(a.elapsed_time(b) * 1e3, 1),
       "tiles_per_cta": float(np.median(t[:, 11]))}
for i, nme in names.items():
    res[nme + "_kcyc_p50"] = round(float(np.median(t[:, i])) / 1e3, 1)
acc_cols = [0, 1, 2, 3, 4, 5, 7, 12, 13]
res["sm_unaccounted_kcyc_p10_p50_p90"] = [round(float(x) / 1e3, 1) for x in
                                          np.percentile(t[:, 14] - t[:, acc_cols].sum(1), [10, 50, 90])]
ends = t[:, 6]
res["finish_spread_us"] = [round(float(x), 1) for x in np.percentile((ends - ends.min()) / 1e3, [0, 10, 50, 90, 100])]
print(json.dumps(res))
