"""Time md_snapkv_select (prefill-time SnapKV selection, window 32, budget 2048) at the target shape."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa
import synth as S  # noqa
import synth.cuda as SC  # noqa
from bench import CONFIGS, SEED  # noqa
cfg = sys.argv[1] if len(sys.argv) > 1 else "llama3_b64_32k"
B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[cfg]
cap = ctx + 64
reg = S.Regime("peaky", sink=sink)
L0 = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda"); v = torch.empty_like(k)
SC.fill_cache(k, SEED, S.T_KCACHE, 0, cap, reg)
w, budget = 32, 2048
q_obs = torch.empty((B, w, Hq, d), dtype=torch.bfloat16, device="cuda"); SC.fill_q(q_obs, SEED + 7, S.T_QVERIFY, Hkv, reg)
plen = torch.from_numpy(L0.astype(np.int32)).cuda()
idx = torch.zeros((B, Hkv, budget), dtype=torch.int32, device="cuda"); cnt = torch.zeros(B, dtype=torch.int32, device="cuda")
ws = torch.empty(md.snapkv_workspace_bytes(B, Hq, Hkv, w, int(L0.max())), dtype=torch.uint8, device="cuda")
scale = float(np.float32(1 / np.sqrt(d)))
f = lambda: md.snapkv_select(k, v, q_obs, plen, int(L0.max()), w, budget, scale, idx, cnt, ws)
f(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): f()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
kbytes = int(np.sum(L0)) * Hkv * d * 2
print(json.dumps({"cfg": cfg, "snapkv_select_ms": round(ms, 3), "k_bytes_GB": round(kbytes / 1e9, 2),
                  "two_pass_GBs": round(2 * kbytes / ms / 1e6, 1)}))
