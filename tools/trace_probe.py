"""Per-CTA phase timeline of one attention call (md_debug_trace): entry, grid-dependency wait,
range located, first K/V tile landed, last epilogue start, end.  Prints percentiles (us)
relative to the earliest CTA entry.  usage: python tools/trace_probe.py [draft|verify] [window]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402
import synth as S  # noqa: E402
import synth.cuda as SC  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "draft"
window = int(sys.argv[2]) if len(sys.argv) > 2 else 1020
B, Hq, Hkv, d, ctx, T = 64, 32, 8, 128, 32768, 5
cap = ctx + 64
k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda")
v = torch.empty_like(k)
SC.fill_cache(k, 1, S.T_KCACHE, 0, cap)
SC.fill_cache(v, 1, S.T_VCACHE, 0, cap)
scale = float(np.float32(1 / np.sqrt(d)))
trace = torch.zeros((1024, 16), dtype=torch.int64, device="cuda")
if mode == "draft":
    q = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_q(q, 1, S.T_QDRAFT, Hkv)
    kv = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    out = torch.empty((B, Hq, d), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, cap), dtype=torch.uint8, device="cuda")
    call = lambda: md.draft_attn_sparse(q, k, v, kv, 4, window, scale, out, None, ws)
else:
    q = torch.empty((B, T, Hq, d), dtype=torch.bfloat16, device="cuda")
    SC.fill_q(q, 1, S.T_QVERIFY, Hkv)
    kv = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    out = torch.empty((B, T, Hq, d), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, ctx), dtype=torch.uint8, device="cuda")
    call = lambda: md.verify_attn_full(q, k, v, kv, ctx, scale, out, None, ws)
for _ in range(3):
    call()
torch.cuda.synchronize()
md.debug_trace(trace)
call()
torch.cuda.synchronize()
md.debug_trace(None)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    call()
b.record()
torch.cuda.synchronize()
t = trace.cpu().numpy().astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
names = {0: "entry", 1: "after_wait", 2: "range_located", 3: "first_tile", 4: "last_epilogue", 5: "end",
         7: "epi_combined", 8: "epi_stored", 9: "epi_merged", 10: "producer_done"}
res = {"mode": mode, "window": window, "ctas": int(len(t)), "call_us_back_to_back": a.elapsed_time(b) / 20 * 1e3}
res["segments"] = [int(x) for x in np.percentile(t[:, 11], [0, 50, 100])]
for i, nme in names.items():
    if not np.all(t[:, i] > 0):
        continue
    col = rel[:, i]
    res[nme] = [round(float(np.percentile(col, q)), 2) for q in (0, 10, 50, 90, 100)]
res["span_end_minus_entry_p50"] = round(float(np.median(rel[:, 5] - rel[:, 0])), 2)
res["first_tile_minus_located_p50"] = round(float(np.median(rel[:, 3] - rel[:, 2])), 2)
res["tail_last_epilogue_to_end_p50"] = round(float(np.median(rel[:, 5] - rel[:, 4])), 2)
print(json.dumps(res))
raw = trace.cpu().numpy()[: len(t)]
np.save(os.path.join("gpurun_out", f"trace_{mode}_{window}.npy"), raw)
