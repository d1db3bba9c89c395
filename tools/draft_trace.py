"""Per-CTA timeline of the StreamingLLM draft call at the target point (B=64, Llama-3.1 GQA,
4 + 1020 keys), rotated over 4 layer caches like bench.py: for several consecutive calls, each
CTA's start (after the grid-dependency wait), first tile, last epilogue, end, SM id and segment
count (md_debug_trace).  Prints the spread of end times and how it splits by segment count and
by SM (is a slow CTA slow because of its SM or because of its work?).
usage: python tools/draft_trace.py"""
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
cap, R = ctx + 64, 4
ks, vs = [], []
for r in range(R):
    k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    SC.fill_cache(k, 1 + r, S.T_KCACHE, 0, cap)
    SC.fill_cache(v, 1 + r, S.T_VCACHE, 0, cap)
    ks.append(k)
    vs.append(v)
q = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
SC.fill_q(q, 1, S.T_QDRAFT, Hkv)
L = S.committed_lengths(7, B, ctx, 4, ragged=True)
kv = torch.from_numpy((L + 1).astype(np.int32)).cuda()
out = torch.empty((B, Hq, d), device="cuda")
ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, 1024), dtype=torch.uint8, device="cuda")
scale = float(np.float32(1 / np.sqrt(d)))
call = lambda i: md.draft_attn_sparse(q, ks[i % R], vs[i % R], kv, 4, 1020, scale, out, None, ws)
if os.environ.get("TRACE_FORM") == "fused_early":  # the form bench.py times: fused append + early KV
    kn = torch.zeros((B, 1, Hkv, d), dtype=torch.bfloat16, device="cuda")
    call = lambda i: md.draft_attn_sparse_append(q, ks[i % R], vs[i % R], kn, kn, kv, 4, 1020, scale, out, None, ws,
                                                 early_kv=True)
for i in range(8):
    call(i)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(40):
    call(i)
b.record()
torch.cuda.synchronize()
res = {"form": os.environ.get("TRACE_FORM", "plain"), "call_us_rotated": round(a.elapsed_time(b) / 40 * 1e3, 2), "calls": []}
ends_by_sm = {}
for c in range(6):
    tr = torch.zeros((1024, 16), dtype=torch.int64, device="cuda")
    md.debug_trace(tr)
    if c % 2 == 1:  # odd calls: traced with a predecessor in flight (its stamps are overwritten)
        call(c + 1)
    call(c)
    torch.cuda.synchronize()
    md.debug_trace(None)
    t = tr.cpu().numpy().astype(np.float64)
    t = t[t[:, 0] > 0]
    t1 = t[:, 1].min()                                # earliest grid-dependency release
    start, first, last_epi, end = (t[:, 1] - t1) / 1e3, (t[:, 3] - t1) / 1e3, (t[:, 4] - t1) / 1e3, (t[:, 5] - t1) / 1e3
    seg = t[:, 11].astype(int)
    sm = t[:, 6].astype(int)
    for s_, e_ in zip(sm, end):
        ends_by_sm.setdefault(int(s_), []).append(float(e_))
    located = (t[:, 2] - t1) / 1e3
    entry = (t[:, 0] - t1) / 1e3
    row = {"ctas": int(len(t)), "start_p50": round(float(np.median(start)), 2),
           "with_predecessor": bool(c % 2 == 1),
           "entry_before_release_p0_p50_p100": [round(float(np.percentile(entry, x)), 2) for x in (0, 50, 100)],
           "range_located_p50_p100": [round(float(np.percentile(located, x)), 2) for x in (50, 100)],
           "first_tile_p0_p50_p100": [round(float(np.percentile(first, x)), 2) for x in (0, 50, 100)],
           "end_p0_p10_p50_p90_p100": [round(float(np.percentile(end, x)), 2) for x in (0, 10, 50, 90, 100)],
           "end_p50_by_segments": {int(s): round(float(np.median(end[seg == s])), 2) for s in np.unique(seg)},
           "ctas_by_segments": {int(s): int((seg == s).sum()) for s in np.unique(seg)},
           "last_epilogue_to_end_p50": round(float(np.median(end - last_epi)), 2),
           "epilogue_phases_p50": {"combine": round(float(np.median(t[:, 7] - t[:, 4])) / 1e3, 2),
                                   "stores": round(float(np.median(t[:, 8] - t[:, 7])) / 1e3, 2),
                                   "to_end": round(float(np.median(t[:, 5] - t[:, 8])) / 1e3, 2)},
           "producer_done_to_end_p50": round(float(np.median(t[:, 5] - t[:, 10])) / 1e3, 2),
           # after the release: first Q loads issued (producer), fused append done / first Q landed (consumer warp 0)
           "q_issued_p50_p90": [round(float(np.percentile((t[:, 14] - t1) / 1e3, x)), 2) for x in (50, 90)] if (t[:, 14] > 0).any() else None,
           "append_done_p50_p90": [round(float(np.percentile((t[:, 12] - t1) / 1e3, x)), 2) for x in (50, 90)] if (t[:, 12] > 0).any() else None,
           "q_landed_p50_p90": [round(float(np.percentile((t[:, 13] - t1) / 1e3, x)), 2) for x in (50, 90)] if (t[:, 13] > 0).any() else None}
    res["calls"].append(row)
# per-SM persistence: correlation of an SM's mean end time between even and odd calls
sms = sorted(ends_by_sm)
ev = np.array([np.mean(ends_by_sm[s][0::2]) for s in sms])
od = np.array([np.mean(ends_by_sm[s][1::2]) for s in sms])
res["sm_end_corr_even_vs_odd_calls"] = round(float(np.corrcoef(ev, od)[0, 1]), 3)
res["sm_mean_end_p0_p50_p100"] = [round(float(np.percentile((ev + od) / 2, x)), 2) for x in (0, 50, 100)]
print(json.dumps(res))
