"""Where does the spec step's time go?  Captures sub-sequences of bench.py's layer pass as
CUDA graphs and times each replay (CUDA events): verify calls alone, verify + their
kv_append, draft calls alone, draft + kv_append, appends alone, the whole pass, and the same
with the appends fused into the attention calls (md_*_append).
usage: python tools/step_probe.py [config]"""
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
qd = torch.empty((B, Hq, d), dtype=torch.bfloat16, device="cuda")
SC.fill_q(qv, SEED, S.T_QVERIFY, Hkv, reg)
SC.fill_q(qd, SEED, S.T_QDRAFT, Hkv, reg)
knew_v = torch.empty((B, T, Hkv, d), dtype=torch.bfloat16, device="cuda")
vnew_v = torch.empty_like(knew_v)
SC.fill_new_kv(knew_v, SEED, S.T_KNEW)
SC.fill_new_kv(vnew_v, SEED, S.T_VNEW)
knew_d, vnew_d = knew_v[:, :1].contiguous(), vnew_v[:, :1].contiguous()
pos = torch.from_numpy(L0[None, :] + np.arange(gamma + 2, dtype=np.int32)[:, None]).cuda()
mkl = int(L0.max()) + T
scale = float(np.float32(1 / np.sqrt(d)))
out_v = torch.empty((B, T, Hq, d), device="cuda")
lse_v = torch.empty((B, T, Hq), device="cuda")
out_d = torch.empty((B, Hq, d), device="cuda")
lse_d = torch.empty((B, Hq), device="cuda")
ws_v = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, T, mkl)), dtype=torch.uint8, device="cuda")
ws_d = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, 1, sink + window)), dtype=torch.uint8, device="cuda")


def verify(l, app):
    if app:
        md.kv_append(kc[l % R], vc[l % R], knew_v, vnew_v, pos[0])
    md.verify_attn_full(qv, kc[l % R], vc[l % R], pos[gamma + 1], mkl, scale, out_v, lse_v, ws_v)


def draft(j, l, app):
    if app:
        md.kv_append(kc[l % R], vc[l % R], knew_d, vnew_d, pos[j])
    md.draft_attn_sparse(qd, kc[l % R], vc[l % R], pos[j + 1], sink, window, scale, out_d, lse_d, ws_d)


def appends():
    for j in range(gamma):
        for l in range(layers):
            md.kv_append(kc[l % R], vc[l % R], knew_d, vnew_d, pos[j])
    for l in range(layers):
        md.kv_append(kc[l % R], vc[l % R], knew_v, vnew_v, pos[0])


def verify_fused(l):
    md.verify_attn_full_append(qv, kc[l % R], vc[l % R], knew_v, vnew_v, pos[gamma + 1], mkl, scale, out_v, lse_v,
                               ws_v)


def draft_fused(j, l):
    md.draft_attn_sparse_append(qd, kc[l % R], vc[l % R], knew_d, vnew_d, pos[j + 1], sink, window, scale, out_d,
                                lse_d, ws_d)


variants = {
    "verify_only": lambda: [verify(l, False) for l in range(layers)],
    "verify_append": lambda: [verify(l, True) for l in range(layers)],
    "draft_only": lambda: [draft(j, l, False) for j in range(gamma) for l in range(layers)],
    "draft_append": lambda: [draft(j, l, True) for j in range(gamma) for l in range(layers)],
    "appends_only": appends,
    "full_pass": lambda: ([draft(j, l, True) for j in range(gamma) for l in range(layers)],
                          [verify(l, True) for l in range(layers)]),
    "verify_fused": lambda: [verify_fused(l) for l in range(layers)],
    "draft_fused": lambda: [draft_fused(j, l) for j in range(gamma) for l in range(layers)],
    "full_pass_fused": lambda: ([draft_fused(j, l) for j in range(gamma) for l in range(layers)],
                                [verify_fused(l) for l in range(layers)]),
}
# PROBE_VARIANTS=a,b PROBE_ROUNDS=k: only those variants, interleaved k times (A/B without drift)
sel = os.environ.get("PROBE_VARIANTS")
rounds = int(os.environ.get("PROBE_ROUNDS", "1"))
order = [n for _ in range(rounds) for n in (sel.split(",") if sel else variants)]
res = {"cfg": cfg}
for k, name in enumerate(order):
    fn = variants[name]
    if rounds > 1:
        name = f"{name}#{k // (len(order) // rounds)}"
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    res[name + "_ms"] = round(a.elapsed_time(b) / 5, 3)
    # the same sequence eagerly (no graph)
    torch.cuda.synchronize()
    a.record()
    for _ in range(3):
        fn()
    b.record()
    torch.cuda.synchronize()
    res[name + "_eager_ms"] = round(a.elapsed_time(b) / 3, 3)
    del g
print(json.dumps(res))
