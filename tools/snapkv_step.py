"""The paper's flagship operating point with SnapKV drafting (Llama-3.1-8B,
prefill 100k, batch 41, gamma 8 / 11, SnapKV drafts; P:1141 footnote: observation window 32,
pooling 5): one attention-only self-speculation step on one B200 through the C ABI.

  prefill (once, not timed):  md_snapkv_select per layer cache -> idx [B, Hkv, budget - w]
  step (timed, one CUDA graph): for j < gamma, for each layer: md_draft_attn_indexed (append fused:
      the listed prompt positions U the tail [L - w, n)); for each layer: md_verify_attn_full_append;
      the drafter's tokens d_j ~ q_j and the acceptance (md_philox_u32_dev + md_spec_accept)

Workload: synthetic (seeded counter-hash KV/Q in the attention-sink regime, Zipf p/q rows at a
target overlap alpha, draft tokens sampled on the device every step), 32 layers cycling over
R = 4 physically distinct layer caches (each 16.8 GB: every call streams from HBM).
The SnapKV budget is not printed for this table ("optimal KV budget"); 2048 is used.
usage: python tools/snapkv_step.py [gamma] [steps] [alpha]     (prints one JSON line)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402
import synth as S  # noqa: E402
import synth.cuda as SC  # noqa: E402
from bench import DRAFT_SEED, SEED, alpha_from_omega, graph_time_calls, overlap_stats, verify_bytes  # noqa: E402

gamma = int(sys.argv[1]) if len(sys.argv) > 1 else 8
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
alpha = float(sys.argv[3]) if len(sys.argv) > 3 else 0.8
B, Hq, Hkv, d, ctx, V, layers, R = 41, 32, 8, 128, 100000, 128256, 32, 4
w, budget, T = 32, 2048, gamma + 1
dev = torch.device("cuda", 0)
md.load_library()
reg = S.Regime("peaky", sink=4)
L0 = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
warm = 2
cap = (ctx + (steps + warm + 2) * T + 64 + 7) // 8 * 8
kc, vc, idx, cnt = [], [], [], []
plen = torch.from_numpy(L0.astype(np.int32)).to(dev)
q_obs = torch.empty((B, w, Hq, d), dtype=torch.bfloat16, device=dev)
SC.fill_q(q_obs, SEED + 7, S.T_QVERIFY, Hkv, reg)
scale = float(np.float32(1 / np.sqrt(d)))
snap_ws = torch.empty(md.snapkv_workspace_bytes(B, Hq, Hkv, w, int(L0.max())), dtype=torch.uint8, device=dev)
for r in range(R):
    k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device=dev)
    v = torch.empty_like(k)
    SC.fill_cache(k, SEED + r, S.T_KCACHE, 0, cap, reg)
    SC.fill_cache(v, SEED + r, S.T_VCACHE, 0, cap, reg)
    ix = torch.zeros((B, Hkv, budget - w), dtype=torch.int32, device=dev)
    cn = torch.zeros(B, dtype=torch.int32, device=dev)
    md.snapkv_select(k, v, q_obs, plen, int(L0.max()), w, budget, scale, ix, cn, snap_ws)
    kc.append(k)
    vc.append(v)
    idx.append(ix)
    cnt.append(cn)
del snap_ws
tail = torch.from_numpy((L0 - w).astype(np.int32)).to(dev)          # Z19: observation window + generated
qv = torch.empty((B, T, Hq, d), dtype=torch.bfloat16, device=dev)
qd = torch.empty((B, Hq, d), dtype=torch.bfloat16, device=dev)
SC.fill_q(qv, SEED, S.T_QVERIFY, Hkv, reg)
SC.fill_q(qd, SEED, S.T_QDRAFT, Hkv, reg)
knew = torch.empty((B, T, Hkv, d), dtype=torch.bfloat16, device=dev)
vnew = torch.empty_like(knew)
SC.fill_new_kv(knew, SEED, S.T_KNEW)
SC.fill_new_kv(vnew, SEED, S.T_VNEW)
knew_d, vnew_d = knew[:, :1].contiguous(), vnew[:, :1].contiguous()
sigma = S.sigma_for_overlap(SEED, V, alpha)
p_np, q_np, _ = S.spec_probs(SEED, B, gamma, V, sigma)
beta, _ = overlap_stats(p_np, q_np)
p_t, q_t = torch.from_numpy(p_np).to(dev), torch.from_numpy(q_np).to(dev)
del p_np, q_np
dtok = torch.empty((B, gamma), dtype=torch.int32, device=dev)
dn = torch.empty(B * gamma, dtype=torch.int32, device=dev)
rnd = torch.empty((B, gamma + 2), dtype=torch.int32, device=dev)
dw = torch.empty((B * gamma, 2), dtype=torch.int32, device=dev)
out_tok = torch.empty((B, T), dtype=torch.int32, device=dev)
nacc = torch.empty(B, dtype=torch.int32, device=dev)
committed = torch.from_numpy(L0.astype(np.int32)).to(dev)
ar = torch.arange(gamma + 2, dtype=torch.int32, device=dev)[:, None]
max_kv = int(L0.max()) + (steps + warm + 2) * T + T
out_v, lse_v = torch.empty((B, T, Hq, d), device=dev), torch.empty((B, T, Hq), device=dev)
out_d, lse_d = torch.empty((B, Hq, d), device=dev), torch.empty((B, Hq), device=dev)
ws_v = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, max_kv), dtype=torch.uint8, device=dev)
ws_d = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, max_kv), dtype=torch.uint8, device=dev)
pos = torch.empty((gamma + 2, B), dtype=torch.int32, device=dev)
step_dev = torch.zeros(1, dtype=torch.int64, device=dev)


def step():
    torch.add(committed[None, :], ar, out=pos)
    for j in range(gamma):
        for l in range(layers):
            md.draft_attn_indexed(qd, kc[l % R], vc[l % R], pos[j + 1], idx[l % R], cnt[l % R], tail, scale, out_d,
                                  lse_d, ws_d, k_new=knew_d, v_new=vnew_d)
    for l in range(layers):
        md.verify_attn_full_append(qv, kc[l % R], vc[l % R], knew, vnew, pos[gamma + 1], max_kv, scale, out_v, lse_v,
                                   ws_v)
    md.philox_u32_dev(DRAFT_SEED, step_dev, dw)
    md.philox_u32_dev(SEED, step_dev, rnd)
    md.spec_accept(q_t.view(B * gamma, 1, V), None, None, dw, dtok.view(B * gamma, 1), dn, mode="sample")
    md.spec_accept(p_t, q_t, dtok, rnd, out_tok, nacc, committed, mode="sample")
    step_dev.add_(1)


for _ in range(warm):
    step()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
with torch.cuda.stream(cs):
    with torch.cuda.graph(g, stream=cs):
        step()
    c0 = committed.clone()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cs)
    for _ in range(steps):
        g.replay()
    b.record(cs)
torch.cuda.synchronize()
ms = a.elapsed_time(b) / steps
tokens = int((committed - c0).sum().item())
kvl = (committed + T).cpu().numpy()
kv_d = (committed + 1).to(torch.int32)
kv_v = torch.from_numpy(kvl.astype(np.int32)).to(dev)
v_ms = graph_time_calls(lambda r: md.verify_attn_full_append(qv, kc[r % R], vc[r % R], knew, vnew, kv_v, max_kv, scale,
                                                             out_v, lse_v, ws_v), 16, R)
d_ms = graph_time_calls(lambda r: md.draft_attn_indexed(qd, kc[r % R], vc[r % R], kv_d, idx[r % R], cnt[r % R], tail,
                                                        scale, out_d, lse_d, ws_d, k_new=knew_d, v_new=vnew_d), 32, R)
listed = cnt[0].cpu().numpy().astype(np.int64)
keys_d = listed + (kv_d.cpu().numpy().astype(np.int64) - tail.cpu().numpy())
db = int(keys_d.sum() * Hkv * d * 4 + B * Hq * d * 6 + B * Hq * 4 + 4 * B * Hkv * d * 2)
vb = verify_bytes(kvl, Hkv, Hq, d, T) + 4 * B * T * Hkv * d * 2
om = tokens / steps / B
print(json.dumps({
    "workload": "paper Table (P:531-545): Llama-3.1-8B GQA 32/8, d=128, prefill 100k, batch 41, SnapKV draft "
                f"(window {w}, pooling 5, budget {budget}), gamma {gamma}, 32 layers (4 rotated 16.8 GB caches)",
    "metric": "spec-step tokens/s (attention-only hot path)", "value": round(tokens / steps / (ms / 1e3), 1),
    "ms_per_step": round(ms, 3), "steps": steps, "tokens_per_step": round(tokens / steps, 1),
    "beta_mean": round(float(beta.mean()), 4), "alpha_implied_by_measured_omega": round(alpha_from_omega(gamma, om), 4),
    "verify_ms": round(v_ms, 4), "verify_gbs": round(vb / v_ms / 1e6, 1), "verify_rows_per_kv_head": 4 * T,
    "draft_indexed_us": round(d_ms * 1e3, 2), "draft_gbs": round(db / d_ms / 1e6, 1),
    "draft_keys_per_unit_mean": round(float(keys_d.mean()), 1),
    "step_share": {"verify": round(layers * v_ms / ms, 3), "draft": round(gamma * layers * d_ms / ms, 3)},
    "timing": "one CUDA graph per step (replayed), CUDA events; per-call times from graph replays of back-to-back calls",
    "data": "synthetic"}), flush=True)
