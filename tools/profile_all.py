"""One launch of every kernel family of the library at the BASELINE target shape (Llama-3.1-8B
GQA, B=64, ctx 32k, gamma=4) for an ncu sweep: kv_append (T=1, T=5), verify (tcgen05), tree
verify, StreamingLLM draft, SnapKV select + indexed draft, PQ encode (a 4k-row slice) + select,
philox, spec_accept (V=128256), spec_accept_tree, kv_compact, tp_barrier (world 1).
Each call is preceded by a warm-up call so ncu (-s / kernel filters) can take the second.
usage: python tools/profile_all.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402
import synth as S  # noqa: E402
import synth.cuda as SC  # noqa: E402
from bench import CONFIGS, SEED  # noqa: E402

B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS["llama3_b64_32k"]
T = gamma + 1
cap = ctx + 64
dev = "cuda"
reg = S.Regime("peaky", sink=sink)
L0 = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device=dev)
v = torch.empty_like(k)
SC.fill_cache(k, SEED, S.T_KCACHE, 0, cap, reg)
SC.fill_cache(v, SEED, S.T_VCACHE, 0, cap, reg)
qv = torch.empty((B, T, Hq, d), dtype=torch.bfloat16, device=dev)
qd = torch.empty((B, Hq, d), dtype=torch.bfloat16, device=dev)
SC.fill_q(qv, SEED, S.T_QVERIFY, Hkv, reg)
SC.fill_q(qd, SEED, S.T_QDRAFT, Hkv, reg)
kn = torch.empty((B, T, Hkv, d), dtype=torch.bfloat16, device=dev)
SC.fill_new_kv(kn, SEED, S.T_KNEW)
kn1 = kn[:, :1].contiguous()
start = torch.from_numpy(L0.astype(np.int32)).to(dev)
kvv = torch.from_numpy((L0 + T).astype(np.int32)).to(dev)
kvd = torch.from_numpy((L0 + 1).astype(np.int32)).to(dev)
mkl = int(L0.max()) + T
scale = float(np.float32(1 / np.sqrt(d)))
out_v = torch.empty((B, T, Hq, d), device=dev)
lse_v = torch.empty((B, T, Hq), device=dev)
out_d = torch.empty((B, Hq, d), device=dev)
lse_d = torch.empty((B, Hq), device=dev)
ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, cap), dtype=torch.uint8, device=dev)
ws1 = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, cap), dtype=torch.uint8, device=dev)


def twice(fn):
    fn()
    fn()
    torch.cuda.synchronize()


twice(lambda: md.kv_append(k, v, kn1, kn1, start))
twice(lambda: md.kv_append(k, v, kn, kn, start))
twice(lambda: md.verify_attn_full(qv, k, v, kvv, mkl, scale, out_v, lse_v, ws))
chain = torch.tensor([(2 << t) - 1 for t in range(T)], dtype=torch.int64).to(torch.int32)
mask = chain[None, :].repeat(B, 1).to(dev)
twice(lambda: md.verify_attn_tree(qv, k, v, kvv, mkl, mask, scale, out_v, lse_v, ws))
twice(lambda: md.draft_attn_sparse(qd, k, v, kvd, sink, window, scale, out_d, lse_d, ws1))
# SnapKV: selection over the prompt (window 32, budget 2048), then the indexed draft
w, budget = 32, 2048
q_obs = torch.empty((B, w, Hq, d), dtype=torch.bfloat16, device=dev)
SC.fill_q(q_obs, SEED + 1, S.T_QVERIFY, Hkv, reg)
plen = torch.from_numpy(L0.astype(np.int32)).to(dev)
idx = torch.zeros((B, Hkv, budget), dtype=torch.int32, device=dev)
cnt = torch.zeros(B, dtype=torch.int32, device=dev)
sws = torch.empty(md.snapkv_workspace_bytes(B, Hq, Hkv, w, cap), dtype=torch.uint8, device=dev)
twice(lambda: md.snapkv_select(k, v, q_obs, plen, int(L0.max()), w, budget, scale, idx, cnt, sws))
tail = (plen - w).contiguous()
twice(lambda: md.draft_attn_indexed(qd, k, v, kvd, idx, cnt, tail, scale, out_d, lse_d, ws1))
# PQ: codebook from key sub-vectors, encode a 4096-row slice (the full prefill encode is 61 ms), select
pos = torch.from_numpy(S.pq_codebook_positions(SEED, B, Hkv, L0)).to(dev)
bi = torch.arange(B, device=dev)[:, None, None]
ui = torch.arange(Hkv, device=dev)[None, :, None]
cb = torch.empty((B, Hkv, 16, 256, 8), dtype=torch.bfloat16, device=dev)
for m in range(16):
    cb[:, :, m] = k[bi, ui, pos[:, :, m]][..., m * 8:(m + 1) * 8]
codes = torch.zeros((B, Hkv, cap, 16), dtype=torch.uint8, device=dev)
zero = torch.zeros(B, dtype=torch.int32, device=dev)
twice(lambda: md.pq_encode(k, v, cb, zero, 4096, codes))
pidx = torch.zeros((B, Hkv, 512), dtype=torch.int32, device=dev)
pcnt = torch.zeros(B, dtype=torch.int32, device=dev)
ptail = torch.zeros(B, dtype=torch.int32, device=dev)
pws = torch.empty(md.pq_workspace_bytes(B, Hkv, cap), dtype=torch.uint8, device=dev)
twice(lambda: md.pq_select(qd, cb, codes, kvd, cap, sink, 512, 508, pidx, pcnt, ptail, pws))
# acceptance
sigma = S.sigma_for_overlap(SEED, V, alpha)
p_np, q_np, d_np = S.spec_probs(SEED, B, gamma, V, sigma)
p_t, q_t, dtok = torch.from_numpy(p_np).to(dev), torch.from_numpy(q_np).to(dev), torch.from_numpy(d_np).to(dev)
rnd = torch.empty((B, gamma + 2), dtype=torch.int32, device=dev)
twice(lambda: md.philox_u32(SEED, 0, rnd))
out_tok = torch.empty((B, T), dtype=torch.int32, device=dev)
nacc = torch.empty(B, dtype=torch.int32, device=dev)
twice(lambda: md.spec_accept(p_t, q_t, dtok, rnd, out_tok, nacc))
# tree acceptance over a chain-shaped tree of T nodes (p, q per node)
pt = torch.cat([p_t, p_t[:, :1]], 1)[:, :T].contiguous()
qt = torch.cat([q_t, q_t[:, :1]], 1)[:, :T].contiguous()
tok = torch.cat([torch.zeros((B, 1), dtype=torch.int32, device=dev), dtok], 1).contiguous()
par = torch.tensor([-1] + list(range(T - 1)), dtype=torch.int32, device=dev)[None, :].repeat(B, 1).contiguous()
rndt = torch.empty((B, T + 1), dtype=torch.int32, device=dev)
md.philox_u32(SEED, 1, rndt)
accn = torch.empty((B, T), dtype=torch.int32, device=dev)
twice(lambda: md.spec_accept_tree(pt, qt, tok, par, rndt, out_tok, nacc, accn))
nodes = torch.tensor([1, 2, 3, 4], dtype=torch.int32, device=dev)[None, :].repeat(B, 1).contiguous()
ncount = torch.full((B,), 2, dtype=torch.int32, device=dev)
twice(lambda: md.kv_compact(k, v, start, nodes, ncount))
# TP barrier, world 1
flags = torch.zeros(1, dtype=torch.int64, device=dev)
fp = torch.tensor([flags.data_ptr()], dtype=torch.int64, device=dev)
ep = torch.zeros(1, dtype=torch.int64, device=dev)
sync = md.tp_sync(fp, ep, 1, 0)
twice(lambda: md.tp_barrier(sync))
print("profile_all done")
