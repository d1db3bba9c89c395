"""A/B of draft-call variants (MD_LIB selects the library): the StreamingLLM draft at the target
point (B=64, Llama-3.1 GQA, 4 + 1020 keys) over 4 rotated layer caches, back to back, plus the
fused-append form the bench runs.  usage: MD_LIB=... python tools/draft_ab.py [label]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402
import synth as S  # noqa: E402
import synth.cuda as SC  # noqa: E402
from bench import graph_time_calls  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("MD_LIB", "product")
# AB_CFG: llama3 (default) | qwen | llama2 | llama3_b128
SHAPES = {"llama3": (64, 32, 8, 32768, 1020), "qwen": (64, 28, 4, 100000, 2044), "llama2": (64, 32, 32, 8192, 508),
          "llama3_b128": (128, 32, 8, 32768, 1020)}
cfg = os.environ.get("AB_CFG", "llama3")
B, Hq, Hkv, ctx, window = SHAPES[cfg]
d = 128
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
kn = torch.zeros((B, 1, Hkv, d), dtype=torch.bfloat16, device="cuda")
out = torch.empty((B, Hq, d), device="cuda")
lse = torch.empty((B, Hq), device="cuda")
ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, window + 4), dtype=torch.uint8, device="cuda")
scale = float(np.float32(1 / np.sqrt(d)))
res = {"variant": label, "cfg": cfg}
for name, call in (("plain", lambda i: md.draft_attn_sparse(q, ks[i % R], vs[i % R], kv, 4, window, scale, out, lse, ws)),
                   ("fused", lambda i: md.draft_attn_sparse_append(q, ks[i % R], vs[i % R], kn, kn, kv, 4, window, scale,
                                                                   out, lse, ws)),
                   ("fused_early", lambda i: md.draft_attn_sparse_append(q, ks[i % R], vs[i % R], kn, kn, kv, 4, window,
                                                                         scale, out, lse, ws, early_kv=True))):
    ts = [graph_time_calls(call, 64, R) * 1e3 for _ in range(5)]  # CUDA-graph replays of 64 calls
    res[name + "_us"] = [round(x, 2) for x in ts]
    res[name + "_us_median"] = round(float(np.median(ts)), 2)
by = B * Hkv * (window + 4) * d * 4
res["GBps_plain"] = round(by / res["plain_us_median"] / 1e3, 1)
print(json.dumps(res))
