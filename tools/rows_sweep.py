"""Verify-call time vs query rows per KV head (R = g * (gamma + 1)) at the BASELINE shapes:
Qwen2.5 (g = 7, ctx 100k, B = 64) and Llama-3.1 (g = 4, ctx 32k, B = 64) for several gamma,
CUDA events over rotated layer caches (every call streams its KV from HBM).
usage: python tools/rows_sweep.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402
import synth as S  # noqa: E402
import synth.cuda as SC  # noqa: E402
from bench import SEED, graph_time_calls, verify_bytes  # noqa: E402


def run(name, B, Hq, Hkv, ctx, gammas, rot=2, reps=10):
    d = 128
    cap = ctx + 64
    reg = S.Regime("peaky", sink=4)
    kc, vc = [], []
    for r in range(rot):
        k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        SC.fill_cache(k, SEED + r, S.T_KCACHE, 0, cap, reg)
        SC.fill_cache(v, SEED + r, S.T_VCACHE, 0, cap, reg)
        kc.append(k)
        vc.append(v)
    for gamma in gammas:
        T = gamma + 1
        L0 = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
        kvl = (L0 + T).astype(np.int32)
        kv_t = torch.from_numpy(kvl).cuda()
        q = torch.empty((B, T, Hq, d), dtype=torch.bfloat16, device="cuda")
        SC.fill_q(q, SEED, S.T_QVERIFY, Hkv, reg)
        out = torch.empty((B, T, Hq, d), device="cuda")
        lse = torch.empty((B, T, Hq), device="cuda")
        mkl = int(kvl.max())
        ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, mkl), dtype=torch.uint8, device="cuda")
        call = lambda i: md.verify_attn_full(q, kc[i % rot], vc[i % rot], kv_t, mkl, 1 / np.sqrt(d), out, lse, ws)
        # CUDA-graph replays of 16 back-to-back calls (no host gaps), median of 5
        ms = float(np.median([graph_time_calls(call, 16, rot) for _ in range(5)]))
        by = verify_bytes(kvl, Hkv, Hq, d, T)
        print(json.dumps({"shape": name, "gamma": gamma, "rows": (Hq // Hkv) * T, "ms": round(ms, 4),
                          "GBps": round(by / ms / 1e6, 1)}), flush=True)
    del kc, vc
    torch.cuda.empty_cache()


if __name__ == "__main__":
    md.load_library()
    which = sys.argv[1] if len(sys.argv) > 1 else "baseline"
    if which == "baseline":
        run("qwen_100k", 64, 28, 4, 100000, [4, 5, 6, 7, 10, 15])
        run("llama3_b64_32k", 64, 32, 8, 32768, [4, 11, 15])
    elif which == "llama_gammas":  # every gamma of the Llama-3.1 GQA shape (R = 4 (gamma + 1))
        run("llama3_b64_32k", 64, 32, 8, 32768, list(range(2, 16)))
    elif which == "paper":  # the paper's Llama-3.1-8B SnapKV rows: prefill 100k, bsz 41, gamma 6/7/8/11
        run("llama3_b41_100k", 41, 32, 8, 100000, [6, 7, 8, 11])
