"""Time the per-step sampling + acceptance of bench.py at the metric point (B=64, gamma=4,
V=128256): 2 x md_philox_u32 + md_spec_accept(gamma=0) on the draft rows q (the drafter's tokens)
+ md_spec_accept on (p, q), CUDA events over back-to-back repetitions (eager and as one graph).
usage: python tools/accept_probe.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_11049_b200 as md  # noqa: E402

B, gamma, V = 64, 4, 128256
g = torch.Generator(device="cuda").manual_seed(1)
z = torch.randn((B, gamma + 1, V), device="cuda", generator=g) * 3
p = torch.softmax(z, -1).float().contiguous()
q = torch.softmax(z[:, :gamma] + 0.5 * torch.randn((B, gamma, V), device="cuda", generator=g), -1).float().contiguous()
dw_full = torch.zeros((B * gamma, 2), dtype=torch.int32, device="cuda")
rnd_full = torch.zeros((B, gamma + 2), dtype=torch.int32, device="cuda")
dw, rnd = dw_full, rnd_full
dtok = torch.zeros((B, gamma), dtype=torch.int32, device="cuda")
dn = torch.zeros(B * gamma, dtype=torch.int32, device="cuda")
out_tok = torch.zeros((B, gamma + 1), dtype=torch.int32, device="cuda")
nacc = torch.zeros(B, dtype=torch.int32, device="cuda")


def step(i):
    md.philox_u32(11, i, dw_full)
    md.philox_u32(12, i, rnd_full)
    md.spec_accept(q.view(B * gamma, 1, V), None, None, dw, dtok.view(B * gamma, 1), dn, mode="sample")
    md.spec_accept(p, q, dtok, rnd, out_tok, nacc, mode="sample")


def timed(fn, n=50):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(n):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


res = {"B": B, "gamma": gamma, "V": V, "sample_and_accept_us": round(timed(step), 1)}
res["accept_only_us"] = round(timed(lambda i: md.spec_accept(p, q, dtok, rnd, out_tok, nacc, mode="sample")), 1)
res["draft_sampling_only_us"] = round(timed(lambda i: md.spec_accept(q.view(B * gamma, 1, V), None, None, dw,
                                                                     dtok.view(B * gamma, 1), dn, mode="sample")), 1)
res["bytes_p_q"] = (p.numel() + q.numel()) * 4
print(json.dumps(res))

# tree acceptance (f3) on a 5-node tree per sequence (root + 2 children + 2 grandchildren under the
# first child), p / q [B, T, V]: a rejection walks sibling residuals, then the final draw
T = 5
pt = torch.softmax(torch.randn((B, T, V), device="cuda", generator=g) * 3, -1).float().contiguous()
qt = torch.softmax(torch.randn((B, T, V), device="cuda", generator=g) * 3, -1).float().contiguous()
tok_t = torch.randint(0, V, (B, T), device="cuda", generator=g, dtype=torch.int64).to(torch.int32)
par_t = torch.tensor([-1, 0, 0, 1, 1], dtype=torch.int32, device="cuda").repeat(B, 1).contiguous()
rnd_t = torch.randint(0, 2 ** 31 - 1, (B, T + 1), device="cuda", generator=g, dtype=torch.int64).to(torch.int32)
out_t = torch.zeros((B, T), dtype=torch.int32, device="cuda")
na_t = torch.zeros(B, dtype=torch.int32, device="cuda")
res2 = {"tree_accept_us": round(timed(lambda i: md.spec_accept_tree(pt, qt, tok_t, par_t, rnd_t, out_t, na_t)), 1),
        "tree_T": T, "tree_tokens_sample": out_t[:2].cpu().tolist()}
print(json.dumps(res2))
