import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2408_11049_b200 as md
from tests.test_gpu_tp import Ranks, _shard
from tests.helpers import AttnCase
import synth as S
world = 2
mode = sys.argv[1]
r = Ranks(world, (4,))
syncs = [r.sync(k) for k in range(world)]
torch.cuda.synchronize()
if mode == "barrier_only":
    for k in range(world):
        md.tp_barrier(syncs[k], stream=r.streams[k])
    torch.cuda.synchronize()
    print("barrier_only OK", [f.tolist() for f in r.flags])
else:
    B, Hq, Hkv, d, T = 3, 32, 8, 128, 5
    lens = [2500, 1700, 300]
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, T=T, seed=93)
    kvl = torch.from_numpy(case.kv_len).cuda()
    rv = Ranks(world, (B, T, Hq, d))
    shards = [_shard(case, world, k) for k in range(world)]
    ws = [torch.zeros(md.attn_workspace_bytes(B, 16, 4, d, T, max(lens)), dtype=torch.uint8, device="cuda") for _ in range(world)]
    outs = [rv.out(k) for k in range(world)]
    syncs = [rv.sync(k) for k in range(world)]
    torch.cuda.synchronize()
    for k in range(world):
        kk, v, qv, qd, _, _ = shards[k]
        md.verify_attn_full_tp(qv, kk, v, kvl, max(lens), case.scale, outs[k], None, ws[k], stream=rv.streams[k])
        if mode == "verify_barrier":
            md.tp_barrier(syncs[k], stream=rv.streams[k])
    torch.cuda.synchronize()
    print(mode, "OK", [f.tolist() for f in rv.flags], float(torch.isnan(rv.bufs[0]).sum()))
