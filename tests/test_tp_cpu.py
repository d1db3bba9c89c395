"""Multi-rank partitioning logic without GPUs (gloo, world_size 2): each rank runs the
oracle on its KV-head shard (paper_2408_11049_b200.tp.head_shard) and the per-head
outputs are all-gathered (tp.gather_heads); the result must equal the unsharded oracle
bit for bit (heads are independent units)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import attention as OA
from paper_2408_11049_b200.tp import gather_heads, head_shard
from tests.helpers import AttnCase


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, Hq, Hkv, d, T = 2, 8, 4, 32, 3
        case = AttnCase(B, Hq, Hkv, d, 90, [90, 41], T=T, seed=3)
        qs, ks = head_shard(Hq, Hkv, rank, world)
        o_loc, _ = OA.verify_attn_full(case.qv_bits[:, :, qs], case.k_bits[:, ks], case.v_bits[:, ks], case.kv_len,
                                       case.scale)
        full_v = gather_heads(torch.from_numpy(o_loc), world).numpy()
        od_loc, _ = OA.draft_attn_sparse(case.qd_bits[:, qs], case.k_bits[:, ks], case.v_bits[:, ks], case.kv_len,
                                         4, 20, case.scale)
        full_d = gather_heads(torch.from_numpy(od_loc), world).numpy()
        if rank == 0:
            ref_v, _ = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
            ref_d, _ = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, 4, 20, case.scale)
            q.put((bool(np.array_equal(full_v, ref_v)), bool(np.array_equal(full_d, ref_d))))
    finally:
        dist.destroy_process_group()


def test_kv_head_tp_gather_equals_unsharded_oracle():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=60)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == (True, True)


def test_head_shard_rejects_non_divisible():
    with pytest.raises(ValueError):
        head_shard(28, 4, 0, 8)
    assert head_shard(32, 8, 3, 4) == (slice(24, 32), slice(6, 8))
