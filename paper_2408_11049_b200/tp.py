"""KV-head tensor parallelism (the paper runs 8-way TP).

Rank r of P owns KV heads [r*Hkv/P, (r+1)*Hkv/P) and the query heads of those GQA
groups, [r*Hq/P, (r+1)*Hq/P), so every md_* attention call runs unchanged on the
local shard (num_kv_heads = Hkv/P).  The only exchange is one all-gather of the
per-head attention outputs after each attention call (the o_proj input needs all
heads); md_spec_accept is replicated (identical inputs -> identical outputs).
Host-side plumbing only: the gather is torch.distributed (NCCL on GPUs, gloo in the
CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def head_shard(Hq: int, Hkv: int, rank: int, world: int):
    """(q_head_slice, kv_head_slice) owned by `rank`; GQA groups never straddle ranks."""
    if Hkv % world:
        raise ValueError(f"{Hkv} KV heads do not split over {world} ranks (use batch sharding)")
    kv_per = Hkv // world
    g = Hq // Hkv
    return slice(rank * kv_per * g, (rank + 1) * kv_per * g), slice(rank * kv_per, (rank + 1) * kv_per)


def gather_rank_major(out_local: torch.Tensor, buf: torch.Tensor, group=None) -> torch.Tensor:
    """The exchange itself: all-gather rank-local outputs into a rank-major [P, ...] buffer
    (one NCCL all_gather_into_tensor; the o_proj input can be consumed rank-major)."""
    world = buf.shape[0]
    flat = buf.view((world * out_local.shape[0],) + tuple(out_local.shape[1:]))
    dist.all_gather_into_tensor(flat, out_local, group=group)
    return buf


def gather_heads(out_local: torch.Tensor, world: int, group=None, buf: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather rank-local outputs [..., Hq/P, d] along the head axis -> [..., Hq, d].

    Uses all_gather_into_tensor into a rank-major [P, ...] buffer, then views it head-major."""
    if world == 1:
        return out_local
    shape = out_local.shape
    if buf is None:
        buf = torch.empty((world,) + tuple(shape), dtype=out_local.dtype, device=out_local.device)
    flat = buf.view((world * shape[0],) + tuple(shape[1:]))      # concatenation along dim 0
    dist.all_gather_into_tensor(flat, out_local.contiguous(), group=group)
    # [P, ..., Hq/P, d] -> [..., P, Hq/P, d] -> [..., Hq, d]
    nd = len(shape)
    perm = list(range(1, nd - 1)) + [0, nd - 1, nd]
    return buf.permute(*perm).reshape(*shape[:-2], world * shape[-2], shape[-1])


class PeerExchange:
    """Fused output exchange: a full-head output buffer on every rank,
    peer-mapped with torch symmetric memory (NVLink / NVSwitch), plus the completion flags of
    md_tp_barrier.  Rank r's md_*_tp calls store its heads into every rank's buffer; after
    `barrier()` on a rank's stream its buffer holds all heads (no NCCL all-gather).
    Host plumbing only: the stores and the barrier are CUDA kernels of the library."""

    def __init__(self, shape, group=None):
        import torch.distributed._symmetric_memory as symm_mem

        import paper_2408_11049_b200 as md

        group = group or dist.group.WORLD
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.buf = symm_mem.empty(tuple(shape), dtype=torch.float32, device=dev)
        hb = symm_mem.rendezvous(self.buf, group.group_name)
        self.flags = symm_mem.empty((self.world,), dtype=torch.int64, device=dev)
        hf = symm_mem.rendezvous(self.flags, group.group_name)
        self.flags.zero_()
        self.peers = torch.tensor(list(hb.buffer_ptrs), dtype=torch.int64, device=dev)
        self.flag_peers = torch.tensor(list(hf.buffer_ptrs), dtype=torch.int64, device=dev)
        self.epoch = torch.zeros(1, dtype=torch.int64, device=dev)
        torch.cuda.synchronize()
        dist.barrier(group)
        self.out = md.tp_out(self.peers, self.world, self.rank)
        self.sync = md.tp_sync(self.flag_peers, self.epoch, self.world, self.rank)

    def barrier(self, stream=None):
        import paper_2408_11049_b200 as md
        md.tp_barrier(self.sync, stream)
