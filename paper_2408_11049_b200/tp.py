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
