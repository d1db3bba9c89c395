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


def tp_dp_grid(world: int, Hq: int, Hkv: int, B: int):
    """(tp, dp) for `world` GPUs: KV-head tensor parallelism of the largest degree that divides
    both the world and the KV heads (GQA groups stay whole), batch data parallelism over the
    rest (independent sequences: no collective).  Llama-3.1-8B (8 KV heads) at P = 8: tp8 x dp1;
    Qwen2.5-7B (4 KV heads, 28 q heads) at P = 8: tp4 x dp2 (the paper ran Qwen on 4 GPUs,
    P:1010-1012).  The batch must split evenly over dp."""
    if world < 1 or Hq % Hkv:
        raise ValueError("bad world / heads")
    tp = max(t for t in range(1, world + 1) if world % t == 0 and Hkv % t == 0)
    dp = world // tp
    if B % dp:
        raise ValueError(f"batch {B} does not split over {dp} data-parallel groups")
    return tp, dp


def rank_plan(rank: int, world: int, B: int, Hq: int, Hkv: int) -> dict:
    """This rank's shard of a (tp x dp) grid: rank = dp_rank * tp + tp_rank; KV heads / query
    heads of tp_rank (head_shard) and sequences [b0, b1) of dp_rank."""
    tp, dp = tp_dp_grid(world, Hq, Hkv, B)
    tp_rank, dp_rank = rank % tp, rank // tp
    qs, ks = head_shard(Hq, Hkv, tp_rank, tp)
    bl = B // dp
    return {"tp": tp, "dp": dp, "tp_rank": tp_rank, "dp_rank": dp_rank, "q_heads": qs, "kv_heads": ks,
            "batch": slice(dp_rank * bl, (dp_rank + 1) * bl)}


def tp_groups(tp: int, dp: int):
    """Every rank creates every TP group (torch.distributed requires it); returns this rank's
    group (None when tp == 1: nothing to exchange)."""
    rank = dist.get_rank()
    mine = None
    for d in range(dp):
        ranks = list(range(d * tp, (d + 1) * tp))
        grp = dist.new_group(ranks)
        if rank in ranks:
            mine = grp
    return mine if tp > 1 else None


def gather_rank_major(out_local: torch.Tensor, buf: torch.Tensor, group=None) -> torch.Tensor:
    """The exchange itself: all-gather rank-local outputs into a rank-major [P, ...] buffer
    (one NCCL all_gather_into_tensor; the o_proj input can be consumed rank-major)."""
    world = buf.shape[0]
    flat = buf.view((world * out_local.shape[0],) + tuple(out_local.shape[1:]))
    if dist.get_backend(group) == "gloo" and out_local.is_cuda:  # CPU-staged (single-GPU rank tests)
        parts = [torch.empty(tuple(out_local.shape), dtype=out_local.dtype) for _ in range(world)]
        dist.all_gather(parts, out_local.cpu(), group=group)
        flat.copy_(torch.cat(parts, 0))
        return buf
    dist.all_gather_into_tensor(flat, out_local, group=group)
    return buf


def all_reduce_host(values, op="max", group=None):
    """Reduce a few host scalars over the ranks (timings, flags, token counts): NCCL reduces on
    the device, gloo on the host."""
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(list(values), dtype=torch.float64, device=dev)
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN, "sum": dist.ReduceOp.SUM}[op],
                    group=group)
    return t.cpu().tolist()


def gather_heads(out_local: torch.Tensor, world: int, group=None, buf: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather rank-local outputs [..., Hq/P, d] along the head axis -> [..., Hq, d].

    Uses all_gather_into_tensor into a rank-major [P, ...] buffer, then views it head-major."""
    if world == 1:
        return out_local
    shape = out_local.shape
    if buf is None:
        buf = torch.empty((world,) + tuple(shape), dtype=out_local.dtype, device=out_local.device)
    flat = buf.view((world * shape[0],) + tuple(shape[1:]))      # concatenation along dim 0
    gather_rank_major(out_local.contiguous(), buf, group=group)
    # [P, ..., Hq/P, d] -> [..., P, Hq/P, d] -> [..., Hq, d]
    nd = len(shape)
    perm = list(range(1, nd - 1)) + [0, nd - 1, nd]
    return buf.permute(*perm).reshape(*shape[:-2], world * shape[-2], shape[-1])


class PeerExchange:
    """Fused output exchange: full-head output buffers on every rank,
    peer-mapped with torch symmetric memory (NVLink / NVSwitch), plus the completion flags of
    md_tp_barrier.  Rank r's md_*_tp calls store its heads into every rank's buffer; after
    `barrier()` on a rank's stream its buffer holds all heads (no NCCL all-gather).
    Two buffer sets alternate between consecutive calls (`flip()`), as the header requires: a
    fast peer may already store call i + 1's heads while this rank still reads call i's result.
    Host plumbing only: the stores and the barrier are CUDA kernels of the library."""

    def __init__(self, shape, group=None, nbuf: int = 2):
        import torch.distributed._symmetric_memory as symm_mem

        import paper_2408_11049_b200 as md

        group = group or dist.group.WORLD
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.bufs, self.outs, self.syncs, self._keep = [], [], [], []
        for _ in range(nbuf):
            buf = symm_mem.empty(tuple(shape), dtype=torch.float32, device=dev)
            hb = symm_mem.rendezvous(buf, group.group_name)
            flags = symm_mem.empty((self.world,), dtype=torch.int64, device=dev)
            hf = symm_mem.rendezvous(flags, group.group_name)
            flags.zero_()
            peers = torch.tensor(list(hb.buffer_ptrs), dtype=torch.int64, device=dev)
            flag_peers = torch.tensor(list(hf.buffer_ptrs), dtype=torch.int64, device=dev)
            epoch = torch.zeros(1, dtype=torch.int64, device=dev)
            self._keep += [flags, peers, flag_peers, epoch, hb, hf]
            self.bufs.append(buf)
            self.outs.append(md.tp_out(peers, self.world, self.rank))
            self.syncs.append(md.tp_sync(flag_peers, epoch, self.world, self.rank))
        torch.cuda.synchronize()
        dist.barrier(group)
        self.cur = 0

    @property
    def buf(self):
        return self.bufs[self.cur]

    @property
    def out(self):
        return self.outs[self.cur]

    def barrier(self, stream=None):
        """Publish this call's stores and wait for every peer's (on the stream), then flip to the
        other buffer set for the next call."""
        import paper_2408_11049_b200 as md
        md.tp_barrier(self.syncs[self.cur], stream)
        self.cur = (self.cur + 1) % len(self.bufs)
