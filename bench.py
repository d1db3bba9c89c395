#!/usr/bin/env python
"""bench.py — MagicDec self-speculative decode hot path on B200 (attention-only spec step).

One STEP = one self-speculation round of the whole hot path over one batch
(T_total = gamma*T_D + T_V):
    for j in 0..gamma-1, for each of the model's layers:  md_draft_attn_sparse_append (kv_append fused)
    the gamma draft tokens: md_philox_u32 + md_spec_accept(gamma = 0) on the draft rows q (the
        drafter's own sampler: d_j ~ q_j, fresh uniforms every step)
    for each layer:                                        md_verify_attn_full_append (kv_append fused)
    md_philox_u32 + md_spec_accept   (committed_len += n + 1 on the device)
Workload (N=1): BASELINE.json's metric point, Llama-3.1-8B-shaped GQA (32 q / 8 kv heads,
d=128, 32 layers), B=64, ctx=32768, gamma=4, StreamingLLM sink 4 + window 1020, V=128256;
synthetic seeded KV/Q (attention-sink regime) and synthetic p/q rows whose overlap
beta = sum_x min(p, q) is set by --alpha (default 0.8, the paper's theory value P:314); the
measured beta, tokens per step and the alpha that Eq.1 implies are reported.
32 layers x 8.6 GB of KV do not fit in 180 GB, so the layers cycle over R=4 physically
distinct 8.6 GB layer caches: every layer-call still streams its full KV from HBM
(R*8.6 GB >> 126 MB L2), in the model's order (a draft step runs through all layers).

metric: spec-step tokens/s (sum over the batch of n_b + 1 emitted tokens / step time),
plus achieved HBM GB/s of verify and draft against the measured copy peak and 8 TB/s.
The number excludes every linear layer by construction: it is NOT comparable to the
paper's end-to-end tokens/s (P:538 etc.).

--gpus N (N > 1): re-launched under torch.distributed.run when WORLD_SIZE is unset; one rank per
GPU on a tp x dp grid: KV-head tensor parallelism of the largest degree dividing
both N and the KV heads, batch data parallelism over the rest (Qwen2.5, 4 KV heads, at N = 8:
tp4 x dp2).  The TP exchange is the fused peer-store epilogue + md_tp_barrier when
it self-tests bit-identical to NCCL, else an NCCL all-gather; DP needs no collective.
--impl reference runs the fp64 CPU oracle (oracle/) on a bounded sample of the same workload
(the oracle is the reference arm for this build); rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha)
    "llama3_b64_32k": (64, 32, 8, 128, 32768, 4, 4, 1020, 128256, 32, 0.8),
    "llama2_8k": (64, 32, 32, 128, 8192, 3, 4, 508, 32000, 32, 0.8),
    "llama3_32k": (128, 32, 8, 128, 32768, 4, 4, 1020, 128256, 32, 0.8),
    "qwen_100k": (64, 28, 4, 128, 100000, 4, 4, 2044, 152064, 28, 0.8),
    "llama3_scaling": (256, 32, 8, 128, 32768, 4, 4, 1020, 128256, 32, 0.8),
    "tiny": (2, 4, 4, 64, 256, 3, 4, 60, 32, 2, 0.8),
}
METRIC = "spec-step tokens/s (attention-only hot path) at B=64, ctx=32k; verify/draft attn HBM GB/s vs 8 TB/s"
SEED = 20240821
DRAFT_SEED = SEED ^ 0x5EED_D4AF7          # Philox key of the drafter's token sampler
NOMINAL_HBM_GBS = 8000.0


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def verify_bytes(kv_len, Hkv, Hq, d, T):
    B = len(kv_len)
    return int(np.sum(kv_len.astype(np.int64)) * Hkv * d * 4 + B * T * Hq * d * (2 + 4) + B * T * Hq * 4)


def draft_bytes(kv_len, Hkv, Hq, d, sink, window):
    keys = np.minimum(kv_len, sink + window).astype(np.int64)
    B = len(kv_len)
    return int(np.sum(keys) * Hkv * d * 4 + B * Hq * d * (2 + 4) + B * Hq * 4)


def append_bytes(B, T, Hkv, d):
    return 2 * B * T * Hkv * d * 2 * 2


def omega_eq1(gamma, alpha):
    """Eq.1: expected tokens per sequence and step."""
    return gamma + 1 if alpha == 1 else (1 - alpha ** (gamma + 1)) / (1 - alpha)


def alpha_from_omega(gamma, om):
    """Invert Eq.1 by bisection (Omega is increasing in alpha)."""
    lo, hi = 0.0, 1.0
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if omega_eq1(gamma, mid) < om:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def overlap_stats(p, q):
    """Per-position overlap beta_bj = sum_x min(p_bj, q_bj) (fp64) and the expected tokens per
    sequence it implies, E[n + 1] = sum_k prod_{i<k} beta_bi (the truncated-geometric law)."""
    beta = np.minimum(p[:, :-1].astype(np.float64), q.astype(np.float64)).sum(-1)     # [B, gamma]
    run = np.cumprod(np.concatenate([np.ones((beta.shape[0], 1)), beta], 1), 1)     # prod_{i<k}, k=0..gamma
    return beta, float(np.mean(run.sum(1)))


def workload_config(name, alpha, world=1):
    """The `config` object both arms print (the workload only: same_config across arms)."""
    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, _ = CONFIGS[name]
    from paper_2408_11049_b200.tp import tp_dp_grid
    tp, dp = tp_dp_grid(world, Hq, Hkv, B)
    kv_gb = B * ctx * Hkv * d * 4 / 1e9
    return {"workload": name, "batch": B, "ctx": ctx, "gamma": gamma, "sink": sink, "window": window,
            "num_q_heads": Hq, "num_kv_heads": Hkv, "head_dim": d, "layers": layers, "vocab": V,
            "target_overlap_alpha": alpha, "attention_only": True,
            "l2": ("inputs larger than L2: each layer-call streams a distinct %.1f GB KV cache" % kv_gb
                   if kv_gb > 0.5 else "correctness-size config: the KV cache fits in L2"),
            "parallelism": f"tp{tp}xdp{dp}" if world > 1 else "single GPU"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index, self.proc, self.rows = index, None, []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=5)
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------------------
# launching N ranks
# ------------------------------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def graph_time_calls(fn, n, rot):
    """Mean device time per call of n back-to-back calls fn(0..n-1) (the caller rotates `rot`
    physically distinct layer caches by the index), as the step runs them: captured in one CUDA
    graph (no host launch gaps; the kernels' programmatic-dependent-launch edges are kept), one
    warm replay, then CUDA events around 3 replays on the capture stream."""
    import torch
    for r in range(rot):
        fn(r)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs):
            for r in range(n):
                fn(r)
        g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cs)
        for _ in range(3):
            g.replay()
        b.record(cs)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (3 * n)


def spawn_ranks(args, argv):
    """`bench.py --gpus N` without a torchrun environment: re-launch this command under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # the communicator init lines go to stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def init_dist(world, local_dev):
    import torch
    import torch.distributed as dist
    if world == 1:
        return None
    # NCCL needs one GPU per rank: more ranks than GPUs (a world-2 run wrapped onto one GPU via
    # LOCAL_RANK) take gloo with CPU-staged exchanges
    wrapped = torch.cuda.is_available() and world > torch.cuda.device_count()
    backend = os.environ.get("MD_DIST_BACKEND", "nccl" if torch.cuda.is_available() and not wrapped else "gloo")
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=local_dev)
    else:
        dist.init_process_group(backend)
    return backend


def run_plan_only(args):
    """--plan-only: the multi-rank plumbing without kernels (CPU, gloo): every rank derives its
    shard of the tp x dp grid, the ranks all-gather their plans and check that the shards tile
    the heads and the batch exactly once; rank 0 prints the plan line."""
    import torch
    import torch.distributed as dist

    from paper_2408_11049_b200.tp import rank_plan, tp_groups
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group(os.environ.get("MD_DIST_BACKEND", "gloo"))
    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[args.config]
    plan = rank_plan(rank, world, B, Hq, Hkv)
    grp = tp_groups(plan["tp"], plan["dp"]) if world > 1 else None
    mine = torch.tensor([plan["tp_rank"], plan["dp_rank"], plan["q_heads"].start, plan["q_heads"].stop,
                         plan["kv_heads"].start, plan["kv_heads"].stop, plan["batch"].start, plan["batch"].stop])
    allp = [torch.zeros_like(mine) for _ in range(world)]
    if world > 1:
        dist.all_gather(allp, mine)
        # the TP group's all-gather of a per-rank tag lands rank-major, as gather_rank_major needs
        tag = torch.tensor([float(rank)])
        got = [torch.zeros(1) for _ in range(plan["tp"])]
        if grp is not None:
            dist.all_gather(got, tag, group=grp)
        tp_ok = [int(x.item()) for x in got] == [plan["dp_rank"] * plan["tp"] + t for t in range(plan["tp"])] \
            if grp is not None else True
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        max_ok = int(t.item()) == world
    else:
        allp, tp_ok, max_ok = [mine], True, True
    cover = np.zeros((B, Hq), np.int32)
    for r in allp:
        r = r.tolist()
        cover[r[6]:r[7], r[2]:r[3]] += 1
    if rank == 0:
        print(json.dumps({"plan_only": True, "n_gpus": world, "tp": plan["tp"], "dp": plan["dp"],
                          "covers_once": bool((cover == 1).all()), "tp_gather_rank_major": bool(tp_ok),
                          "max_over_ranks": bool(max_ok), "config": workload_config(args.config, alpha, world),
                          "shards": [r.tolist() for r in allp]}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------------------------------
# the GPU arm
# ------------------------------------------------------------------------------------------
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2408_11049_b200 as md
    import synth as S
    import synth.cuda as SC
    from paper_2408_11049_b200.tp import all_reduce_host, gather_rank_major, rank_plan, tp_groups

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one process per GPU; LOCAL_RANK wraps only when testing several ranks on fewer GPUs
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = init_dist(world, dev)
    md.load_library()

    B, Hq_full, Hkv_full, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[args.config]
    if args.alpha is not None:
        alpha = args.alpha
    if args.layers:
        layers = args.layers
    T = gamma + 1
    plan = rank_plan(rank, world, B, Hq_full, Hkv_full)
    tp, dp = plan["tp"], plan["dp"]
    tp_group = tp_groups(tp, dp) if world > 1 else None
    qsl, kvsl, bsl = plan["q_heads"], plan["kv_heads"], plan["batch"]
    Hq, Hkv, Bl = qsl.stop - qsl.start, kvsl.stop - kvsl.start, bsl.stop - bsl.start
    steps_total = args.warmup + args.steps + 2
    cap = (ctx + steps_total * T + 16 + 7) // 8 * 8
    R = args.rot
    reg = S.Regime("peaky", sink=sink)

    # ---- inputs resident in HBM: this rank's (sequences, KV heads) slice of the full workload,
    # generated from global coordinates, so every shard holds exactly the single-GPU values
    L0_full = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
    L0 = L0_full[bsl]
    kc, vc = [], []
    for r in range(R):
        k = torch.empty((Bl, Hkv, cap, d), dtype=torch.bfloat16, device=dev)
        v = torch.empty_like(k)
        SC.fill_cache(k, SEED + r, S.T_KCACHE, 0, cap, reg, b0=bsl.start, h0=kvsl.start, Hkv_total=Hkv_full)
        SC.fill_cache(v, SEED + r, S.T_VCACHE, 0, cap, reg, b0=bsl.start, h0=kvsl.start, Hkv_total=Hkv_full)
        kc.append(k)
        vc.append(v)
    qv_full = torch.empty((B, T, Hq_full, d), dtype=torch.bfloat16, device=dev)
    qd_full = torch.empty((B, Hq_full, d), dtype=torch.bfloat16, device=dev)
    SC.fill_q(qv_full, SEED, S.T_QVERIFY, Hkv_full, reg)
    SC.fill_q(qd_full, SEED, S.T_QDRAFT, Hkv_full, reg)
    qv = qv_full[bsl][:, :, qsl].contiguous()
    qd = qd_full[bsl][:, qsl].contiguous()
    knew_full = torch.empty((B, T, Hkv_full, d), dtype=torch.bfloat16, device=dev)
    vnew_full = torch.empty_like(knew_full)
    SC.fill_new_kv(knew_full, SEED, S.T_KNEW)
    SC.fill_new_kv(vnew_full, SEED, S.T_VNEW)
    knew_v = knew_full[bsl][:, :, kvsl].contiguous()
    vnew_v = vnew_full[bsl][:, :, kvsl].contiguous()
    knew_d, vnew_d = knew_v[:, :1].contiguous(), vnew_v[:, :1].contiguous()
    del qv_full, qd_full, knew_full, vnew_full

    # ---- the acceptance inputs: target / draft rows p, q (what the model's LM head would hand
    # md_spec_accept); the draft TOKENS are sampled from q on the device at every step
    sigma = S.sigma_for_overlap(SEED, V, alpha)
    p_np, q_np, _ = S.spec_probs(SEED, B, gamma, V, sigma)
    beta, omega_beta = overlap_stats(p_np, q_np)
    p_t = torch.from_numpy(p_np[bsl]).to(dev)
    q_t = torch.from_numpy(q_np[bsl]).to(dev)
    del p_np, q_np
    dtok = torch.empty((Bl, gamma), dtype=torch.int32, device=dev)
    dn = torch.empty(Bl * gamma, dtype=torch.int32, device=dev)
    rnd_full = torch.empty((B, gamma + 2), dtype=torch.int32, device=dev)      # Philox of the whole batch:
    dw_full = torch.empty((B * gamma, 2), dtype=torch.int32, device=dev)        # a shard reads its rows
    rnd, dw = rnd_full[bsl], dw_full[bsl.start * gamma:bsl.stop * gamma]
    out_tok = torch.empty((Bl, T), dtype=torch.int32, device=dev)
    nacc = torch.empty(Bl, dtype=torch.int32, device=dev)
    committed = torch.from_numpy(L0.copy()).to(dev)
    ar = torch.arange(gamma + 2, dtype=torch.int32, device=dev)[:, None]

    scale = float(np.float32(1.0 / np.sqrt(d)))
    max_kv = int(L0_full.max()) + steps_total * T + T
    assert max_kv <= cap
    out_v = torch.empty((Bl, T, Hq, d), device=dev)
    lse_v = torch.empty((Bl, T, Hq), device=dev)
    out_d = torch.empty((Bl, Hq, d), device=dev)
    lse_d = torch.empty((Bl, Hq), device=dev)
    ws_v = torch.zeros(max(1, md.attn_workspace_bytes(Bl, Hq, Hkv, d, T, max_kv)), dtype=torch.uint8, device=dev)
    ws_d = torch.zeros(max(1, md.attn_workspace_bytes(Bl, Hq, Hkv, d, 1, min(sink + window, cap))),
                       dtype=torch.uint8, device=dev)
    gath_v = torch.empty((tp, Bl, T, Hq, d), device=dev) if tp > 1 else None
    gath_d = torch.empty((tp, Bl, Hq, d), device=dev) if tp > 1 else None
    # f1: the fused exchange (peer stores + md_tp_barrier) replaces the all-gather when the peer
    # buffers can be mapped and a self-test call agrees bit for bit with the NCCL all-gather of
    # the plain call; otherwise (or with --tp-exchange nccl) the NCCL all-gather is used
    xv = xd = None
    exchange = backend if tp > 1 else "none"     # an all-gather on the process group's backend
    if tp > 1 and args.tp_exchange in ("p2p", "auto"):
        ok = 1
        try:
            from paper_2408_11049_b200.tp import PeerExchange, gather_heads
            xv = PeerExchange((Bl, T, Hq * tp, d), group=tp_group)
            xd = PeerExchange((Bl, Hq * tp, d), group=tp_group)
            kv_t = torch.from_numpy((L0 + 1).astype(np.int32)).to(dev)
            buf = xd.buf
            md.draft_attn_sparse_tp(qd, kc[0], vc[0], kv_t, sink, window, scale, xd.out, None, ws_d)
            xd.barrier()
            md.draft_attn_sparse(qd, kc[0], vc[0], kv_t, sink, window, scale, out_d, None, ws_d)
            ref = gather_heads(out_d, tp, group=tp_group)
            torch.cuda.synchronize()
            ok = int(torch.equal(buf, ref))
        except Exception as e:  # noqa: BLE001 - any failure selects the NCCL path
            print(f"rank {rank}: fused exchange unavailable ({type(e).__name__}: {e}); using the {backend} all-gather",
                  file=sys.stderr, flush=True)
            ok = 0
        if all_reduce_host([ok], "min")[0] == 1:
            exchange = "p2p"
        else:
            xv = xd = None

    # a1 fused into a2/a3 (md_*_append): one launch per layer-call instead of append + attention
    fused = not args.no_fused_append

    def layer_pass(pos):
        # pos[j] = committed + j  (rows: draft j start = pos[j], draft j kv_len = pos[j+1],
        #                          verify start = pos[0], verify kv_len = pos[gamma+1])
        for j in range(gamma):
            for l in range(layers):
                kb, vb = kc[l % R], vc[l % R]
                kn_, vn_ = (knew_d, vnew_d) if fused else (None, None)
                if not fused:
                    md.kv_append(kb, vb, knew_d, vnew_d, pos[j])
                if xd is not None:
                    md.draft_attn_sparse_tp(qd, kb, vb, pos[j + 1], sink, window, scale, xd.out, lse_d, ws_d,
                                            k_new=kn_, v_new=vn_)
                    xd.barrier()
                    continue
                if fused:  # MD_ATTN_EARLY_KV: pos is written by torch.add (an ordinary kernel) before the
                    # first call and the previous call appends into another layer's cache (header contract)
                    md.draft_attn_sparse_append(qd, kb, vb, knew_d, vnew_d, pos[j + 1], sink, window, scale, out_d,
                                                lse_d, ws_d, early_kv=True)
                else:
                    md.draft_attn_sparse(qd, kb, vb, pos[j + 1], sink, window, scale, out_d, lse_d, ws_d)
                if tp > 1:
                    gather_rank_major(out_d, gath_d, group=tp_group)
        for l in range(layers):
            kb, vb = kc[l % R], vc[l % R]
            kn_, vn_ = (knew_v, vnew_v) if fused else (None, None)
            if not fused:
                md.kv_append(kb, vb, knew_v, vnew_v, pos[0])
            if xv is not None:
                md.verify_attn_full_tp(qv, kb, vb, pos[gamma + 1], max_kv, scale, xv.out, lse_v, ws_v,
                                       k_new=kn_, v_new=vn_)
                xv.barrier()
                continue
            if fused:
                md.verify_attn_full_append(qv, kb, vb, knew_v, vnew_v, pos[gamma + 1], max_kv, scale, out_v, lse_v,
                                           ws_v)
            else:
                md.verify_attn_full(qv, kb, vb, pos[gamma + 1], max_kv, scale, out_v, lse_v, ws_v)
            if tp > 1:
                gather_rank_major(out_v, gath_v, group=tp_group)

    def sample_and_accept(step_i=None, step_dev=None):
        # the drafter's tokens d_j ~ q_j (md_spec_accept with gamma = 0 samples from its p rows), then
        # the acceptance of those drafts against p; fresh Philox words for both at every step
        if step_dev is None:
            md.philox_u32(DRAFT_SEED, step_i, dw_full)
            md.philox_u32(SEED, step_i, rnd_full)
        else:
            md.philox_u32_dev(DRAFT_SEED, step_dev, dw_full)
            md.philox_u32_dev(SEED, step_dev, rnd_full)
        md.spec_accept(q_t.view(Bl * gamma, 1, V), None, None, dw, dtok.view(Bl * gamma, 1), dn, mode="sample")
        md.spec_accept(p_t, q_t, dtok, rnd, out_tok, nacc, committed, mode="sample")

    # per layer-call: one attention kernel (append fused); + 2 philox + 2 accept per step
    launches_per_step = gamma * layers + layers + 4
    if not fused:
        launches_per_step += gamma * layers + layers
    if tp > 1:
        launches_per_step += gamma * layers + layers  # the exchange after every attention call

    pos_buf = torch.empty((gamma + 2, Bl), dtype=torch.int32, device=dev)
    use_graph = not args.no_graph and (tp == 1 or exchange == "p2p")  # NCCL calls stay eager
    graph = None
    step_dev = torch.zeros(1, dtype=torch.int64, device=dev)

    def layer_step():
        torch.add(committed[None, :], ar, out=pos_buf)
        layer_pass(pos_buf)

    if use_graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        c_save = committed.clone()
        with torch.cuda.stream(s):
            layer_step()  # warm-up outside the capture (kernel attributes, allocator)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        committed.copy_(c_save)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            layer_step()
        torch.cuda.synchronize()
        committed.copy_(c_save)

    def step_g(i):
        # the layer loop (gamma x layers draft calls + layers verify calls) replays as one CUDA
        # graph; draft-token sampling and acceptance follow it
        if graph is not None:
            graph.replay()
        else:
            layer_step()
        sample_and_accept(step_i=i)

    for i in range(args.warmup):
        step_g(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    c0 = committed.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record()
        marks = []
        for i in range(args.steps):
            step_g(args.warmup + i)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            marks.append(ev)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    per_step = np.diff([0.0] + [e0.elapsed_time(ev) for ev in marks])
    tok_local = int((committed - c0).sum().item())
    if world > 1:
        ms = all_reduce_host([ms], "max")[0]
        # each dp group's tokens are counted by its tp ranks alike: sum over ranks / tp
        tokens = int(round(all_reduce_host([tok_local], "sum")[0])) // tp
        dist.barrier()
    else:
        tokens = tok_local
    ms_per_step = ms / args.steps
    value = tokens / (ms / 1e3)
    omega_meas = tokens / args.steps / B

    # ---- per-kernel roofline: verify and draft calls timed alone with CUDA events on the launch stream
    kvl_now = (committed + T).cpu().numpy()
    kv_len_v = torch.from_numpy(kvl_now.astype(np.int32)).to(dev)
    kv_len_d = torch.from_numpy((committed + 1).cpu().numpy().astype(np.int32)).to(dev)
    nrep = max(8 * R, 32)

    def time_calls(fn):
        return graph_time_calls(fn, nrep, R)

    # the kernels the step runs: with the fused append, the *_append calls (their algorithmic
    # bytes add the new rows read from k_new / v_new and written to the cache: 4 B*T*Hkv*d*2)
    if fused:
        v_ms = time_calls(lambda r: md.verify_attn_full_append(qv, kc[r % R], vc[r % R], knew_v, vnew_v, kv_len_v,
                                                               max_kv, scale, out_v, lse_v, ws_v))
        d_ms = time_calls(lambda r: md.draft_attn_sparse_append(qd, kc[r % R], vc[r % R], knew_d, vnew_d, kv_len_d,
                                                                sink, window, scale, out_d, lse_d, ws_d, early_kv=True))
    else:
        v_ms = time_calls(lambda r: md.verify_attn_full(qv, kc[r % R], vc[r % R], kv_len_v, max_kv, scale, out_v,
                                                        lse_v, ws_v))
        d_ms = time_calls(lambda r: md.draft_attn_sparse(qd, kc[r % R], vc[r % R], kv_len_d, sink, window, scale,
                                                         out_d, lse_d, ws_d))
    vb = verify_bytes(kvl_now, Hkv, Hq, d, T) + (4 * Bl * T * Hkv * d * 2 if fused else 0)
    db = draft_bytes(kvl_now - T + 1, Hkv, Hq, d, sink, window) + (4 * Bl * Hkv * d * 2 if fused else 0)
    v_gbs, d_gbs = vb / v_ms / 1e6, db / d_ms / 1e6
    peak, peak_kind = load_peaks()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath) and world == 1:
        traffic = json.load(open(tpath)).get(args.config, {}).get("verify_dram_bytes_per_launch")
    per_rank = None
    if world > 1:
        tv = all_reduce_host([v_ms, d_ms], "max")
        per_rank = {"verify_ms_max_over_ranks": round(tv[0], 4), "draft_ms_max_over_ranks": round(tv[1], 4)}

    # ---- scaling efficiency of the sharded calls: rank 0 also times ONE unsharded call of the
    # full problem on its own GPU (T(1)); E = T(1) / (P * T(P)) with T(P) the slowest rank's call
    eff = None
    if world > 1 and not args.skip_efficiency:
        eff = efficiency_check(args, md, S, SC, torch, dist, dev, rank, world, per_rank, reg, cap, max_kv, L0_full)

    # ---- AR context: one autoregressive step (T=1 decode) over the same caches, attention only
    ar_ms = None
    if world == 1 and not args.skip_ar:
        out_a = torch.empty((Bl, 1, Hq, d), device=dev)
        lse_a = torch.empty((Bl, 1, Hq), device=dev)
        ws_a = torch.zeros(max(1, md.attn_workspace_bytes(Bl, Hq, Hkv, d, 1, max_kv)), dtype=torch.uint8, device=dev)
        qa = qv[:, :1].contiguous()
        ar_ms = time_calls(lambda r: md.verify_attn_full(qa, kc[r % R], vc[r % R], kv_len_d, max_kv, scale, out_a,
                                                         lse_a, ws_a)) * layers

    # ---- e2e: the same step with every input copied from pinned host memory and the result read back
    e2e = None
    if not args.skip_e2e:
        e2e = e2e_measure(args, md, torch, dist, dev, world, tp, tp_group, gamma, layers, R, kc, vc, qd, qv, knew_d,
                          vnew_d, knew_v, vnew_v, p_t, q_t, dtok, dn, dw, dw_full, rnd, rnd_full, out_tok, nacc,
                          committed, ar, pos_buf, sink, window, scale, max_kv, out_d, lse_d, out_v, lse_v, ws_d,
                          ws_v, gath_d, gath_v, fused, Bl, V)

    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.skip_cpu:
            cpu = cpu_baseline(args.config, tokens / args.steps, args.cpu_seconds)
        cfg = workload_config(args.config, alpha, world)
        result = {
            "metric": METRIC,
            "value": round(value, 2),
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4),
            "ms_per_step_p10_p50_p90": [round(float(np.percentile(per_step, q)), 3) for q in (10, 50, 90)],
            "higher_is_better": True,
            "scaling": "strong",  # the workload's batch is split over the N GPUs (KV-head TP x batch DP)
            "vs_baseline": None,
            "dtype": "bf16",
            "data": ("synthetic (seeded counter-hash KV/Q, attention-sink regime; Zipf p/q rows with measured "
                     "overlap beta = %.3f, draft tokens sampled from q on the device every step: measured "
                     "%.3f tokens per sequence and step = Eq.1 at alpha %.3f)" %
                     (float(beta.mean()), omega_meas, alpha_from_omega(gamma, omega_meas))),
            "config": cfg,
            "acceptance": {"target_alpha": alpha, "sigma": round(sigma, 5), "beta_mean": round(float(beta.mean()), 4),
                           "beta_min": round(float(beta.min()), 4), "beta_max": round(float(beta.max()), 4),
                           "omega_measured": round(omega_meas, 4), "omega_expected_from_beta": round(omega_beta, 4),
                           "omega_eq1_at_target_alpha": round(omega_eq1(gamma, alpha), 4),
                           "alpha_implied_by_measured_omega": round(alpha_from_omega(gamma, omega_meas), 4)},
            "impl_details": {"cuda_graph": "layer loop" if use_graph else False,
                             "kv_append": "fused into the attention calls" if fused else "separate launches",
                             "layer_caches_rotated": R,
                             "exchange": (f"tp{tp} KV-head shards, {exchange} exchange; dp{dp} batch shards, "
                                          "no collective") if world > 1 else "none",
                             "dist_backend": backend},
            "tokens_per_step": round(tokens / args.steps, 3),
            "gpu_launches": launches_per_step * args.steps,
            "roofline": {"bound": "hbm", "achieved": round(v_gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(v_gbs / peak, 4), "traffic": traffic,
                         "kernel": ("md_verify_attn_full_append" if fused else "md_verify_attn_full")
                         + ((" (attn_tc_kernel: tcgen05 MMAs with TMEM accumulators, stream-K persistent, fused split merge"
                             if d == 128 and (Hq // Hkv) * T > 8 else
                             " (attn_keys_kernel: mma.sync swap-AB, stream-K persistent with dynamic tail, fused split merge")
                            + (", fused kv_append)" if fused else ")")),
                         "algorithmic_bytes_per_launch": vb, "ms_per_launch": round(v_ms, 4),
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}; a copy: read + write)"},
            "verify_gbs": round(v_gbs, 1),
            "verify_frac_of_8tbs": round(v_gbs / NOMINAL_HBM_GBS, 4),
            "draft_gbs": round(d_gbs, 1),
            "draft_frac_of_8tbs": round(d_gbs / NOMINAL_HBM_GBS, 4),
            "draft_frac_of_measured": round(d_gbs / peak, 4),
            "draft_ms_per_launch": round(d_ms, 4),
            "draft_bytes_per_launch": db,
            "per_rank": per_rank,
            "scaling_efficiency": eff,
            "ar_attention_ms_per_token_step": None if ar_ms is None else round(ar_ms, 3),
            "ar_tokens_per_s": None if ar_ms is None else round(B / (ar_ms / 1e3), 1),
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


def efficiency_check(args, md, S, SC, torch, dist, dev, rank, world, per_rank, reg, cap, max_kv, L0_full):
    """Rank 0 times the UNSHARDED verify and draft calls of the full problem on its own GPU
    (T(1), two rotated full-size layer caches); E(P) = T(1) / (P * T(P)), T(P) the slowest rank's
    sharded call."""
    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, _ = CONFIGS[args.config]
    T = gamma + 1
    res = None
    if rank == 0:
        kc, vc = [], []
        for r in range(2):
            k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device=dev)
            v = torch.empty_like(k)
            SC.fill_cache(k, SEED + r, S.T_KCACHE, 0, cap, reg)
            SC.fill_cache(v, SEED + r, S.T_VCACHE, 0, cap, reg)
            kc.append(k)
            vc.append(v)
        qv = torch.empty((B, T, Hq, d), dtype=torch.bfloat16, device=dev)
        qd = torch.empty((B, Hq, d), dtype=torch.bfloat16, device=dev)
        SC.fill_q(qv, SEED, S.T_QVERIFY, Hkv, reg)
        SC.fill_q(qd, SEED, S.T_QDRAFT, Hkv, reg)
        kvl = (L0_full + T).astype(np.int32)
        kv_v = torch.from_numpy(kvl).to(dev)
        kv_d = torch.from_numpy((L0_full + 1).astype(np.int32)).to(dev)
        scale = float(np.float32(1.0 / np.sqrt(d)))
        ov = torch.empty((B, T, Hq, d), device=dev)
        od = torch.empty((B, Hq, d), device=dev)
        ws_v = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, max_kv), dtype=torch.uint8, device=dev)
        ws_d = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, 1, sink + window), dtype=torch.uint8, device=dev)

        def tcall(fn):
            return graph_time_calls(fn, 16, 2)

        t1v = tcall(lambda i: md.verify_attn_full(qv, kc[i % 2], vc[i % 2], kv_v, max_kv, scale, ov, None, ws_v))
        t1d = tcall(lambda i: md.draft_attn_sparse(qd, kc[i % 2], vc[i % 2], kv_d, sink, window, scale, od, None,
                                                   ws_d))
        tpv, tpd = per_rank["verify_ms_max_over_ranks"], per_rank["draft_ms_max_over_ranks"]
        res = {"verify_ms_1gpu_unsharded": round(t1v, 4), "draft_ms_1gpu_unsharded": round(t1d, 4),
               "verify_ms_sharded_max_over_ranks": tpv, "draft_ms_sharded_max_over_ranks": tpd,
               "E_verify": round(t1v / (world * tpv), 4), "E_draft": round(t1d / (world * tpd), 4),
               "note": "E(P) = T(1) / (P T(P)) per attention call, same box; T(1) on rank 0's GPU"}
        del kc, vc
        torch.cuda.empty_cache()
    dist.barrier()
    return res


def e2e_measure(args, md, torch, dist, dev, world, tp, tp_group, gamma, layers, R, kc, vc, qd, qv, knew_d, vnew_d,
                knew_v, vnew_v, p_t, q_t, dtok, dn, dw, dw_full, rnd, rnd_full, out_tok, nacc, committed, ar,
                pos_buf, sink, window, scale, max_kv, out_d, lse_d, out_v, lse_v, ws_d, ws_v, gath_d, gath_v, fused,
                Bl, V):
    """The same step through the public API with every input copied from pinned host memory:
    per call its Q and new K/V rows, per step p / q, and the emitted tokens read back."""
    from paper_2408_11049_b200.tp import gather_rank_major
    h_qd, h_qv = qd.cpu().pin_memory(), qv.cpu().pin_memory()
    h_kd, h_vd = knew_d.cpu().pin_memory(), vnew_d.cpu().pin_memory()
    h_kv, h_vv = knew_v.cpu().pin_memory(), vnew_v.cpu().pin_memory()
    h_p, h_q = p_t.cpu().pin_memory(), q_t.cpu().pin_memory()
    h_out = torch.empty(tuple(out_tok.shape), dtype=torch.int32).pin_memory()
    h_n = torch.empty(tuple(nacc.shape), dtype=torch.int32).pin_memory()
    h2d = (gamma * layers * (h_qd.nbytes + h_kd.nbytes + h_vd.nbytes) +
           layers * (h_qv.nbytes + h_kv.nbytes + h_vv.nbytes) + h_p.nbytes + h_q.nbytes)
    d2h = h_out.nbytes + h_n.nbytes
    T = gamma + 1
    # Every call has its own device staging slot, and all of a step's H2D copies are issued up
    # front on their own stream, in call order; the compute stream waits only at a few group
    # boundaries (calls [0,1), [1,8), [8,32), then every 32), so the copy engine runs ahead
    # while consecutive kernels keep their programmatic-dependent-launch overlap.  p / q ride
    # behind the verify inputs and are waited for only by the acceptance.
    copy_s = torch.cuda.Stream()
    ncalls = gamma * layers + layers
    nd = gamma * layers
    st = [(torch.empty_like(qd), torch.empty_like(knew_d), torch.empty_like(vnew_d)) if c < nd else
          (torch.empty_like(qv), torch.empty_like(knew_v), torch.empty_like(vnew_v)) for c in range(ncalls)]
    bounds_c = sorted({0, 1, 8, 32} | set(range(32, ncalls, 32)) | {ncalls})
    bounds_c = [b for b in bounds_c if b <= ncalls]
    group_of = {}
    for gi in range(len(bounds_c) - 1):
        for c in range(bounds_c[gi], bounds_c[gi + 1]):
            group_of[c] = gi
    ready = [torch.cuda.Event() for _ in range(len(bounds_c) - 1)]
    pq_ready, step_done = torch.cuda.Event(), torch.cuda.Event()
    state = {"in_graph": False}
    step_dev = torch.zeros(1, dtype=torch.int64, device=dev)

    def issue_copies(cur):
        with torch.cuda.stream(copy_s):
            if state["in_graph"]:  # fork the copy stream from the capturing stream
                fork = torch.cuda.Event()
                fork.record(cur)
                copy_s.wait_event(fork)
            else:  # eager: the previous step's calls and acceptance are done with the slots / p, q
                copy_s.wait_event(step_done)
            for c in range(ncalls):
                src = (h_qd, h_kd, h_vd) if c < nd else (h_qv, h_kv, h_vv)
                for x, y in zip(st[c], src):
                    x.copy_(y, non_blocking=True)
                if c + 1 in bounds_c:
                    ready[group_of[c]].record(copy_s)
            p_t.copy_(h_p, non_blocking=True)
            q_t.copy_(h_q, non_blocking=True)
            pq_ready.record(copy_s)

    def e2e_step(i):
        cur = torch.cuda.current_stream()
        issue_copies(cur)
        torch.add(committed[None, :], ar, out=pos_buf)
        for c in range(ncalls):
            if c in bounds_c:
                cur.wait_event(ready[group_of[c]])
            l = c % layers
            kb, vb_ = kc[l % R], vc[l % R]
            q_, k_, v_ = st[c]
            if c < nd:
                j = c // layers
                if fused:
                    md.draft_attn_sparse_append(q_, kb, vb_, k_, v_, pos_buf[j + 1], sink, window, scale, out_d,
                                                lse_d, ws_d, early_kv=True)
                else:
                    md.kv_append(kb, vb_, k_, v_, pos_buf[j])
                    md.draft_attn_sparse(q_, kb, vb_, pos_buf[j + 1], sink, window, scale, out_d, lse_d, ws_d)
                if tp > 1:
                    gather_rank_major(out_d, gath_d, group=tp_group)
            else:
                if fused:
                    md.verify_attn_full_append(q_, kb, vb_, k_, v_, pos_buf[gamma + 1], max_kv, scale, out_v,
                                               lse_v, ws_v)
                else:
                    md.kv_append(kb, vb_, k_, v_, pos_buf[0])
                    md.verify_attn_full(q_, kb, vb_, pos_buf[gamma + 1], max_kv, scale, out_v, lse_v, ws_v)
                if tp > 1:
                    gather_rank_major(out_v, gath_v, group=tp_group)
        cur.wait_event(pq_ready)
        if state["in_graph"]:
            md.philox_u32_dev(DRAFT_SEED, step_dev, dw_full)  # the step counter lives in device memory
            md.philox_u32_dev(SEED, step_dev, rnd_full)
            step_dev.add_(1)
        else:
            md.philox_u32(DRAFT_SEED, i, dw_full)
            md.philox_u32(SEED, i, rnd_full)
        md.spec_accept(q_t.view(Bl * gamma, 1, V), None, None, dw, dtok.view(Bl * gamma, 1), dn, mode="sample")
        md.spec_accept(p_t, q_t, dtok, rnd, out_tok, nacc, committed, mode="sample")
        h_out.copy_(out_tok, non_blocking=True)
        h_n.copy_(nacc, non_blocking=True)
        if not state["in_graph"]:
            step_done.record(cur)

    step_done.record(torch.cuda.current_stream())
    e2e_step(10_000)
    torch.cuda.synchronize()
    g_e2e = None
    if tp == 1 and not args.no_graph:
        try:
            state["in_graph"] = True
            g_e2e = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_e2e):
                e2e_step(0)
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001 - the eager loop below is the same step
            print(f"e2e graph capture failed ({type(e).__name__}: {e}); timing the eager loop", file=sys.stderr)
            g_e2e = None
            torch.cuda.synchronize()
        state["in_graph"] = False
        if g_e2e is not None:
            g_e2e.replay()  # warm-up replay
            torch.cuda.synchronize()
    # the timed steps draw the same uniforms as the device-timed steps (Philox steps
    # warmup .. warmup + steps - 1), so both see the same acceptances and tokens per step
    step_dev.fill_(args.warmup)
    k_e2e = max(1, args.steps)
    c1 = committed.clone()
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    a.record()
    for i in range(k_e2e):
        if g_e2e is not None:
            g_e2e.replay()
        else:
            e2e_step(args.warmup + i)
    b_.record()
    torch.cuda.synchronize()
    e_ms = a.elapsed_time(b_)
    e_tok = int((committed - c1).sum().item())
    if world > 1:
        from paper_2408_11049_b200.tp import all_reduce_host
        e_ms = all_reduce_host([e_ms], "max")[0]
        e_tok = int(round(all_reduce_host([e_tok], "sum")[0])) // tp
    return {"value": round(e_tok / (e_ms / 1e3), 2), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": k_e2e, "ms_per_step": round(e_ms / k_e2e, 4),
            "tokens_per_step": round(e_tok / k_e2e, 1),
            "cuda_graph": ("whole step incl. H2D / D2H copies" if g_e2e is not None else False)}


# ------------------------------------------------------------------------------------------
# the oracle (reference arm / cpu_baseline)
# ------------------------------------------------------------------------------------------
def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"nproc": usable, "cpu_count": os.cpu_count(), "cpu_model": model}


_UNIT_CACHE = {}


def _oracle_unit(args):
    """Oracle time of one (sequence, KV head) unit of one layer: gamma draft calls (O3) + one verify
    call (O2) over the unit's g query heads, inputs regenerated from the seeded generators (not
    timed).  Runs in a worker process."""
    config, b, kvh = args
    import synth as S
    from oracle import attention as OA
    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[config]
    T, g = gamma + 1, Hq // Hkv
    reg = S.Regime("peaky", sink=sink)
    L0 = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
    n = int(L0[b]) + T
    kb = S.k_to_bf16_bits(S.kv_cache_k(SEED, S.T_KCACHE, B, Hkv, d, 0, n, b_sel=[b], h_sel=[kvh], regime=reg))
    vb = S.k_to_bf16_bits(S.kv_cache_k(SEED, S.T_VCACHE, B, Hkv, d, 0, n, b_sel=[b], h_sel=[kvh], regime=reg))
    qvb = S.k_to_bf16_bits(S.q_rows_k(SEED, S.T_QVERIFY, B, T, Hq, Hkv, d, b_sel=[b], regime=reg))
    qdb = S.k_to_bf16_bits(S.q_rows_k(SEED, S.T_QDRAFT, B, 1, Hq, Hkv, d, b_sel=[b], regime=reg))[:, 0]
    hs = slice(kvh * g, (kvh + 1) * g)
    scale = float(np.float32(1 / np.sqrt(d)))
    t0 = time.perf_counter()
    for j in range(gamma):
        OA.draft_attn_sparse(qdb[:, hs], kb, vb, np.array([int(L0[b]) + j + 1]), sink, window, scale)
    OA.verify_attn_full(qvb[:, :, hs], kb, vb, np.array([n]), scale)
    return time.perf_counter() - t0


def _units_sample(config, n, salt=0):
    B, Hq, Hkv = CONFIGS[config][:3]
    rng = np.random.default_rng(1234 + salt)
    flat = rng.choice(B * Hkv, size=min(n, B * Hkv), replace=False)
    return [(config, int(u // Hkv), int(u % Hkv)) for u in flat]


def oracle_pool(procs):
    """Worker processes for the multi-process oracle leg (spawned: no CUDA state is inherited)."""
    import multiprocessing as mp
    return mp.get_context("spawn").Pool(procs, initializer=_blas_1)


def oracle_units_rate(config, n_units, procs, salt=0, pool=None):
    """(units per second, seconds, units) of the oracle over a seeded sample of (b, kv head) units,
    on `procs` worker processes of `pool` (procs = 1: in this process)."""
    units = _units_sample(config, n_units, salt)
    t0 = time.perf_counter()
    if procs == 1:
        per = [_oracle_unit(u) for u in units]
    else:
        per = pool.map(_oracle_unit, units, chunksize=1)
    wall = time.perf_counter() - t0
    # the workers regenerate their inputs (untimed inside _oracle_unit): the rate counts the
    # oracle's own compute, sum(per) over `procs` workers in parallel
    busy = sum(per)
    eff_wall = max(busy / procs, max(per))
    return len(units) / eff_wall, wall, len(units)


def _blas_1():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=1)
    except Exception:  # pragma: no cover
        pass


def accept_inputs(config, alpha):
    """The acceptance rows p, q of the workload (the same seeded generator as the GPU arm)."""
    import synth as S
    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, _ = CONFIGS[config]
    sigma = S.sigma_for_overlap(SEED, V, alpha)
    p, q, _ = S.spec_probs(SEED, B, gamma, V, sigma)
    return p, q


def oracle_accept_seconds(config, p, q, step):
    """Oracle time of one step's draft-token sampling (gamma = 0 acceptance over the q rows) and
    acceptance over the batch; returns (seconds, tokens emitted) on the same inputs and Philox
    words as the GPU arm's step `step` (so the same tokens: the acceptance is bit-exact)."""
    from oracle import accept as OACC
    from oracle import philox as OPH
    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, _ = CONFIGS[config]
    t0 = time.perf_counter()
    dw = OPH.philox_words(DRAFT_SEED, step, B * gamma, 2)
    dt, _, _ = OACC.spec_accept(q.reshape(B * gamma, 1, V), np.zeros((B * gamma, 0, V), np.float32),
                                np.zeros((B * gamma, 0), np.int32), dw, "sample")
    d = dt[:, 0].reshape(B, gamma).astype(np.int32)
    rnd = OPH.philox_words(SEED, step, B, gamma + 2)
    _, n, _ = OACC.spec_accept(p, q, d, rnd, "sample")
    return time.perf_counter() - t0, int((n + 1).sum())


def cpu_baseline(config, tokens_per_step, budget_s=20.0):
    """The oracle timed on this host's cores: a multi-process leg over (b, kv head) units on every
    usable core and a single-process leg, each on a seeded sample of units of one layer and
    extrapolated to a whole step (B x Hkv units x layers) plus the batch's acceptance."""
    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[config]
    info = host_info()
    cores = info["nproc"]
    p, q = accept_inputs(config, alpha)
    with _blas_threads_1():
        t_acc, _ = oracle_accept_seconds(config, p, q, 0)
        r1, w1, n1 = oracle_units_rate(config, 2, 1, salt=1)
    per_unit = 1.0 / r1
    n_mt = max(cores, int(min(4 * cores, budget_s * 0.6 / max(per_unit, 1e-3) * cores)))
    with oracle_pool(cores) as pool:
        rm, wm, nm = oracle_units_rate(config, n_mt, cores, salt=2, pool=pool)
    units_step = B * Hkv * layers
    step_st = units_step / r1 + t_acc
    step_mt = units_step / rm + t_acc
    return {"value": round(tokens_per_step / step_mt, 4), "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "threads": cores, "nproc": info["nproc"], "cpu_model": info["cpu_model"],
            "sample": (f"{nm} (b, kv head) units of 1 of {layers} layers (gamma={gamma} draft calls + 1 verify "
                       f"over each unit's {Hq // Hkv} query heads, full context) on {cores} worker processes, "
                       f"+ the whole batch's draft sampling and acceptance (V={V}); extrapolated to "
                       f"{units_step} units per step"),
            "multi_thread": {"workers": cores, "units": nm, "units_per_s": round(rm, 4), "wall_s": round(wm, 2),
                             "tokens_per_s": round(tokens_per_step / step_mt, 4),
                             "seconds_per_step_extrapolated": round(step_mt, 1)},
            "single_thread": {"workers": 1, "units": n1, "units_per_s": round(r1, 4), "wall_s": round(w1, 2),
                              "tokens_per_s": round(tokens_per_step / step_st, 4),
                              "seconds_per_step_extrapolated": round(step_st, 1)},
            "accept_seconds_per_step": round(t_acc, 3)}


def _blas_threads_1():
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=1)
    except Exception:  # pragma: no cover
        import contextlib
        return contextlib.nullcontext()


def run_reference(args):
    """The reference arm: the fp64 oracle as it stands, on this host's cores, for the same
    workload, Philox steps and therefore the same tokens per step as the GPU arm (its acceptance
    is bit-identical).  Each step is a bounded sample: the batch's full draft sampling and
    acceptance plus a seeded sample of (b, kv head) attention units of one layer on every core;
    `value` extrapolates the sample to the whole step (B x Hkv units x layers) and `ms_per_step`
    is the measured time of the sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[args.config]
    if args.alpha is not None:
        alpha = args.alpha
    world = int(os.environ.get("WORLD_SIZE", "1"))
    info = host_info()
    cores = info["nproc"]
    units_step = B * Hkv * layers
    ext, meas, toks = [], [], 0
    p, q = accept_inputs(args.config, alpha)
    with _blas_threads_1(), oracle_pool(cores) as pool:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            t_acc, tk = oracle_accept_seconds(args.config, p, q, i)
            rate, wall, nu = oracle_units_rate(args.config, cores, cores, salt=100 + i, pool=pool)
            if i >= args.warmup:
                meas.append(time.perf_counter() - t0)
                ext.append(units_step / rate + t_acc)
                toks += tk
    tokens_per_step = toks / args.steps
    step_s = float(np.mean(ext))
    value = tokens_per_step / step_s
    sample = (f"per step: the whole batch's draft sampling + acceptance (same Philox steps as the GPU arm: "
              f"identical tokens) + {cores} of {units_step} (b, kv head) layer units on {cores} worker processes, "
              f"extrapolated")
    res = {"metric": METRIC, "value": round(value, 4), "unit": "tokens/s", "impl": "reference", "n_gpus": 0,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(float(np.mean(meas)) * 1e3, 2),
           "extrapolated_ms_per_step": round(step_s * 1e3, 1), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (the same seeded generators and Philox steps)",
           "config": workload_config(args.config, alpha, world),
           "tokens_per_step": round(tokens_per_step, 3),
           "cpu_baseline": {"value": round(value, 4), "unit": "tokens/s", "cores": cores, "kind": "oracle",
                            "threads": cores, "nproc": info["nproc"], "cpu_model": info["cpu_model"],
                            "sample": sample},
           "e2e": {"value": round(value, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)
    return res


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="llama3_b64_32k", choices=sorted(CONFIGS))
    ap.add_argument("--alpha", type=float, default=None,
                    help="target draft/target overlap beta (default: the config's 0.8; the paper's range 0.68-0.93)")
    ap.add_argument("--layers", type=int, default=0, help="override the model's layer count")
    ap.add_argument("--rot", type=int, default=4, help="physically distinct layer caches cycled through")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-fused-append", action="store_true",
                    help="separate md_kv_append launches instead of the *_append attention calls")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="budget of the cpu_baseline oracle legs")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-ar", action="store_true")
    ap.add_argument("--skip-efficiency", action="store_true", help="N>1: skip the unsharded T(1) timing on rank 0")
    ap.add_argument("--plan-only", action="store_true", help="multi-rank plumbing only (no kernels; gloo on CPU)")
    ap.add_argument("--tp-exchange", choices=["auto", "nccl", "p2p"], default="auto",
                    help="N>1: the fused peer-store exchange (f1) when it self-tests OK (auto), or NCCL")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours" and not args.plan_only:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args, argv)
    if args.plan_only:
        run_plan_only(args)
        return 0
    run_gpu(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
