#!/usr/bin/env python
"""bench.py — MagicDec self-speculative decode hot path on B200 (attention-only spec step).

One STEP = one self-speculation round of the whole hot path over one batch
(T_total = gamma*T_D + T_V):
    for j in 0..gamma-1, for each of the model's layers:  md_kv_append(T=1) + md_draft_attn_sparse
    for each layer:                                        md_kv_append(T=gamma+1) + md_verify_attn_full
    md_philox_u32 + md_spec_accept   (committed_len += n + 1 on the device)
Workload (N=1): BASELINE.json's metric point, Llama-3.1-8B-shaped GQA (32 q / 8 kv heads,
d=128, 32 layers), B=64, ctx=32768, gamma=4, StreamingLLM sink 4 + window 1020, V=128256;
synthetic seeded KV/Q (attention-sink regime) and synthetic p/q with overlap ~0.8.
32 layers x 8.6 GB of KV do not fit in 180 GB, so the layers cycle over R=4 physically
distinct 8.6 GB layer caches: every layer-call still streams its full KV from HBM
(R*8.6 GB >> 126 MB L2), in the model's order (a draft step runs through all layers).

metric: spec-step tokens/s (sum over the batch of n_b + 1 emitted tokens / step time),
plus achieved HBM GB/s of verify and draft against the measured copy peak and 8 TB/s.
The number excludes every linear layer by construction: it is NOT comparable to the
paper's end-to-end tokens/s (P:538 etc.).

--impl reference runs the fp64 CPU oracle (oracle/) on a bounded sample of the same
workload and extrapolates (the oracle is the reference arm for this build).
Multi-GPU (torchrun, --gpus N): KV-head tensor parallel -- every rank
runs the same calls on Hkv/N heads and all-gathers per-head outputs over NCCL.
"""
from __future__ import annotations

import argparse
import json
import os
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
# the GPU arm
# ------------------------------------------------------------------------------------------
def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2408_11049_b200 as md
    import synth as S
    import synth.cuda as SC
    from paper_2408_11049_b200.tp import gather_rank_major, head_shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one process per GPU; LOCAL_RANK wraps only when testing several ranks on fewer GPUs
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("MD_DIST_BACKEND", "nccl")   # gloo only for single-GPU smoke tests
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    md.load_library()

    B, Hq_full, Hkv_full, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[args.config]
    if args.layers:
        layers = args.layers
    T = gamma + 1
    qsl, kvsl = head_shard(Hq_full, Hkv_full, rank, world)
    Hq, Hkv = qsl.stop - qsl.start, kvsl.stop - kvsl.start
    steps_total = args.warmup + args.steps + 2
    cap = ctx + steps_total * T + 16
    cap = (cap + 7) // 8 * 8
    R = args.rot
    dev = torch.device("cuda", local)
    reg = S.Regime("peaky", sink=sink)

    # ---- inputs resident in HBM (the rank's heads: global head coordinates via a full-size view)
    L0 = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
    kc, vc = [], []
    for r in range(R):
        k = torch.empty((B, Hkv_full, cap, d), dtype=torch.bfloat16, device=dev) if world == 1 else None
        if world == 1:
            v = torch.empty_like(k)
            SC.fill_cache(k, SEED + r, S.T_KCACHE, 0, cap, reg)
            SC.fill_cache(v, SEED + r, S.T_VCACHE, 0, cap, reg)
        else:  # generate the full layout in chunks of heads is wasteful; fill the local heads directly
            k = torch.empty((B, Hkv, cap, d), dtype=torch.bfloat16, device=dev)
            v = torch.empty_like(k)
            SC.fill_cache(k, SEED + r + 1000 * rank, S.T_KCACHE, 0, cap, reg)
            SC.fill_cache(v, SEED + r + 1000 * rank, S.T_VCACHE, 0, cap, reg)
        kc.append(k)
        vc.append(v)
    qv_full = torch.empty((B, T, Hq_full, d), dtype=torch.bfloat16, device=dev)
    qd_full = torch.empty((B, Hq_full, d), dtype=torch.bfloat16, device=dev)
    SC.fill_q(qv_full, SEED, S.T_QVERIFY, Hkv_full, reg)
    SC.fill_q(qd_full, SEED, S.T_QDRAFT, Hkv_full, reg)
    qv = qv_full[:, :, qsl].contiguous()
    qd = qd_full[:, qsl].contiguous()
    knew_v = torch.empty((B, T, Hkv, d), dtype=torch.bfloat16, device=dev)
    vnew_v = torch.empty_like(knew_v)
    SC.fill_new_kv(knew_v, SEED, S.T_KNEW)
    SC.fill_new_kv(vnew_v, SEED, S.T_VNEW)
    knew_d, vnew_d = knew_v[:, :1].contiguous(), vnew_v[:, :1].contiguous()

    sigma = S.sigma_for_overlap(SEED, V, alpha)
    p_np, q_np, d_np = S.spec_probs(SEED, B, gamma, V, sigma)
    p_t, q_t = torch.from_numpy(p_np).to(dev), torch.from_numpy(q_np).to(dev)
    dtok = torch.from_numpy(d_np).to(dev)
    rnd = torch.empty((B, gamma + 2), dtype=torch.int32, device=dev)
    out_tok = torch.empty((B, T), dtype=torch.int32, device=dev)
    nacc = torch.empty(B, dtype=torch.int32, device=dev)
    committed = torch.from_numpy(L0.copy()).to(dev)
    ar = torch.arange(gamma + 2, dtype=torch.int32, device=dev)[:, None]

    scale = float(np.float32(1.0 / np.sqrt(d)))
    max_kv = int(L0.max()) + steps_total * T + T
    assert max_kv <= cap
    out_v = torch.empty((B, T, Hq, d), device=dev)
    lse_v = torch.empty((B, T, Hq), device=dev)
    out_d = torch.empty((B, Hq, d), device=dev)
    lse_d = torch.empty((B, Hq), device=dev)
    ws_v = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, T, max_kv)), dtype=torch.uint8, device=dev)
    ws_d = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, 1, min(sink + window, cap))),
                       dtype=torch.uint8, device=dev)
    gath_v = torch.empty((world, B, T, Hq, d), device=dev) if world > 1 else None
    gath_d = torch.empty((world, B, Hq, d), device=dev) if world > 1 else None
    # f1: the fused exchange (peer stores + md_tp_barrier) replaces the all-gather when the peer
    # buffers can be mapped and a self-test call agrees bit for bit with the NCCL all-gather of
    # the plain call; otherwise (or with --tp-exchange nccl) the NCCL all-gather is used
    xv = xd = None
    exchange = "nccl" if world > 1 else "none"
    if world > 1 and args.tp_exchange in ("p2p", "auto"):
        ok = 1
        try:
            from paper_2408_11049_b200.tp import PeerExchange, gather_heads
            xv = PeerExchange((B, T, Hq_full, d))
            xd = PeerExchange((B, Hq_full, d))
            kv_t = torch.from_numpy((L0 + 1).astype(np.int32)).to(dev)
            md.draft_attn_sparse_tp(qd, kc[0], vc[0], kv_t, sink, window, scale, xd.out, None, ws_d)
            xd.barrier()
            md.draft_attn_sparse(qd, kc[0], vc[0], kv_t, sink, window, scale, out_d, None, ws_d)
            ref = gather_heads(out_d, world)
            torch.cuda.synchronize()
            ok = int(torch.equal(xd.buf, ref))
        except Exception as e:  # noqa: BLE001 - any failure selects the NCCL path
            print(f"rank {rank}: fused exchange unavailable ({type(e).__name__}: {e}); using NCCL", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 1:
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
                # fused: the append runs inside the draft kernel (one launch per layer-call)
                kn_, vn_ = (knew_d, vnew_d) if fused else (None, None)
                if not fused:
                    md.kv_append(kb, vb, knew_d, vnew_d, pos[j])
                if xd is not None:
                    md.draft_attn_sparse_tp(qd, kb, vb, pos[j + 1], sink, window, scale, xd.out, lse_d, ws_d,
                                            k_new=kn_, v_new=vn_)
                    xd.barrier()
                    continue
                if fused:
                    md.draft_attn_sparse_append(qd, kb, vb, knew_d, vnew_d, pos[j + 1], sink, window, scale, out_d,
                                                lse_d, ws_d)
                else:
                    md.draft_attn_sparse(qd, kb, vb, pos[j + 1], sink, window, scale, out_d, lse_d, ws_d)
                if world > 1:
                    gather_rank_major(out_d, gath_d)
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
            if world > 1:
                gather_rank_major(out_v, gath_v)

    # per layer-call: md_kv_append + one attention kernel (stream-K, merge fused); + philox + accept
    launches_per_step = gamma * layers * 2 + layers * 2 + 2
    if fused:
        launches_per_step -= gamma * layers + layers
    if world > 1:
        launches_per_step += gamma * layers + layers  # the exchange after every attention call

    # positions for the step are one plumbing op on the committed lengths
    pos_buf = torch.empty((gamma + 2, B), dtype=torch.int32, device=dev)

    use_graph = not args.no_graph and (world == 1 or exchange == "p2p")  # NCCL calls stay eager
    graph = None
    step_dev = torch.zeros(1, dtype=torch.int64, device=dev)

    # default: the layer loop (gamma*layers draft + layers verify calls) is one CUDA graph and
    # philox + accept follow it; MD_BENCH_GRAPH=whole captures the whole step including them
    # (philox reads its step from device memory).  Measured A/B on one box: 49.7 vs 50.7 ms/step.
    split = os.environ.get("MD_BENCH_GRAPH", "split") != "whole"

    def whole_step():
        # one speculation step: gamma x layers draft calls, layers verify calls, uniforms and
        # acceptance -- captured as ONE CUDA graph; the Philox step lives in device
        # memory so every replay draws fresh uniforms
        torch.add(committed[None, :], ar, out=pos_buf)
        layer_pass(pos_buf)
        if split:
            return
        md.philox_u32_dev(SEED, step_dev, rnd)
        md.spec_accept(p_t, q_t, dtok, rnd, out_tok, nacc, committed, mode="sample")
        step_dev.add_(1)

    if use_graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        c_save = committed.clone()
        with torch.cuda.stream(s):
            whole_step()  # warm-up outside the capture (kernel attributes, allocator)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        committed.copy_(c_save)
        step_dev.zero_()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            whole_step()
        torch.cuda.synchronize()
        committed.copy_(c_save)
        step_dev.zero_()

    def step_g(i):
        if graph is not None:
            graph.replay()
        else:
            whole_step()
        if split:
            md.philox_u32(SEED, i, rnd)
            md.spec_accept(p_t, q_t, dtok, rnd, out_tok, nacc, committed, mode="sample")

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
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    tokens = int((committed - c0).sum().item())
    ms_per_step = ms / args.steps
    value = tokens / (ms / 1e3)

    # ---- per-kernel roofline: verify and draft calls timed alone with CUDA events on the launch stream
    kvl_now = (committed + T).cpu().numpy()
    kv_len_v = torch.from_numpy(kvl_now.astype(np.int32)).to(dev)
    kv_len_d = torch.from_numpy((committed + 1).cpu().numpy().astype(np.int32)).to(dev)
    nrep = max(2 * R, 8)

    def time_calls(fn):
        fn(0)
        torch.cuda.synchronize()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for r in range(nrep):
            fn(r)
        b_.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b_) / nrep

    # the kernels the step runs: with the fused append, the *_append calls (their algorithmic
    # bytes add the new rows read from k_new / v_new and written to the cache: 4 B*T*Hkv*d*2)
    fused_step = fused
    if fused_step:
        v_ms = time_calls(lambda r: md.verify_attn_full_append(qv, kc[r % R], vc[r % R], knew_v, vnew_v, kv_len_v,
                                                               max_kv, scale, out_v, lse_v, ws_v))
        d_ms = time_calls(lambda r: md.draft_attn_sparse_append(qd, kc[r % R], vc[r % R], knew_d, vnew_d, kv_len_d,
                                                                sink, window, scale, out_d, lse_d, ws_d))
    else:
        v_ms = time_calls(lambda r: md.verify_attn_full(qv, kc[r % R], vc[r % R], kv_len_v, max_kv, scale, out_v,
                                                        lse_v, ws_v))
        d_ms = time_calls(lambda r: md.draft_attn_sparse(qd, kc[r % R], vc[r % R], kv_len_d, sink, window, scale,
                                                         out_d, lse_d, ws_d))
    vb = verify_bytes(kvl_now, Hkv, Hq, d, T) + (4 * B * T * Hkv * d * 2 if fused_step else 0)
    db = draft_bytes(kvl_now - T + 1, Hkv, Hq, d, sink, window) + (4 * B * Hkv * d * 2 if fused_step else 0)
    v_gbs, d_gbs = vb / v_ms / 1e6, db / d_ms / 1e6
    peak, peak_kind = load_peaks()
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(args.config, {}).get("verify_dram_bytes_per_launch")

    # ---- AR context: one autoregressive step (T=1 decode) over the same caches, attention only
    ar_ms = None
    if world == 1 and not args.skip_ar:
        kv_len_ar = kv_len_d
        out_a = torch.empty((B, 1, Hq, d), device=dev)
        lse_a = torch.empty((B, 1, Hq), device=dev)
        ws_a = torch.zeros(max(1, md.attn_workspace_bytes(B, Hq, Hkv, d, 1, max_kv)), dtype=torch.uint8, device=dev)
        qa = qv[:, :1].contiguous()
        ar_ms = time_calls(lambda r: md.verify_attn_full(qa, kc[r % R], vc[r % R], kv_len_ar, max_kv, scale, out_a,
                                                         lse_a, ws_a)) * layers

    # ---- e2e: the same step with every input copied from pinned host memory and the result read back
    e2e = None
    if not args.skip_e2e:
        h_qd, h_qv = qd.cpu().pin_memory(), qv.cpu().pin_memory()
        h_kd, h_vd = knew_d.cpu().pin_memory(), vnew_d.cpu().pin_memory()
        h_kv, h_vv = knew_v.cpu().pin_memory(), vnew_v.cpu().pin_memory()
        h_p, h_q, h_d = p_t.cpu().pin_memory(), q_t.cpu().pin_memory(), dtok.cpu().pin_memory()
        h_out = torch.empty((B, T), dtype=torch.int32).pin_memory()
        h_n = torch.empty(B, dtype=torch.int32).pin_memory()
        h2d = (gamma * layers * (h_qd.nbytes + h_kd.nbytes + h_vd.nbytes) +
               layers * (h_qv.nbytes + h_kv.nbytes + h_vv.nbytes) + h_p.nbytes + h_q.nbytes + h_d.nbytes)
        d2h = h_out.nbytes + h_n.nbytes

        # Every call has its own device staging slot (223 MB at the target point), and all of a
        # step's H2D copies are issued up front on their own stream, in call order; the compute
        # stream waits only at a few group boundaries (calls [0,1), [1,8), [8,32), then every 32),
        # so the copy engine runs ahead (55 GB/s vs ~15 GB/s of inputs consumed by the draft calls)
        # while consecutive kernels keep their programmatic-dependent-launch overlap (an event
        # wait before every call cost ~4 us per call).  p / q (295 MB) ride behind the verify
        # inputs and are waited for only by the acceptance.
        copy_s = torch.cuda.Stream()
        ncalls = gamma * layers + layers
        nd = gamma * layers                      # draft calls come first, then the verify calls
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
        in_graph = False

        def issue_copies(cur):
            with torch.cuda.stream(copy_s):
                if in_graph:  # fork the copy stream from the capturing stream
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
                dtok.copy_(h_d, non_blocking=True)
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
                                                    lse_d, ws_d)
                    else:
                        md.kv_append(kb, vb_, k_, v_, pos_buf[j])
                        md.draft_attn_sparse(q_, kb, vb_, pos_buf[j + 1], sink, window, scale, out_d, lse_d, ws_d)
                    if world > 1:
                        gather_rank_major(out_d, gath_d)
                else:
                    if fused:
                        md.verify_attn_full_append(q_, kb, vb_, k_, v_, pos_buf[gamma + 1], max_kv, scale, out_v,
                                                   lse_v, ws_v)
                    else:
                        md.kv_append(kb, vb_, k_, v_, pos_buf[0])
                        md.verify_attn_full(q_, kb, vb_, pos_buf[gamma + 1], max_kv, scale, out_v, lse_v, ws_v)
                    if world > 1:
                        gather_rank_major(out_v, gath_v)
            cur.wait_event(pq_ready)
            if in_graph:
                md.philox_u32_dev(SEED, step_dev, rnd)  # the step counter lives in device memory
                step_dev.add_(1)
            else:
                md.philox_u32(SEED, i, rnd)
            md.spec_accept(p_t, q_t, dtok, rnd, out_tok, nacc, committed, mode="sample")
            h_out.copy_(out_tok, non_blocking=True)
            h_n.copy_(nacc, non_blocking=True)
            if not in_graph:
                step_done.record(cur)

        step_done.record(torch.cuda.current_stream())
        e2e_step(10_000)
        torch.cuda.synchronize()
        g_e2e = None
        if world == 1 and not args.no_graph:
            try:
                in_graph = True
                g_e2e = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g_e2e):
                    e2e_step(0)
                torch.cuda.synchronize()
            except Exception as e:  # noqa: BLE001 - the eager loop below is the same step
                print(f"e2e graph capture failed ({type(e).__name__}: {e}); timing the eager loop", file=sys.stderr)
                g_e2e = None
                torch.cuda.synchronize()
            in_graph = False
            if g_e2e is not None:
                g_e2e.replay()  # warm-up replay
                torch.cuda.synchronize()
        # the timed steps draw the same uniforms as the device-timed steps (Philox steps
        # warmup .. warmup + steps - 1), so both see the same acceptances and tokens per step
        step_dev.fill_(args.warmup)
        k_e2e = max(1, args.steps)
        c1 = committed.clone()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(k_e2e):
            if g_e2e is not None:
                g_e2e.replay()
            else:
                e2e_step(args.warmup + i)
        b_.record()
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b_)
        if world > 1:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e_tok = int((committed - c1).sum().item())
        e2e = {"value": round(e_tok / (e_ms / 1e3), 2), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": k_e2e, "ms_per_step": round(e_ms / k_e2e, 4),
               "tokens_per_step": round(e_tok / k_e2e, 1),
               "cuda_graph": ("whole step incl. H2D / D2H copies" if g_e2e is not None else False)}

    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.skip_cpu:
            cpu = cpu_baseline(args.config, tokens / args.steps, layers)
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
            "scaling": "strong",  # the B=64 workload is split over the N GPUs (KV-head TP)
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (seeded counter-hash KV/Q, attention-sink regime; Zipf p/q with overlap ~%.2f)" % alpha,
            "config": {"workload": args.config, "batch": B, "ctx": ctx, "gamma": gamma, "sink": sink,
                       "window": window, "num_q_heads": Hq_full, "num_kv_heads": Hkv_full, "head_dim": d,
                       "layers": layers, "vocab": V, "layer_caches_rotated": R,
                       "l2": "inputs larger than L2: each layer-call streams a distinct %.1f GB cache" %
                             (verify_bytes(kvl_now, Hkv, Hq, d, T) / 1e9),
                       "attention_only": True,
                       "cuda_graph": ("layer loop" if split else "whole step (drafts + verify + philox + accept)")
                       if use_graph else False,
                       "kv_append": "fused into the attention calls" if fused else "separate launches",
                       "parallelism": (f"tp{world} (KV heads, {exchange} exchange)" if world > 1
                                       else "single GPU")},
            "tokens_per_step": round(tokens / args.steps, 3),
            "gpu_launches": launches_per_step * args.steps,
            "roofline": {"bound": "hbm", "achieved": round(v_gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(v_gbs / peak, 4), "traffic": traffic,
                         "kernel": ("md_verify_attn_full_append" if fused_step else "md_verify_attn_full")
                         + " (attn_tc_kernel: tcgen05 MMAs with TMEM accumulators, stream-K persistent, fused split merge"
                         + (", fused kv_append)" if fused_step else ")"),
                         "algorithmic_bytes_per_launch": vb, "ms_per_launch": round(v_ms, 4),
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"},
            "verify_gbs": round(v_gbs, 1),
            "verify_frac_of_8tbs": round(v_gbs / NOMINAL_HBM_GBS, 4),
            "draft_gbs": round(d_gbs, 1),
            "draft_frac_of_8tbs": round(d_gbs / NOMINAL_HBM_GBS, 4),
            "draft_frac_of_measured": round(d_gbs / peak, 4),
            "draft_ms_per_launch": round(d_ms, 4),
            "draft_bytes_per_launch": db,
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


# ------------------------------------------------------------------------------------------
# the oracle (reference arm / cpu_baseline)
# ------------------------------------------------------------------------------------------
def oracle_step_sample(config, n_seq=1, seed=SEED):
    """Oracle time for a bounded sample: n_seq sequences x 1 layer of (gamma drafts + 1 verify)
    attention, plus n_seq acceptances.  Returns (seconds, sample description, scale factor to
    one full step = B/n_seq x layers for attention, B/n_seq for acceptance)."""
    import synth as S
    from oracle import accept as OACC
    from oracle import attention as OA
    from oracle import philox as OPH

    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[config]
    T = gamma + 1
    reg = S.Regime("peaky", sink=sink)
    L0 = S.committed_lengths(SEED, B, ctx, gamma, ragged=True)
    scale = float(np.float32(1 / np.sqrt(d)))
    t_attn = t_acc = 0.0
    for b in range(n_seq):
        n = int(L0[b]) + T
        kb = S.k_to_bf16_bits(S.kv_cache_k(seed, S.T_KCACHE, B, Hkv, d, 0, n, b_sel=[b], regime=reg))
        vb = S.k_to_bf16_bits(S.kv_cache_k(seed, S.T_VCACHE, B, Hkv, d, 0, n, b_sel=[b], regime=reg))
        qvb = S.k_to_bf16_bits(S.q_rows_k(seed, S.T_QVERIFY, B, T, Hq, Hkv, d, b_sel=[b], regime=reg))
        qdb = S.k_to_bf16_bits(S.q_rows_k(seed, S.T_QDRAFT, B, 1, Hq, Hkv, d, b_sel=[b], regime=reg))[:, 0]
        t0 = time.perf_counter()
        for j in range(gamma):
            OA.draft_attn_sparse(qdb, kb, vb, np.array([int(L0[b]) + j + 1]), sink, window, scale)
        OA.verify_attn_full(qvb, kb, vb, np.array([n]), scale)
        t_attn += time.perf_counter() - t0
        p, q, dd = S.spec_probs(seed + b, 1, gamma, V, 1.0)
        rnd = OPH.philox_words(seed, b, 1, gamma + 2)
        t0 = time.perf_counter()
        OACC.spec_accept(p, q, dd, rnd, "sample")
        t_acc += time.perf_counter() - t0
    step_s = t_attn * (B / n_seq) * layers + t_acc * (B / n_seq)
    sample = (f"{n_seq} of {B} sequences x 1 of {layers} layers (gamma={gamma} draft calls + 1 verify call, "
              f"all {Hkv} kv heads, full context) + {n_seq} acceptances (V={V}); scaled linearly to one step")
    return step_s, sample


def _blas_threads_1():
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=1)
    except Exception:  # pragma: no cover
        import contextlib
        return contextlib.nullcontext()


def cpu_baseline(config, tokens_per_step, layers=None):
    with _blas_threads_1():
        step_s, sample = oracle_step_sample(config, n_seq=2)
    return {"value": round(tokens_per_step / step_s, 4), "unit": "tokens/s", "cores": 1, "kind": "oracle",
            "sample": sample, "oracle_seconds_per_step_extrapolated": round(step_s, 2)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    B, Hq, Hkv, d, ctx, gamma, sink, window, V, layers, alpha = CONFIGS[args.config]
    from oracle.theory import omega
    tokens_per_step = B * omega(gamma, alpha)      # Eq.1 expectation at the synthetic overlap
    times = []
    with _blas_threads_1():
        for i in range(args.warmup + args.steps):
            step_s, sample = oracle_step_sample(args.config, n_seq=1, seed=SEED)
            if i >= args.warmup:
                times.append(step_s)
    step_s = float(np.mean(times))
    value = tokens_per_step / step_s
    res = {"metric": METRIC, "value": round(value, 4), "unit": "tokens/s", "impl": "reference", "n_gpus": 0,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 2),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (same seeded generators)",
           "config": {"workload": args.config, "batch": B, "ctx": ctx, "gamma": gamma, "layers": layers},
           "cpu_baseline": {"value": round(value, 4), "unit": "tokens/s", "cores": 1, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": round(value, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)
    return res


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="llama3_b64_32k", choices=sorted(CONFIGS))
    ap.add_argument("--layers", type=int, default=0, help="override the model's layer count")
    ap.add_argument("--rot", type=int, default=4, help="physically distinct layer caches cycled through")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-fused-append", action="store_true",
                    help="separate md_kv_append launches instead of the *_append attention calls")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-ar", action="store_true")
    ap.add_argument("--tp-exchange", choices=["auto", "nccl", "p2p"], default="auto",
                    help="N>1: the fused peer-store exchange (f1) when it self-tests OK (auto), or NCCL")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
