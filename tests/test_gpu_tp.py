"""GPU checks of the fused tensor-parallel output exchange and of the
graph-replayable Philox call.  One GPU here, so the P ranks are simulated in one process:
each rank has its own KV-head shard, its own stream and its own full-head output buffer, the
peer table holds every rank's buffer, and the md_tp_barrier kernels of the ranks run
concurrently on their streams.  Every rank's buffer must end up holding the full-head result,
which must equal the oracle's unsharded attention."""
import numpy as np
import pytest
import torch

import paper_2408_11049_b200 as md
import synth as S
from oracle import attention as OA
from oracle import philox as OPH
from tests.helpers import AttnCase, bits_to_torch_bf16

pytestmark = pytest.mark.gpu
ATOL_O = 2e-3


def _shard(case, world, rank):
    kvper = case.Hkv // world
    qper = case.Hq // world
    ks = slice(rank * kvper, (rank + 1) * kvper)
    qs = slice(rank * qper, (rank + 1) * qper)
    k = bits_to_torch_bf16(np.ascontiguousarray(case.k_bits[:, ks]))
    v = bits_to_torch_bf16(np.ascontiguousarray(case.v_bits[:, ks]))
    qv = bits_to_torch_bf16(np.ascontiguousarray(case.qv_bits[:, :, qs]))
    qd = bits_to_torch_bf16(np.ascontiguousarray(case.qd_bits[:, qs]))
    return k, v, qv, qd, qper, kvper


class Ranks:
    def __init__(self, world, out_shape):
        self.world = world
        self.bufs = [torch.full(out_shape, float("nan"), device="cuda") for _ in range(world)]
        self.peers = torch.tensor([b.data_ptr() for b in self.bufs], dtype=torch.int64, device="cuda")
        self.flags = [torch.zeros(world, dtype=torch.int64, device="cuda") for _ in range(world)]
        self.flag_peers = torch.tensor([f.data_ptr() for f in self.flags], dtype=torch.int64, device="cuda")
        self.epochs = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(world)]
        self.streams = [torch.cuda.Stream() for _ in range(world)]

    def out(self, rank):
        return md.tp_out(self.peers, self.world, rank)

    def sync(self, rank):
        return md.tp_sync(self.flag_peers, self.epochs[rank], self.world, rank)


@pytest.mark.parametrize("world", [2, 4])
def test_fused_tp_verify_and_draft(world):
    B, Hq, Hkv, d, T = 3, 32, 8, 128, 5
    lens = [2500, 1700, 300]
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, T=T, seed=91 + world, regime=S.Regime("peaky", sink=4))
    kvl = torch.from_numpy(case.kv_len).cuda()
    ref_v, _ = OA.verify_attn_full(case.qv_bits, case.k_bits, case.v_bits, case.kv_len, case.scale)
    ref_d, _ = OA.draft_attn_sparse(case.qd_bits, case.k_bits, case.v_bits, case.kv_len, 4, 252, case.scale)
    rv = Ranks(world, (B, T, Hq, d))
    rd = Ranks(world, (B, Hq, d))
    shards = [_shard(case, world, r) for r in range(world)]
    qper, kvper = Hq // world, Hkv // world
    # every allocation before the first barrier is enqueued: an allocation may synchronise the
    # device, and a rank's barrier cannot finish before the other ranks' calls are enqueued
    ws = [torch.zeros(md.attn_workspace_bytes(B, qper, kvper, d, T, max(lens)), dtype=torch.uint8, device="cuda")
          for _ in range(world)]
    wsd = [torch.zeros(md.attn_workspace_bytes(B, qper, kvper, d, 1, 256), dtype=torch.uint8, device="cuda")
           for _ in range(world)]
    outs_v = [rv.out(r) for r in range(world)]
    outs_d = [rd.out(r) for r in range(world)]
    syncs_v = [rv.sync(r) for r in range(world)]
    syncs_d = [rd.sync(r) for r in range(world)]
    # warm-up: the first launch of a kernel variant sets its shared-memory attribute, which may
    # synchronise the device (harmless with one process per GPU, a deadlock for ranks simulated
    # in one process once a barrier spins)
    k, v, qv, qd, _, _ = shards[0]
    md.verify_attn_full(qv, k, v, kvl, max(lens), case.scale, torch.empty_like(rv.bufs[0][:, :, :qper]), None, ws[0])
    md.draft_attn_sparse(qd, k, v, kvl, 4, 252, case.scale, torch.empty_like(rd.bufs[0][:, :qper]), None, wsd[0])
    torch.cuda.synchronize()
    for it in range(2):  # twice: the epochs advance
        for r in range(world):
            k, v, qv, qd, _, _ = shards[r]
            s = rv.streams[r]
            md.verify_attn_full_tp(qv, k, v, kvl, max(lens), case.scale, outs_v[r], None, ws[r], stream=s)
            md.tp_barrier(syncs_v[r], stream=s)
            md.draft_attn_sparse_tp(qd, k, v, kvl, 4, 252, case.scale, outs_d[r], None, wsd[r], stream=s)
            md.tp_barrier(syncs_d[r], stream=s)
        torch.cuda.synchronize()
        for r in range(world):
            assert np.max(np.abs(rv.bufs[r].cpu().numpy() - ref_v)) <= ATOL_O
            assert np.max(np.abs(rd.bufs[r].cpu().numpy() - ref_d)) <= ATOL_O
            assert int(rv.epochs[r].item()) == it + 1
            assert rv.flags[r].cpu().tolist() == [it + 1] * world


def test_fused_tp_append_verify_and_draft():
    """The _tp_append calls: each rank appends its own KV heads' new rows inside its attention
    kernel and stores its heads into every rank's buffer; against the oracle's kv_append +
    unsharded attention (verify appends T rows at kv_len - T, then the draft one row at kv_len - 1)."""
    world, B, Hq, Hkv, d, T = 2, 3, 32, 8, 128, 5
    lens = [2500, 1700, 300]
    case = AttnCase(B, Hq, Hkv, d, max(lens) + 8, lens, T=T, seed=17)
    kvl = torch.from_numpy(case.kv_len).cuda()
    kn = S.k_to_bf16_bits(S.new_kv_k(5, S.T_KNEW, B, T, Hkv, d))
    vn = S.k_to_bf16_bits(S.new_kv_k(5, S.T_VNEW, B, T, Hkv, d))
    knd = S.k_to_bf16_bits(S.new_kv_k(6, S.T_KNEW, B, 1, Hkv, d))
    vnd = S.k_to_bf16_bits(S.new_kv_k(6, S.T_VNEW, B, 1, Hkv, d))
    kc, vc = case.k_bits.copy(), case.v_bits.copy()
    OA.kv_append(kc, vc, kn, vn, case.kv_len - T)
    ref_v, _ = OA.verify_attn_full(case.qv_bits, kc, vc, case.kv_len, case.scale)
    OA.kv_append(kc, vc, knd, vnd, case.kv_len - 1)
    ref_d, _ = OA.draft_attn_sparse(case.qd_bits, kc, vc, case.kv_len, 4, 252, case.scale)
    rv, rd = Ranks(world, (B, T, Hq, d)), Ranks(world, (B, Hq, d))
    shards = [_shard(case, world, r) for r in range(world)]
    qper, kvper = Hq // world, Hkv // world
    part = lambda a, r: bits_to_torch_bf16(np.ascontiguousarray(a[:, :, r * kvper:(r + 1) * kvper]))
    news = [(part(kn, r), part(vn, r), part(knd, r), part(vnd, r)) for r in range(world)]
    ws = [torch.zeros(md.attn_workspace_bytes(B, qper, kvper, d, T, max(lens)), dtype=torch.uint8, device="cuda")
          for _ in range(world)]
    wsd = [torch.zeros(md.attn_workspace_bytes(B, qper, kvper, d, 1, 256), dtype=torch.uint8, device="cuda")
           for _ in range(world)]
    outs_v, outs_d = [rv.out(r) for r in range(world)], [rd.out(r) for r in range(world)]
    syncs_v, syncs_d = [rv.sync(r) for r in range(world)], [rd.sync(r) for r in range(world)]
    # warm-up of both kernel variants on scratch copies (shared-memory attributes; see above)
    k, v, qv, qd, _, _ = shards[0]
    k0, v0 = k.clone(), v.clone()
    md.verify_attn_full_append(qv, k0, v0, news[0][0], news[0][1], kvl, max(lens), case.scale,
                               torch.empty_like(rv.bufs[0][:, :, :qper]), None, ws[0])
    md.draft_attn_sparse_append(qd, k0, v0, news[0][2], news[0][3], kvl, 4, 252, case.scale,
                                torch.empty_like(rd.bufs[0][:, :qper]), None, wsd[0])
    torch.cuda.synchronize()
    for r in range(world):
        k, v, qv, qd, _, _ = shards[r]
        s = rv.streams[r]
        md.verify_attn_full_tp(qv, k, v, kvl, max(lens), case.scale, outs_v[r], None, ws[r], stream=s,
                               k_new=news[r][0], v_new=news[r][1])
        md.tp_barrier(syncs_v[r], stream=s)
        md.draft_attn_sparse_tp(qd, k, v, kvl, 4, 252, case.scale, outs_d[r], None, wsd[r], stream=s,
                                k_new=news[r][2], v_new=news[r][3])
        md.tp_barrier(syncs_d[r], stream=s)
    torch.cuda.synchronize()
    for r in range(world):
        assert np.max(np.abs(rv.bufs[r].cpu().numpy() - ref_v)) <= ATOL_O
        assert np.max(np.abs(rd.bufs[r].cpu().numpy() - ref_d)) <= ATOL_O
        k, v = shards[r][0], shards[r][1]
        got = k.cpu().view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(got, kc[:, r * kvper:(r + 1) * kvper])


def test_tp_world1_equals_plain_call():
    """world = 1: the _tp call writes exactly what the plain call writes (bit for bit)."""
    case = AttnCase(2, 32, 8, 128, 1100, [1000, 777], T=5, seed=95).to_cuda()
    out = torch.empty((2, 5, 32, 128), device="cuda")
    ws = torch.zeros(md.attn_workspace_bytes(2, 32, 8, 128, 5, 1000), dtype=torch.uint8, device="cuda")
    md.verify_attn_full(case.qv, case.k, case.v, case.kv_len_t, 1000, case.scale, out, None, ws)
    r = Ranks(1, (2, 5, 32, 128))
    md.verify_attn_full_tp(case.qv, case.k, case.v, case.kv_len_t, 1000, case.scale, r.out(0), None, ws)
    md.tp_barrier(r.sync(0))
    torch.cuda.synchronize()
    assert torch.equal(out, r.bufs[0])


def test_tp_rejects_bad_descriptor():
    case = AttnCase(1, 4, 1, 128, 64, [60], T=1, seed=96).to_cuda()
    peers = torch.zeros(2, dtype=torch.int64, device="cuda")
    with pytest.raises(md.MDError):
        md.verify_attn_full_tp(case.qv, case.k, case.v, case.kv_len_t, 60, case.scale, md.tp_out(peers, 2, 2))


def test_philox_dev_step_in_a_graph():
    """A captured graph that draws uniforms with the step in device memory and then advances it
    reproduces the host-step Philox words of consecutive steps on every replay."""
    B, W, seed = 5, 6, 1234
    step = torch.tensor([41], dtype=torch.int64, device="cuda")
    out = torch.empty((B, W), dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            md.philox_u32_dev(seed, step, out, stream=s)
            step.add_(1)
    torch.cuda.current_stream().wait_stream(s)
    step.fill_(41)
    for k in range(3):
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint32), OPH.philox_words(seed, 41 + k, B, W))
