"""The MD_DEBUG build (libmagicdec_b200_debug.so: "device-side preconditions are
undefined behaviour in release builds ... building with MD_DEBUG traps on a violation").

Each scenario runs in a child process (a device trap poisons the CUDA context): valid calls
through the debug library give the release library's bits; each violated precondition of
include/magicdec_b200.h makes the child fail with a CUDA launch error instead of returning."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2408_11049_b200 as md

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(os.path.dirname(md.__file__), "libmagicdec_b200_debug.so")

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2408_11049_b200 as md
import synth as S
scenario, out_path = sys.argv[1], sys.argv[2]
dev = torch.device("cuda", 0)
B, Hq, Hkv, d, cap, gamma, V = 3, 8, 2, 128, 320, 3, 40
T = gamma + 1
to_dev = lambda bits: torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(dev)
kc = to_dev(S.k_to_bf16_bits(S.kv_cache_k(5, S.T_KCACHE, B, Hkv, d, 0, cap)))
vc = to_dev(S.k_to_bf16_bits(S.kv_cache_k(5, S.T_VCACHE, B, Hkv, d, 0, cap)))
L = np.array([300, 257, 64], np.int32)
kv = torch.from_numpy(L).to(dev)
qv = to_dev(S.k_to_bf16_bits(S.new_kv_k(6, S.T_QVERIFY, B, T, Hq, d)))
qd = to_dev(S.k_to_bf16_bits(S.new_kv_k(7, S.T_QDRAFT, B, 1, Hq, d)).reshape(B, Hq, d))
kn = to_dev(S.k_to_bf16_bits(S.new_kv_k(8, S.T_KNEW, B, T, Hkv, d)))
vn = to_dev(S.k_to_bf16_bits(S.new_kv_k(9, S.T_VNEW, B, T, Hkv, d)))
scale = float(np.float32(1 / np.sqrt(d)))
ws = torch.zeros(md.attn_workspace_bytes(B, Hq, Hkv, d, T, cap), dtype=torch.uint8, device=dev)
ov = torch.zeros((B, T, Hq, d), device=dev)
od = torch.zeros((B, Hq, d), device=dev)
rng = np.random.default_rng(3)
p = rng.random((B, gamma + 1, V)); p /= p.sum(-1, keepdims=True)
q = rng.random((B, gamma, V)); q /= q.sum(-1, keepdims=True)
pt = torch.from_numpy(p.astype(np.float32)).to(dev)
qt = torch.from_numpy(q.astype(np.float32)).to(dev)
dt = torch.from_numpy(rng.integers(0, V, (B, gamma)).astype(np.int32)).to(dev)
rnd = torch.zeros((B, gamma + 2), dtype=torch.int32, device=dev)
md.philox_u32(11, 0, rnd)
otok = torch.zeros((B, gamma + 1), dtype=torch.int32, device=dev)
nacc = torch.zeros(B, dtype=torch.int32, device=dev)
if scenario == "valid":
    md.kv_append(kc, vc, kn, vn, torch.from_numpy(L - T).to(dev))
    md.verify_attn_full(qv, kc, vc, kv, cap, scale, ov, None, ws)
    md.draft_attn_sparse(qd, kc, vc, kv, 4, 60, scale, od, None, ws)
    md.spec_accept(pt, qt, dt, rnd, otok, nacc)
elif scenario == "verify_kv_len_over_capacity":
    md.verify_attn_full(qv, kc, vc, torch.from_numpy(np.array([300, cap + 64, 64], np.int32)).to(dev), cap, scale,
                        ov, None, ws)
elif scenario == "verify_kv_len_below_T":
    md.verify_attn_full(qv, kc, vc, torch.from_numpy(np.array([300, 2, 64], np.int32)).to(dev), cap, scale, ov,
                        None, ws)
elif scenario == "draft_kv_len_zero":
    md.draft_attn_sparse(qd, kc, vc, torch.from_numpy(np.array([300, 0, 64], np.int32)).to(dev), 4, 60, scale, od,
                         None, ws)
elif scenario == "append_past_capacity":
    md.kv_append(kc, vc, kn, vn, torch.from_numpy(np.array([0, cap - 2, 5], np.int32)).to(dev))
elif scenario == "accept_token_out_of_range":
    dt[1, 0] = V + 3
    md.spec_accept(pt, qt, dt, rnd, otok, nacc)
elif scenario == "accept_nan_probability":
    pt[2, 1, :] = float("nan")
    dt[2, 0] = 0
    md.spec_accept(pt, qt, dt, rnd, otok, nacc)
else:
    raise SystemExit("unknown scenario")
torch.cuda.synchronize()
np.savez(out_path, ov=ov.cpu().numpy(), od=od.cpu().numpy(), otok=otok.cpu().numpy(), nacc=nacc.cpu().numpy(),
         kc=kc.view(torch.int16).cpu().numpy(), vc=vc.view(torch.int16).cpu().numpy())
print("CHILD_OK")
'''


def run_child(scenario, lib, tmp_path):
    script = tmp_path / "child.py"
    script.write_text(CHILD.format(root=ROOT))
    out = tmp_path / f"{scenario}_{os.path.basename(lib)}.npz"
    env = dict(os.environ, MD_LIB=lib)
    r = subprocess.run([sys.executable, str(script), scenario, str(out)], capture_output=True, text=True, env=env,
                       timeout=240)
    return r, out


def test_debug_library_exports_the_abi():
    if not os.path.exists(DEBUG_LIB):
        pytest.skip("debug library not built")
    out = subprocess.run(["nm", "-D", "--defined-only", DEBUG_LIB], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(md.ABI_SYMBOLS) <= exported


@pytest.mark.gpu
def test_debug_build_valid_calls_match_release(tmp_path):
    assert os.path.exists(DEBUG_LIB), "build() makes libmagicdec_b200_debug.so"
    rd, od = run_child("valid", DEBUG_LIB, tmp_path)
    assert rd.returncode == 0 and "CHILD_OK" in rd.stdout, rd.stderr[-2000:]
    rr, orr = run_child("valid", md.LIB_PATH, tmp_path)
    assert rr.returncode == 0 and "CHILD_OK" in rr.stdout, rr.stderr[-2000:]
    a, b = np.load(od), np.load(orr)
    for k in ("ov", "od", "otok", "nacc", "kc", "vc"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.gpu
@pytest.mark.parametrize("scenario", ["verify_kv_len_over_capacity", "verify_kv_len_below_T", "draft_kv_len_zero",
                                      "append_past_capacity", "accept_token_out_of_range",
                                      "accept_nan_probability"])
def test_debug_build_traps_on_violated_preconditions(scenario, tmp_path):
    r, _ = run_child(scenario, DEBUG_LIB, tmp_path)
    assert r.returncode != 0 and "CHILD_OK" not in r.stdout, (scenario, r.stdout[-500:])
    err = r.stderr.lower()
    assert "cuda" in err or "launch" in err or "illegal" in err or "trap" in err, r.stderr[-2000:]
