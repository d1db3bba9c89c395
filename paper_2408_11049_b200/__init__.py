"""paper_2408_11049_b200 — thin Python binding of the MagicDec B200 C ABI.

Argument marshalling only: every step of the hot path runs in the CUDA kernels of
`libmagicdec_b200.so` (declared in include/magicdec_b200.h).  PyTorch is used for
device memory and streams.  There is no CPU fallback: a missing library or a CPU
tensor raises.

Functions mirror the C calls (same names without the `md_` prefix):
    kv_append, attn_workspace_bytes, verify_attn_full, draft_attn_sparse,
    draft_attn_indexed, snapkv_workspace_bytes, snapkv_select, philox_u32, spec_accept,
    verify_attn_tree, spec_accept_tree, kv_compact (tree speculation),
    pq_encode, pq_workspace_bytes, pq_select (PQCache dynamic selection)
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MD_LIB") or os.path.join(_HERE, "libmagicdec_b200.so")  # MD_LIB: A/B experiments

MD_OK, MD_ERR_INVALID_ARG, MD_ERR_UNSUPPORTED, MD_ERR_WORKSPACE, MD_ERR_CUDA = 0, 1, 2, 3, 4
MD_ACCEPT_SAMPLE, MD_ACCEPT_GREEDY = 0, 1

# the symbols include/magicdec_b200.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = ("md_abi_version", "md_last_error", "md_kv_append", "md_attn_workspace_bytes",
               "md_verify_attn_full", "md_draft_attn_sparse", "md_draft_attn_indexed", "md_snapkv_workspace_bytes",
               "md_snapkv_select", "md_philox_u32", "md_spec_accept", "md_debug_trace",
               "md_verify_attn_tree", "md_spec_accept_tree", "md_kv_compact", "md_pq_encode", "md_pq_workspace_bytes",
               "md_pq_select", "md_verify_attn_full_tp", "md_draft_attn_sparse_tp", "md_tp_barrier",
               "md_philox_u32_dev", "md_draft_attn_sparse_windows", "md_verify_attn_full_append",
               "md_draft_attn_sparse_append", "md_verify_attn_full_tp_append", "md_draft_attn_sparse_tp_append",
               "md_draft_attn_indexed_append", "md_attn_workspace_bytes_det", "md_verify_attn_full_det",
               "md_draft_attn_sparse_det", "md_draft_attn_sparse_append_ex")


class MDError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"md status {status}: {msg}")
        self.status = status


class KVCache(ctypes.Structure):
    """md_kv_cache: caller-owned [B][Hkv][cap][d] bf16 K and V with element strides."""
    _fields_ = [("k", ctypes.c_void_p), ("v", ctypes.c_void_p),
                ("batch", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("capacity", ctypes.c_int32),
                ("stride_b", ctypes.c_int64), ("stride_h", ctypes.c_int64), ("stride_s", ctypes.c_int64)]


class TPOut(ctypes.Structure):
    """md_tp_out: device array of every rank's full-head output buffer + (world, rank)."""
    _fields_ = [("out_peers", ctypes.c_void_p), ("world", ctypes.c_int32), ("rank", ctypes.c_int32)]


class TPSync(ctypes.Structure):
    """md_tp_sync: device array of every rank's uint64 flags[world], this rank's epoch counter."""
    _fields_ = [("flags_peers", ctypes.c_void_p), ("epoch", ctypes.c_void_p), ("world", ctypes.c_int32),
                ("rank", ctypes.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the CUDA library (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -m paper_2408_11049_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    c_void_p, i32, i64, f32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_size_t
    u64 = ctypes.c_uint64
    pc = ctypes.POINTER(KVCache)
    lib.md_abi_version.restype = ctypes.c_int
    lib.md_last_error.restype = ctypes.c_char_p
    lib.md_kv_append.argtypes = [pc, c_void_p, c_void_p, i32, c_void_p, c_void_p]
    lib.md_attn_workspace_bytes.argtypes = [i32, i32, i32, i32, i32, i32]
    lib.md_attn_workspace_bytes.restype = sz
    lib.md_verify_attn_full.argtypes = [pc, c_void_p, i32, i32, c_void_p, i32, f32, c_void_p, c_void_p,
                                        c_void_p, sz, c_void_p]
    lib.md_draft_attn_sparse.argtypes = [pc, c_void_p, i32, c_void_p, i32, i32, f32, c_void_p, c_void_p,
                                         c_void_p, sz, c_void_p]
    lib.md_draft_attn_sparse_windows.argtypes = [pc, c_void_p, i32, c_void_p, i32, i32, c_void_p, f32, c_void_p,
                                                 c_void_p, c_void_p, sz, c_void_p]
    lib.md_verify_attn_full_append.argtypes = [pc, c_void_p, i32, i32, c_void_p, c_void_p, c_void_p, i32, f32,
                                               c_void_p, c_void_p, c_void_p, sz, c_void_p]
    lib.md_draft_attn_sparse_append.argtypes = [pc, c_void_p, i32, c_void_p, c_void_p, c_void_p, i32, i32, f32,
                                                c_void_p, c_void_p, c_void_p, sz, c_void_p]
    lib.md_draft_attn_sparse_append_ex.argtypes = [pc, c_void_p, i32, c_void_p, c_void_p, c_void_p, i32, i32, f32,
                                                   c_void_p, c_void_p, c_void_p, sz, ctypes.c_uint32, c_void_p]
    lib.md_draft_attn_indexed_append.argtypes = [pc, c_void_p, i32, c_void_p, c_void_p, c_void_p, c_void_p, i32,
                                                 c_void_p, c_void_p, f32, c_void_p, c_void_p, c_void_p, sz, c_void_p]
    lib.md_draft_attn_indexed.argtypes = [pc, c_void_p, i32, c_void_p, c_void_p, i32, c_void_p, c_void_p, f32,
                                          c_void_p, c_void_p, c_void_p, sz, c_void_p]
    lib.md_snapkv_workspace_bytes.argtypes = [i32, i32, i32, i32, i32]
    lib.md_snapkv_workspace_bytes.restype = sz
    lib.md_snapkv_select.argtypes = [pc, c_void_p, i32, c_void_p, i32, i32, i32, c_void_p, f32, c_void_p, i32, c_void_p,
                                     c_void_p, sz, c_void_p]
    lib.md_philox_u32.argtypes = [u64, u64, i32, i32, c_void_p, c_void_p]
    lib.md_spec_accept.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, i32, i32, i32, ctypes.c_int,
                                   c_void_p, c_void_p, c_void_p, c_void_p]
    lib.md_debug_trace.argtypes = [c_void_p, sz]
    lib.md_verify_attn_tree.argtypes = [pc, c_void_p, i32, i32, c_void_p, i32, c_void_p, f32, c_void_p, c_void_p,
                                        c_void_p, sz, c_void_p]
    lib.md_spec_accept_tree.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, i32, i32, i32,
                                        ctypes.c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
    lib.md_kv_compact.argtypes = [pc, c_void_p, c_void_p, i32, c_void_p, c_void_p]
    ptp, psync = ctypes.POINTER(TPOut), ctypes.POINTER(TPSync)
    lib.md_verify_attn_full_tp.argtypes = [pc, c_void_p, i32, i32, c_void_p, i32, f32, ptp, c_void_p, c_void_p, sz,
                                           c_void_p]
    lib.md_draft_attn_sparse_tp.argtypes = [pc, c_void_p, i32, c_void_p, i32, i32, f32, ptp, c_void_p, c_void_p, sz,
                                            c_void_p]
    lib.md_verify_attn_full_tp_append.argtypes = [pc, c_void_p, i32, i32, c_void_p, c_void_p, c_void_p, i32, f32,
                                                  ptp, c_void_p, c_void_p, sz, c_void_p]
    lib.md_draft_attn_sparse_tp_append.argtypes = [pc, c_void_p, i32, c_void_p, c_void_p, c_void_p, i32, i32, f32,
                                                   ptp, c_void_p, c_void_p, sz, c_void_p]
    lib.md_tp_barrier.argtypes = [psync, c_void_p]
    lib.md_philox_u32_dev.argtypes = [u64, c_void_p, i32, i32, c_void_p, c_void_p]
    lib.md_attn_workspace_bytes_det.argtypes = [i32, i32, i32, i32, i32, i32, i32]
    lib.md_attn_workspace_bytes_det.restype = sz
    lib.md_verify_attn_full_det.argtypes = [pc, c_void_p, i32, i32, c_void_p, i32, i32, f32, c_void_p, c_void_p,
                                            c_void_p, sz, c_void_p]
    lib.md_draft_attn_sparse_det.argtypes = [pc, c_void_p, i32, c_void_p, i32, i32, i32, f32, c_void_p, c_void_p,
                                             c_void_p, sz, c_void_p]
    lib.md_pq_encode.argtypes = [pc, c_void_p, c_void_p, i32, c_void_p, i32, c_void_p]
    lib.md_pq_workspace_bytes.argtypes = [i32, i32, i32]
    lib.md_pq_workspace_bytes.restype = sz
    lib.md_pq_select.argtypes = [c_void_p, i32, i32, i32, i32, c_void_p, c_void_p, i32, c_void_p, i32, i32, i32, i32,
                                 c_void_p, i32, c_void_p, c_void_p, c_void_p, sz, c_void_p]
    for name in ("md_kv_append", "md_verify_attn_full", "md_draft_attn_sparse", "md_draft_attn_indexed",
                 "md_snapkv_select", "md_philox_u32", "md_spec_accept", "md_debug_trace", "md_verify_attn_tree",
                 "md_spec_accept_tree", "md_kv_compact", "md_pq_encode", "md_pq_select", "md_verify_attn_full_tp",
                 "md_draft_attn_sparse_tp", "md_tp_barrier", "md_philox_u32_dev", "md_draft_attn_sparse_windows"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(status: int):
    if status != MD_OK:
        raise MDError(status, _lib.md_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("md tensors must be CUDA tensors (no CPU fallback)")
    return t.data_ptr()


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def make_cache(k: torch.Tensor, v: torch.Tensor) -> KVCache:
    """md_kv_cache from two [B, Hkv, cap, d] bf16 views (any strides with unit last stride)."""
    if k.shape != v.shape or k.stride() != v.stride() or k.dtype != torch.bfloat16 or v.dtype != torch.bfloat16:
        raise ValueError("k and v caches must be bf16 with identical shapes and strides")
    if k.dim() != 4 or k.stride(3) != 1:
        raise ValueError("cache must be [B, Hkv, cap, d] with unit stride on d")
    B, H, cap, d = k.shape
    return KVCache(_ptr(k), _ptr(v), B, H, d, cap, k.stride(0), k.stride(1), k.stride(2))


def abi_version() -> int:
    return load_library().md_abi_version()


def kv_append(k_cache, v_cache, k_new, v_new, start_pos, stream=None):
    """cache[b, h, start_pos[b] + t] = new[b, t, h] for K and V; new is [B, T, Hkv, d] contiguous
    (no temporary copies: the kernel reads the caller's tensors asynchronously on `stream`)."""
    _need_contiguous(k_new, v_new)
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    T = k_new.shape[1]
    _check(lib.md_kv_append(ctypes.byref(c), _ptr(k_new), _ptr(v_new), T, _ptr(start_pos), _stream(stream)))


def attn_workspace_bytes(batch, num_q_heads, num_kv_heads, head_dim, T, max_kv_len) -> int:
    return int(load_library().md_attn_workspace_bytes(batch, num_q_heads, num_kv_heads, head_dim, T, max_kv_len))


def _ws(workspace):
    if workspace is None:
        return None, 0
    return _ptr(workspace), workspace.numel() * workspace.element_size()


def verify_attn_full(q, k_cache, v_cache, kv_len, max_kv_len, scale, out, lse=None, workspace=None, stream=None):
    """q [B, T, Hq, d] bf16 -> out [B, T, Hq, d] fp32 (and lse [B, T, Hq] fp32)."""
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    ws, wsb = _ws(workspace)
    _check(lib.md_verify_attn_full(ctypes.byref(c), _ptr(q), q.shape[2], q.shape[1], _ptr(kv_len), int(max_kv_len),
                                   float(scale), _ptr(out), _ptr(lse), ws, wsb, _stream(stream)))


def attn_workspace_bytes_det(batch, num_q_heads, num_kv_heads, head_dim, T, max_keys, split_keys) -> int:
    return int(load_library().md_attn_workspace_bytes_det(batch, num_q_heads, num_kv_heads, head_dim, T, max_keys,
                                                          split_keys))


def verify_attn_full_det(q, k_cache, v_cache, kv_len, max_kv_len, split_keys, scale, out, lse=None, workspace=None,
                         stream=None):
    """verify_attn_full with the deterministic fixed-split plan (bits independent of the grid and
    of sharding); workspace from attn_workspace_bytes_det."""
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    ws, wsb = _ws(workspace)
    _check(lib.md_verify_attn_full_det(ctypes.byref(c), _ptr(q), q.shape[2], q.shape[1], _ptr(kv_len),
                                       int(max_kv_len), int(split_keys), float(scale), _ptr(out), _ptr(lse), ws, wsb,
                                       _stream(stream)))


def draft_attn_sparse_det(q, k_cache, v_cache, kv_len, sink, window, split_keys, scale, out, lse=None,
                          workspace=None, stream=None):
    """draft_attn_sparse with the deterministic fixed-split plan."""
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    ws, wsb = _ws(workspace)
    _check(lib.md_draft_attn_sparse_det(ctypes.byref(c), _ptr(q), q.shape[1], _ptr(kv_len), int(sink), int(window),
                                        int(split_keys), float(scale), _ptr(out), _ptr(lse), ws, wsb,
                                        _stream(stream)))


def verify_attn_tree(q, k_cache, v_cache, kv_len, max_kv_len, tree_mask, scale, out, lse=None, workspace=None,
                     stream=None):
    """Tree verify: q [B, T, Hq, d] bf16, tree_mask [B, T] (int32 storage of uint32; bit j of (b, t) =
    node t sees node j) -> out [B, T, Hq, d] fp32 (and lse [B, T, Hq])."""
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    ws, wsb = _ws(workspace)
    _check(lib.md_verify_attn_tree(ctypes.byref(c), _ptr(q), q.shape[2], q.shape[1], _ptr(kv_len), int(max_kv_len),
                                   _ptr(tree_mask), float(scale), _ptr(out), _ptr(lse), ws, wsb, _stream(stream)))


def draft_attn_sparse(q, k_cache, v_cache, kv_len, sink, window, scale, out, lse=None, workspace=None, stream=None,
                      windows=None):
    """q [B, Hq, d] bf16 over the sink + window rows -> out [B, Hq, d] fp32 (and lse [B, Hq]).
    windows: optional int32 [B] device tensor of per-sequence windows (each <= window)."""
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    ws, wsb = _ws(workspace)
    if windows is not None:
        _check(lib.md_draft_attn_sparse_windows(ctypes.byref(c), _ptr(q), q.shape[1], _ptr(kv_len), int(sink),
                                                int(window), _ptr(windows), float(scale), _ptr(out), _ptr(lse), ws,
                                                wsb, _stream(stream)))
        return
    _check(lib.md_draft_attn_sparse(ctypes.byref(c), _ptr(q), q.shape[1], _ptr(kv_len), int(sink), int(window),
                                    float(scale), _ptr(out), _ptr(lse), ws, wsb, _stream(stream)))


def _need_contiguous(*ts):
    for t in ts:
        if not t.is_contiguous():
            raise ValueError("k_new / v_new must be contiguous [B, T, Hkv, d]")


def verify_attn_full_append(q, k_cache, v_cache, k_new, v_new, kv_len, max_kv_len, scale, out, lse=None,
                            workspace=None, stream=None):
    """kv_append(k_new, v_new at kv_len - T) fused into verify_attn_full: one kernel launch.
    k_new / v_new [B, T, Hkv, d] bf16 contiguous."""
    _need_contiguous(k_new, v_new)
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    ws, wsb = _ws(workspace)
    _check(lib.md_verify_attn_full_append(ctypes.byref(c), _ptr(q), q.shape[2], q.shape[1], _ptr(k_new),
                                          _ptr(v_new), _ptr(kv_len), int(max_kv_len), float(scale), _ptr(out),
                                          _ptr(lse), ws, wsb, _stream(stream)))


MD_ATTN_EARLY_KV = 1


def draft_attn_sparse_append(q, k_cache, v_cache, k_new, v_new, kv_len, sink, window, scale, out, lse=None,
                             workspace=None, stream=None, early_kv=False):
    """kv_append(k_new, v_new at kv_len - 1) fused into draft_attn_sparse: one kernel launch.
    k_new / v_new [B, 1, Hkv, d] bf16 contiguous.  early_kv: md_draft_attn_sparse_append_ex with
    MD_ATTN_EARLY_KV (the caller's guarantee of the header: kv_len and the attended rows are not
    written by the md_* call just before this one on the stream)."""
    _need_contiguous(k_new, v_new)
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    ws, wsb = _ws(workspace)
    if early_kv:
        _check(lib.md_draft_attn_sparse_append_ex(ctypes.byref(c), _ptr(q), q.shape[1], _ptr(k_new), _ptr(v_new),
                                                  _ptr(kv_len), int(sink), int(window), float(scale), _ptr(out),
                                                  _ptr(lse), ws, wsb, MD_ATTN_EARLY_KV, _stream(stream)))
        return
    _check(lib.md_draft_attn_sparse_append(ctypes.byref(c), _ptr(q), q.shape[1], _ptr(k_new), _ptr(v_new),
                                           _ptr(kv_len), int(sink), int(window), float(scale), _ptr(out), _ptr(lse),
                                           ws, wsb, _stream(stream)))


def draft_attn_indexed(q, k_cache, v_cache, kv_len, idx, idx_count, tail_start, scale, out, lse=None,
                       workspace=None, stream=None, k_new=None, v_new=None):
    """SnapKV draft: q [B, Hq, d] over idx[b, u, :idx_count[b]] U [tail_start[b], kv_len[b]).
    idx is int32 [B, Hkv, K] (K % 4 == 0).  With k_new / v_new ([B, 1, Hkv, d]) the step's append
    at kv_len - 1 is fused in (md_draft_attn_indexed_append)."""
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    ws, wsb = _ws(workspace)
    if k_new is not None:
        _need_contiguous(k_new, v_new)
        _check(lib.md_draft_attn_indexed_append(ctypes.byref(c), _ptr(q), q.shape[1], _ptr(k_new), _ptr(v_new),
                                                _ptr(kv_len), _ptr(idx), idx.shape[2], _ptr(idx_count),
                                                _ptr(tail_start), float(scale), _ptr(out), _ptr(lse), ws, wsb,
                                                _stream(stream)))
        return
    _check(lib.md_draft_attn_indexed(ctypes.byref(c), _ptr(q), q.shape[1], _ptr(kv_len), _ptr(idx), idx.shape[2],
                                     _ptr(idx_count), _ptr(tail_start), float(scale), _ptr(out), _ptr(lse), ws, wsb,
                                     _stream(stream)))


def snapkv_workspace_bytes(batch, num_q_heads, num_kv_heads, w, max_prefill_len) -> int:
    return int(load_library().md_snapkv_workspace_bytes(batch, num_q_heads, num_kv_heads, w, max_prefill_len))


def snapkv_select(k_cache, v_cache, q_obs, prefill_len, max_prefill_len, w, budget, scale, idx, idx_count,
                  workspace=None, stream=None, budgets=None):
    """SnapKV selection at prefill: q_obs [B, w, Hq, d] bf16 -> idx [B, Hkv, K] int32 (ascending
    positions, K >= budget - w), idx_count [B] int32.  budgets: optional [B] int32 device tensor
    of per-sequence budgets (each clamped to [w, budget])."""
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    if workspace is None:
        workspace = torch.empty(snapkv_workspace_bytes(q_obs.shape[0], q_obs.shape[2], k_cache.shape[1], w,
                                                       max_prefill_len), dtype=torch.uint8, device=q_obs.device)
    ws, wsb = _ws(workspace)
    _check(lib.md_snapkv_select(ctypes.byref(c), _ptr(q_obs), q_obs.shape[2], _ptr(prefill_len), int(max_prefill_len),
                                int(w), int(budget), _ptr(budgets) if budgets is not None else None, float(scale),
                                _ptr(idx), idx.shape[2], _ptr(idx_count), ws, wsb,
                                _stream(stream)))


def pq_encode(k_cache, v_cache, codebook, start_pos, count, codes, stream=None):
    """PQ codes of cache rows [start_pos[b], start_pos[b] + count): codebook [B, Hkv, 16, 256, d/16] bf16,
    codes [B, Hkv, code_cap, 16] uint8."""
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    _check(lib.md_pq_encode(ctypes.byref(c), _ptr(codebook), _ptr(start_pos), int(count), _ptr(codes),
                            codes.shape[2], _stream(stream)))


def pq_workspace_bytes(batch, num_kv_heads, max_kv_len) -> int:
    return int(load_library().md_pq_workspace_bytes(batch, num_kv_heads, max_kv_len))


def pq_select(q, codebook, codes, kv_len, max_kv_len, sink, window, budget, idx, idx_count, tail_start,
              workspace=None, stream=None):
    """Dynamic PQ selection for the draft query q [B, Hq, d] bf16 -> idx [B, Hkv, K] int32 (sink rows then
    the top-`budget` candidates ascending; K >= sink + budget), idx_count [B], tail_start [B]."""
    lib = load_library()
    B, Hq, d = q.shape
    Hkv = codebook.shape[1]
    if workspace is None:
        workspace = torch.empty(pq_workspace_bytes(B, Hkv, max_kv_len), dtype=torch.uint8, device=q.device)
    ws, wsb = _ws(workspace)
    _check(lib.md_pq_select(_ptr(q), B, Hq, Hkv, d, _ptr(codebook), _ptr(codes), codes.shape[2], _ptr(kv_len),
                            int(max_kv_len), int(sink), int(window), int(budget), _ptr(idx), idx.shape[2],
                            _ptr(idx_count), _ptr(tail_start), ws, wsb, _stream(stream)))


def tp_out(out_peers_dev, world, rank) -> TPOut:
    """md_tp_out from an int64 CUDA tensor of device pointers (every rank's full-head buffer)."""
    return TPOut(_ptr(out_peers_dev), int(world), int(rank))


def tp_sync(flags_peers_dev, epoch_dev, world, rank) -> TPSync:
    return TPSync(_ptr(flags_peers_dev), _ptr(epoch_dev), int(world), int(rank))


def verify_attn_full_tp(q, k_cache, v_cache, kv_len, max_kv_len, scale, tp, lse=None, workspace=None, stream=None,
                        k_new=None, v_new=None):
    """Rank-local verify whose outputs land in every rank's [B, T, world*Hq, d] buffer (tp: TPOut).
    With k_new / v_new ([B, T, Hkv_local, d]) the rank's append is fused in (md_verify_attn_full_tp_append)."""
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    ws, wsb = _ws(workspace)
    if k_new is not None:
        _need_contiguous(k_new, v_new)
        _check(lib.md_verify_attn_full_tp_append(ctypes.byref(c), _ptr(q), q.shape[2], q.shape[1], _ptr(k_new),
                                                 _ptr(v_new), _ptr(kv_len), int(max_kv_len), float(scale),
                                                 ctypes.byref(tp), _ptr(lse), ws, wsb, _stream(stream)))
        return
    _check(lib.md_verify_attn_full_tp(ctypes.byref(c), _ptr(q), q.shape[2], q.shape[1], _ptr(kv_len),
                                      int(max_kv_len), float(scale), ctypes.byref(tp), _ptr(lse), ws, wsb,
                                      _stream(stream)))


def draft_attn_sparse_tp(q, k_cache, v_cache, kv_len, sink, window, scale, tp, lse=None, workspace=None, stream=None,
                         k_new=None, v_new=None):
    """Rank-local StreamingLLM draft whose outputs land in every rank's [B, world*Hq, d] buffer.
    With k_new / v_new ([B, 1, Hkv_local, d]) the rank's append is fused in (md_draft_attn_sparse_tp_append)."""
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    ws, wsb = _ws(workspace)
    if k_new is not None:
        _need_contiguous(k_new, v_new)
        _check(lib.md_draft_attn_sparse_tp_append(ctypes.byref(c), _ptr(q), q.shape[1], _ptr(k_new), _ptr(v_new),
                                                  _ptr(kv_len), int(sink), int(window), float(scale),
                                                  ctypes.byref(tp), _ptr(lse), ws, wsb, _stream(stream)))
        return
    _check(lib.md_draft_attn_sparse_tp(ctypes.byref(c), _ptr(q), q.shape[1], _ptr(kv_len), int(sink), int(window),
                                       float(scale), ctypes.byref(tp), _ptr(lse), ws, wsb, _stream(stream)))


def tp_barrier(sync, stream=None):
    """Completion barrier of the fused exchange (sync: TPSync)."""
    _check(load_library().md_tp_barrier(ctypes.byref(sync), _stream(stream)))


def philox_u32_dev(seed, step_dev, out, stream=None):
    """As philox_u32 with the step read from a device uint64 (int64 tensor of one element)."""
    lib = load_library()
    _check(lib.md_philox_u32_dev(int(seed) & (2**64 - 1), _ptr(step_dev), out.shape[0], out.shape[1], _ptr(out),
                                 _stream(stream)))


def philox_u32(seed, step, out, stream=None):
    """out [B, words] uint32 (torch.int32 storage) <- Philox4x32-10 words."""
    lib = load_library()
    _check(lib.md_philox_u32(int(seed) & (2**64 - 1), int(step) & (2**64 - 1), out.shape[0], out.shape[1],
                             _ptr(out), _stream(stream)))


def spec_accept(p, q, draft_tokens, rnd, out_tokens, num_accepted, committed_len=None, mode="sample",
                stream=None):
    """Batched acceptance.  p [B, gamma+1, V] fp32, q [B, gamma, V] fp32, draft_tokens [B, gamma] int32,
    rnd [B, gamma+2] (int32 storage of uint32) -> out_tokens [B, gamma+1], num_accepted [B]."""
    lib = load_library()
    B, G1, V = p.shape
    m = MD_ACCEPT_SAMPLE if mode == "sample" else MD_ACCEPT_GREEDY
    _check(lib.md_spec_accept(_ptr(p), _ptr(q), _ptr(draft_tokens), _ptr(rnd), B, G1 - 1, V, m, _ptr(out_tokens),
                              _ptr(num_accepted), _ptr(committed_len), _stream(stream)))


def spec_accept_tree(p, q, tokens, parent, rnd, out_tokens, num_accepted, accepted_nodes=None, committed_len=None,
                     mode="sample", stream=None):
    """Tree acceptance.  p, q [B, T, V] fp32 (distributions at each node), tokens / parent [B, T] int32,
    rnd [B, T+1] -> out_tokens [B, T], num_accepted [B], accepted_nodes [B, T]."""
    lib = load_library()
    B, T, V = p.shape
    m = MD_ACCEPT_SAMPLE if mode == "sample" else MD_ACCEPT_GREEDY
    _check(lib.md_spec_accept_tree(_ptr(p), _ptr(q), _ptr(tokens), _ptr(parent), _ptr(rnd), B, T, V, m,
                                   _ptr(out_tokens), _ptr(num_accepted), _ptr(accepted_nodes), _ptr(committed_len),
                                   _stream(stream)))


def kv_compact(k_cache, v_cache, base, nodes, count, stream=None):
    """cache[b, :, base[b] + 1 + i] = cache[b, :, base[b] + nodes[b, i]] for i < count[b]."""
    lib = load_library()
    c = make_cache(k_cache, v_cache)
    _check(lib.md_kv_compact(ctypes.byref(c), _ptr(base), _ptr(nodes), nodes.shape[1], _ptr(count),
                             _stream(stream)))


def debug_trace(buf=None):
    """Diagnostics: stamp per-CTA phase times of every attention call into buf (int64 [G, 16])."""
    lib = load_library()
    _check(lib.md_debug_trace(_ptr(buf), 0 if buf is None else buf.numel() * 8))
