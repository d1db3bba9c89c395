"""ctypes binding of synth/libmd_synth.so, the GPU twin of the numpy generators in
synth/__init__.py (inputs only; bit-identical, checked by tests/test_gpu_synth.py)."""
from __future__ import annotations

import ctypes
import os

import torch

from . import T_KCACHE, Regime, FLAT

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmd_synth.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing: run `python -m paper_2408_11049_b200.build`")
        _lib = ctypes.CDLL(_LIB)
        ll, i = ctypes.c_longlong, ctypes.c_int
        _lib.mds_fill_cache.argtypes = [ctypes.c_void_p, i, i, i, ll, ll, ll, i, i, ctypes.c_ulonglong, i, i, i, i,
                                        i, ctypes.c_void_p]
        _lib.mds_fill_q.argtypes = [ctypes.c_void_p, i, i, i, i, i, ctypes.c_ulonglong, i, i, i, ctypes.c_void_p]
        _lib.mds_fill_cache_offgrid.argtypes = [ctypes.c_void_p, i, i, i, ll, ll, ll, i, i, ctypes.c_ulonglong, i, i,
                                                i, i, ctypes.c_void_p]
        _lib.mds_fill_flat_offgrid.argtypes = [ctypes.c_void_p, ll, ctypes.c_ulonglong, i, ctypes.c_void_p]
        _lib.mds_fill_cache_slice.argtypes = [ctypes.c_void_p, i, i, i, ll, ll, ll, i, i, ctypes.c_ulonglong, i, i, i,
                                              i, i, i, i, i, ctypes.c_void_p]
    return _lib


def fill_cache(x: torch.Tensor, seed: int, tensor: int, pos0: int, npos: int, regime: Regime = FLAT,
               b0: int = 0, h0: int = 0, Hkv_total: int | None = None):
    """x: [B, Hkv, cap, d] bf16 view; fills rows [pos0, pos0 + npos) like synth.kv_cache_k.
    (b0, h0, Hkv_total): x is the slice [b0, b0 + B) x [h0, h0 + Hkv) of a cache with Hkv_total
    KV heads (a tensor-parallel / batch shard gets exactly the full cache's values)."""
    B, H, cap, d = x.shape
    assert x.dtype == torch.bfloat16 and x.stride(3) == 1 and pos0 + npos <= cap
    s = torch.cuda.current_stream().cuda_stream
    rc = _load().mds_fill_cache_slice(x.data_ptr(), B, H, d, x.stride(0), x.stride(1), x.stride(2), pos0, npos, seed,
                                      tensor, int(regime.kind == "peaky" and tensor == T_KCACHE), regime.sink,
                                      regime.a_k, regime.needle_period, b0, h0, H if Hkv_total is None else Hkv_total,
                                      s)
    if rc:
        raise RuntimeError(f"mds_fill_cache failed: {rc}")


def fill_q(x: torch.Tensor, seed: int, tensor: int, Hkv: int, regime: Regime = FLAT):
    """x: contiguous [B, T, Hq, d] (or [B, Hq, d] for T = 1) bf16, like synth.q_rows_k."""
    assert x.dtype == torch.bfloat16 and x.is_contiguous()
    if x.dim() == 3:
        B, Hq, d = x.shape
        T = 1
    else:
        B, T, Hq, d = x.shape
    s = torch.cuda.current_stream().cuda_stream
    rc = _load().mds_fill_q(x.data_ptr(), B, T, Hq, Hkv, d, seed, tensor, int(regime.kind == "peaky"), regime.a_q, s)
    if rc:
        raise RuntimeError(f"mds_fill_q failed: {rc}")


def fill_new_kv(x: torch.Tensor, seed: int, tensor: int):
    """x: contiguous [B, T, Hkv, d] bf16, like synth.new_kv_k."""
    B, T, H, d = x.shape
    s = torch.cuda.current_stream().cuda_stream
    rc = _load().mds_fill_q(x.data_ptr(), B, T, H, H, d, seed, tensor, 0, 0, s)
    if rc:
        raise RuntimeError(f"mds_fill_q failed: {rc}")


def fill_cache_offgrid(x: torch.Tensor, seed: int, tensor: int, pos0: int, npos: int, b0: int = 0, h0: int = 0,
                       Hkv_total: int | None = None):
    """Off-grid twin of synth.kv_cache_bits_offgrid for rows [pos0, pos0 + npos) of x [B, Hkv, cap, d]."""
    B, H, cap, d = x.shape
    assert x.dtype == torch.bfloat16 and x.stride(3) == 1 and pos0 + npos <= cap
    rc = _load().mds_fill_cache_offgrid(x.data_ptr(), B, H, d, x.stride(0), x.stride(1), x.stride(2), pos0, npos,
                                        seed, tensor, b0, h0, H if Hkv_total is None else Hkv_total,
                                        torch.cuda.current_stream().cuda_stream)
    if rc:
        raise RuntimeError(f"mds_fill_cache_offgrid failed: {rc}")


def fill_flat_offgrid(x: torch.Tensor, seed: int, tensor: int):
    """Off-grid twin of synth.flat_bits_offgrid for a contiguous bf16 tensor."""
    assert x.dtype == torch.bfloat16 and x.is_contiguous()
    rc = _load().mds_fill_flat_offgrid(x.data_ptr(), x.numel(), seed, tensor, torch.cuda.current_stream().cuda_stream)
    if rc:
        raise RuntimeError(f"mds_fill_flat_offgrid failed: {rc}")
