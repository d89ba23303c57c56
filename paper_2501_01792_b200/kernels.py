"""Kernel-level calls through the C ABI (host numpy buffers in / out).

fp16 (IEEE binary16) tensors cross the boundary as uint16 bit patterns.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from ._native import check, lib, ptr


def f32_to_f16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> IEEE binary16 bits (fp64 inputs go via fp32)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    return f.astype(np.float16).view(np.uint16)


def f16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(b, dtype=np.uint16).view(np.float16).astype(np.float32)


def _u16(a):
    a = np.ascontiguousarray(a, dtype=np.uint16)
    return a, ptr(a, C.c_uint16)


def gemm_f16(a_bits: np.ndarray, wt_bits: np.ndarray, epi: int = 0, bn: int = 0) -> np.ndarray:
    """C = A . W with W passed transposed (Wt [N x K]); epi 0 f16, 1 relu, 3 f32."""
    M, K = a_bits.shape
    N, K2 = wt_bits.shape
    assert K == K2
    a, ap = _u16(a_bits)
    w, wp = _u16(wt_bits)
    out = np.zeros((M, N), dtype=np.float32 if epi == 3 else np.uint16)
    check(lib().hc_gemm_f16(epi, M, N, K, ap, wp, out.ctypes.data_as(C.c_void_p), bn))
    return out


def gemm_f16_splitk(a_bits: np.ndarray, wt_bits: np.ndarray, splits: int, epi: int = 0, bn: int = 128) -> np.ndarray:
    """Split-K C = A . W (W transposed [N x K]); f16 out (epi 0 store, 1 relu)."""
    M, K = a_bits.shape
    N, _ = wt_bits.shape
    a, ap = _u16(a_bits)
    w, wp = _u16(wt_bits)
    out = np.zeros((M, N), np.uint16)
    check(lib().hc_gemm_f16_splitk(epi, M, N, K, ap, wp, ptr(out, C.c_uint16), bn, splits))
    return out


def gemm_f16_wstream(a_bits: np.ndarray, wt_bits: np.ndarray, epi: int = 0, bias_bits=None, res_bits=None,
                     ctas: int = 0) -> np.ndarray:
    """Weight-streaming decode GEMM (swap-AB stream-K, M <= 256): C = A . W
    (+ bias[n]) (+ res[m][n]), relu for epi 1, fp32 for epi 3; `ctas` CTAs
    share the k-block iterations (0 = one per SM)."""
    M, K = a_bits.shape
    N, _ = wt_bits.shape
    a, ap = _u16(a_bits)
    w, wp = _u16(wt_bits)
    bp = rp = None
    if bias_bits is not None:
        b, bp = _u16(bias_bits)
    if res_bits is not None:
        r, rp = _u16(res_bits)
    out = np.zeros((M, N), dtype=np.float32 if epi == 3 else np.uint16)
    check(lib().hc_gemm_f16_wstream(epi, M, N, K, ap, wp, bp, rp, out.ctypes.data_as(C.c_void_p), ctas))
    return out


def recompute_kv_paged(act_pool_bits: np.ndarray, wkv_t_bits: np.ndarray, heads: int,
                       tiles: np.ndarray, bn: int = 0) -> np.ndarray:
    """act_pool [n_blocks, tpb, d] -> kv [n_blocks, 2, H, tpb, hd] (f16 bits)."""
    nb, tpb, d = act_pool_bits.shape
    a, ap = _u16(act_pool_bits)
    w, wp = _u16(wkv_t_bits)
    t = np.ascontiguousarray(tiles, dtype=np.int32)
    out = np.zeros((nb, 2, heads, tpb, d // heads), dtype=np.uint16)
    check(lib().hc_recompute_kv_paged(nb, tpb, d, heads, ap, wp, ptr(t, C.c_int), len(t),
                                      ptr(out, C.c_uint16), bn))
    return out


def decode_attention(q_bits, region0, region1, blk_ref, n_blocks, ctx_len, heads, scaled=True,
                     splits=0):
    B, d = q_bits.shape
    n0, _, H, tpb, hd = region0.shape
    n1 = region1.shape[0]
    q, qp = _u16(q_bits)
    r0, r0p = _u16(region0)
    r1, r1p = _u16(region1)
    ref = np.ascontiguousarray(blk_ref, dtype=np.int32)
    nb = np.ascontiguousarray(n_blocks, dtype=np.int32)
    cl = np.ascontiguousarray(ctx_len, dtype=np.int32)
    out = np.zeros((B, d), dtype=np.uint16)
    check(lib().hc_decode_attention(B, H, hd, tpb, qp, r0p, n0, r1p, n1, ptr(ref, C.c_int), ref.shape[1],
                                    ptr(nb, C.c_int), ptr(cl, C.c_int), int(scaled), splits,
                                    ptr(out, C.c_uint16)))
    return out


def prefill_attention(qkv_bits, n_req, P, heads, scaled=True):
    rows, d3 = qkv_bits.shape
    d = d3 // 3
    q, qp = _u16(qkv_bits)
    out = np.zeros((rows, d), dtype=np.uint16)
    check(lib().hc_prefill_attention(n_req, P, heads, d // heads, qp, int(scaled), ptr(out, C.c_uint16)))
    return out


def device_count() -> int:
    return lib().hc_device_count()


def device_pci_bus_id(device: int) -> str:
    buf = C.create_string_buffer(64)
    check(lib().hc_device_pci_bus_id(device, buf, 64))
    return buf.value.decode()
