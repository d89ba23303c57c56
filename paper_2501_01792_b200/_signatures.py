"""ctypes signatures of every symbol declared in include/hybridcache.h.

tests/test_abi.py checks that this table and the header agree and that the
built library exports every symbol.
"""
import ctypes as C

i, l, d, u64, vp, cp = C.c_int, C.c_long, C.c_double, C.c_uint64, C.c_void_p, C.c_char_p
ip, lp, dp, u16p = C.POINTER(C.c_int), C.POINTER(C.c_long), C.POINTER(C.c_double), C.POINTER(C.c_uint16)
vpp = C.POINTER(C.c_void_p)

SIGNATURES = {
    # library
    "hc_last_error": (cp, []),
    "hc_abi_version": (i, []),
    "hc_device_count": (i, []),
    "hc_set_device": (i, [i]),
    # kernels (host buffers in / out)
    "hc_gemm_bf16": (i, [i, i, i, i, u16p, u16p, vp, i]),
    "hc_recompute_kv_paged": (i, [i, i, i, i, u16p, u16p, ip, i, u16p, i]),
    "hc_decode_attention": (i, [i, i, i, i, u16p, u16p, l, u16p, l, ip, i, ip, ip, i, i, u16p]),
    "hc_prefill_attention": (i, [i, i, i, i, u16p, i, u16p]),
}
