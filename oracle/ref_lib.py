"""ctypes binding to oracle/_ref/libhybridsim_ref.so — TEST INFRASTRUCTURE ONLY.

The .so is the UNMODIFIED reference library (hybridsim) built from its own
sources by oracle/Makefile plus oracle/ref_shim.cpp. Used to pin the
restatement (hybridsim_oracle.py), to generate tests/golden fixtures, and as
bench.py's ``cpu_baseline`` (kind "reference").
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libhybridsim_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)


def available() -> bool:
    return os.path.exists(LIB_PATH)


_lib = None


def set_threads(n: int) -> int:
    """OpenMP threads of the reference library (0 = query); returns the count in effect."""
    return int(lib().ref_set_threads(int(n)))


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle` where /root/reference exists")
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_set_threads.restype = C.c_int
        L.ref_weights_new.argtypes = [C.c_int] * 6 + [C.c_uint64, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_weights_free.argtypes = [C.c_void_p]
        L.ref_weights_shape.argtypes = [C.c_void_p, C.c_int, C.c_int, _ip, _ip]
        L.ref_weights_get.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.ref_weights_set.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.ref_forward_prompt.argtypes = [C.c_void_p, _ip, C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        L.ref_generation_step.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_int,
                                          _dp, _dp, _dp]
        L.ref_recompute_kv.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, _dp, _dp]
        L.ref_token_recompute_kv.argtypes = [C.c_void_p, _ip, C.c_int, C.c_int, C.c_int, _dp, _dp]
        L.ref_attention_step.argtypes = [_dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.ref_project_ffn.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, _dp]
        L.ref_equivalence.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp, _ip]
        L.ref_flop_count.argtypes = [C.c_int, C.c_int, C.c_int, C.c_long, C.c_int, C.c_int]
        L.ref_flop_count.restype = C.c_double
        L.ref_cache_new.argtypes = [C.c_int, C.c_long, C.c_long, C.c_long, C.c_long, C.c_int]
        L.ref_cache_new.restype = C.c_void_p
        L.ref_cache_free.argtypes = [C.c_void_p]
        L.ref_cache_create_request.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
        L.ref_cache_append_block.argtypes = [C.c_void_p, C.c_char_p, C.c_int, _ip, _ip]
        L.ref_cache_fill_token.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_cache_free_request.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_cache_context_len.argtypes = [C.c_void_p, C.c_char_p, _ip]
        L.ref_cache_blocks_by_kind.argtypes = [C.c_void_p, C.c_char_p, _lp, _lp]
        L.ref_cache_free_blocks.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_cache_free_blocks.restype = C.c_long
        L.ref_cache_dump_json.argtypes = [C.c_void_p, C.c_char_p, C.c_long]
        L.ref_cache_dump_json.restype = C.c_long
        L.ref_bytes_of.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_bytes_of.restype = C.c_ulong
        L.ref_next_block_kind.argtypes = [C.c_long, C.c_long, C.c_long, C.c_long, _ip]
        L.ref_initial_cache_allocation.argtypes = [_dp, C.c_int, C.c_long, _lp]
        L.ref_alloc_remaining.argtypes = [_dp, _dp, C.c_int, C.c_long, C.c_long, _lp]
        L.ref_plan_host_allocation.argtypes = [_dp, _dp, C.c_int, C.c_long, _lp]
        L.ref_fit_linear.argtypes = [_dp, _dp, C.c_int, _dp]
        L.ref_model_preset.argtypes = [C.c_char_p, _ip]
        L.ref_parse_artifacts.argtypes = [C.c_char_p, C.c_char_p, _dp, _lp]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int) -> None:
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_ip)


def model_preset(name: str):
    """ModelConfig::preset (model.cpp:37-43) -> (layers, d, heads, ffn, vocab, tpb)."""
    out = (C.c_int * 6)()
    _check(lib().ref_model_preset(name.encode(), out))
    return tuple(out)


def parse_bundle(path: str):
    """TimingBundle::from_json (timing.cpp:155-163) of a bundle.json ->
    (kv slope, kv intercept, load slope, load intercept, t_load_w, s_weight_layer, s_weight_total)."""
    out = np.zeros(7)
    alloc = (C.c_long * 6)()
    with open(path) as fh:
        text = fh.read().encode()
    _check(lib().ref_parse_artifacts(text, None, dptr(out), alloc))
    return tuple(out)


class RefWeights:
    """DecoderWeights::generate on the reference, with get/set of tensors."""

    def __init__(self, layers, d, heads, ffn, vocab, tpb, seed, max_seq):
        self.h = C.c_void_p()
        _check(lib().ref_weights_new(layers, d, heads, ffn, vocab, tpb, seed, max_seq, C.byref(self.h)))
        self.layers, self.d = layers, d

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            lib().ref_weights_free(self.h)

    def _shape(self, which, layer):
        r, c = C.c_int(), C.c_int()
        _check(lib().ref_weights_shape(self.h, which, layer, C.byref(r), C.byref(c)))
        return r.value, c.value

    def get(self, which: int, layer: int = 0) -> np.ndarray:
        out = np.zeros(self._shape(which, layer))
        _check(lib().ref_weights_get(self.h, which, layer, dptr(out)))
        return out

    def set(self, which: int, layer: int, arr: np.ndarray) -> None:
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        assert arr.shape == self._shape(which, layer)
        _check(lib().ref_weights_set(self.h, which, layer, dptr(arr)))

    def forward_prompt(self, ids: Sequence[int], scaled=True):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        n, L, d = len(ids), self.layers, self.d
        ins, k, v, out = (np.zeros((L, n, d)), np.zeros((L, n, d)), np.zeros((L, n, d)),
                          np.zeros((n, d)))
        _check(lib().ref_forward_prompt(self.h, iptr(ids), n, int(scaled), dptr(ins), dptr(k),
                                        dptr(v), dptr(out)))
        return ins, k, v, out

    def generation_step(self, token, pos, ctx_k: np.ndarray, ctx_v: np.ndarray, scaled=True):
        ctx_k = np.ascontiguousarray(ctx_k, dtype=np.float64)
        ctx_v = np.ascontiguousarray(ctx_v, dtype=np.float64)
        L, ctx, d = ctx_k.shape
        out, nk, nv = np.zeros((1, d)), np.zeros((L, d)), np.zeros((L, d))
        _check(lib().ref_generation_step(self.h, token, pos, dptr(ctx_k), dptr(ctx_v), ctx,
                                         int(scaled), dptr(out), dptr(nk), dptr(nv)))
        return out, nk, nv

    def recompute_kv(self, layer: int, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        k, v = np.zeros_like(a), np.zeros_like(a)
        _check(lib().ref_recompute_kv(self.h, layer, dptr(a), a.shape[0], dptr(k), dptr(v)))
        return k, v

    def project_ffn(self, layer: int, att: np.ndarray):
        att = np.ascontiguousarray(att, dtype=np.float64)
        out = np.zeros_like(att)
        _check(lib().ref_project_ffn(self.h, layer, dptr(att), att.shape[0], dptr(out)))
        return out


def attention_step(q, k, v, heads, scaled=True):
    q = np.ascontiguousarray(q, dtype=np.float64).reshape(1, -1)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.zeros_like(q)
    _check(lib().ref_attention_step(dptr(q), dptr(k), dptr(v), k.shape[0], k.shape[1], heads,
                                    int(scaled), dptr(out)))
    return out


class RefCache:
    def __init__(self, tpb, kv_host=0, kv_gpu=0, act_host=0, act_gpu=0, kv_on_gpu=False):
        self.h = lib().ref_cache_new(tpb, kv_host, kv_gpu, act_host, act_gpu, int(kv_on_gpu))
        if not self.h:
            raise RefError(1, lib().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_cache_free(self.h)

    def create_request(self, rid: str, prompt_len: int):
        _check(lib().ref_cache_create_request(self.h, rid.encode(), prompt_len))

    def append_block(self, rid: str, kind: str):
        loc, pbn = C.c_int(), C.c_int()
        _check(lib().ref_cache_append_block(self.h, rid.encode(), 1 if kind == "ACT" else 0,
                                            C.byref(loc), C.byref(pbn)))
        return ("gpu" if loc.value else "host"), pbn.value

    def fill_token(self, rid: str):
        _check(lib().ref_cache_fill_token(self.h, rid.encode()))

    def free_request(self, rid: str):
        _check(lib().ref_cache_free_request(self.h, rid.encode()))

    def context_len(self, rid: str) -> int:
        n = C.c_int()
        _check(lib().ref_cache_context_len(self.h, rid.encode(), C.byref(n)))
        return n.value

    def blocks_by_kind(self, rid: str):
        a, k = C.c_long(), C.c_long()
        _check(lib().ref_cache_blocks_by_kind(self.h, rid.encode(), C.byref(a), C.byref(k)))
        return a.value, k.value

    def free_blocks(self, kind: str, loc: str) -> int:
        return lib().ref_cache_free_blocks(self.h, 1 if kind == "ACT" else 0, 1 if loc == "gpu" else 0)

    def dump_json(self) -> str:
        n = lib().ref_cache_dump_json(self.h, None, 0)
        buf = C.create_string_buffer(n)
        lib().ref_cache_dump_json(self.h, buf, n)
        return buf.value.decode()


def next_block_kind(act_req, kv_req, act_host, kv_host) -> str:
    k = C.c_int()
    _check(lib().ref_next_block_kind(act_req, kv_req, act_host, kv_host, C.byref(k)))
    return "ACT" if k.value else "KV"


def _bundle_arr(b) -> np.ndarray:
    return np.array([b[0], b[1], b[2], b[3], b[4]], dtype=np.float64)


def plan_host_allocation(bundle5, mem4, tpb, act_gpu) -> List[int]:
    out = (C.c_long * 6)()
    b, m = _bundle_arr(bundle5), np.asarray(mem4, dtype=np.float64)
    _check(lib().ref_plan_host_allocation(dptr(b), dptr(m), tpb, act_gpu, out))
    return list(out)


def initial_cache_allocation(bundle5, tpb, act_gpu):
    out = (C.c_long * 2)()
    b = _bundle_arr(bundle5)
    _check(lib().ref_initial_cache_allocation(dptr(b), tpb, act_gpu, out))
    return tuple(out)


def alloc_remaining(bundle5, mem4, tpb, act_init, kv_init):
    out = (C.c_long * 2)()
    b, m = _bundle_arr(bundle5), np.asarray(mem4, dtype=np.float64)
    _check(lib().ref_alloc_remaining(dptr(b), dptr(m), tpb, act_init, kv_init, out))
    return tuple(out)


def fit_linear(xs, ys):
    x = np.ascontiguousarray(xs, dtype=np.float64)
    y = np.ascontiguousarray(ys, dtype=np.float64)
    out = np.zeros(4)
    _check(lib().ref_fit_linear(dptr(x), dptr(y), len(x), dptr(out)))
    return out


def equivalence(seed, fault=False, scaled=True):
    dev, ex = C.c_double(), C.c_int()
    _check(lib().ref_equivalence(seed, int(fault), int(scaled), C.byref(dev), C.byref(ex)))
    return dev.value, bool(ex.value)
