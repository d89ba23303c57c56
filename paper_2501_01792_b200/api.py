"""Python mirror of the reference engine API (hybridsim, /root/reference/proj),
backed by the C ABI of libhybridcache_b200.so.

Same names, argument meaning and error behaviour as the reference's C++
headers: model.hpp (ModelConfig, generate), cache.hpp (HybridCache, block
tables, bytes_of), plan.hpp / timing.hpp (next_block_kind, planner, fits),
flops.hpp (flop_count) — plus the B200 Engine (prefill / decode-step calls
over the hybrid cache). Errors raise InputError / CapacityError / ConfigError
exactly where the reference throws them.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from ._native import check, lib, ptr
from .errors import CapacityError, ConfigError, InputError  # noqa: F401  (re-exported)
from ._signatures import EngineOptionsC, ModelConfigC
from .errors import InputError


class BlockKind(IntEnum):
    KV = 0
    ACT = 1

    def __str__(self):
        return self.name


class Location(IntEnum):
    HostMem = 0
    GpuMem = 1

    def __str__(self):
        return "host" if self == Location.HostMem else "gpu"


# ----------------------------------------------------------------- model ---
@dataclass
class ModelConfig:
    """model.hpp:15-36"""
    name: str = "custom"
    num_layers: int = 1
    hidden_dim: int = 64
    num_heads: int = 1
    ffn_dim: int = 0
    vocab_size: int = 256
    tokens_per_block: int = 16
    bytes_per_scalar: int = 2
    seed: int = 0

    @property
    def head_dim(self) -> int:
        return self.hidden_dim // self.num_heads

    def to_c(self) -> ModelConfigC:
        return ModelConfigC(self.num_layers, self.hidden_dim, self.num_heads, self.ffn_dim, self.vocab_size,
                            self.tokens_per_block, self.bytes_per_scalar)

    def validate(self) -> "ModelConfig":
        c = self.to_c()
        check(lib().hc_model_validate(C.byref(c)))
        self.ffn_dim = c.ffn_dim
        return self

    @classmethod
    def preset(cls, name: str) -> "ModelConfig":
        c = ModelConfigC()
        check(lib().hc_model_preset(name.encode(), C.byref(c)))
        return cls(name, c.num_layers, c.hidden_dim, c.num_heads, c.ffn_dim, c.vocab_size,
                   c.tokens_per_block, c.bytes_per_scalar)

    @staticmethod
    def preset_names() -> List[str]:
        return ["opt-6.7b", "opt-13b", "opt-30b", "opt-66b"]


def generate_weights(cfg: ModelConfig, seed: int, max_seq: int, rescale: bool = True) -> Dict[str, np.ndarray]:
    """DecoderWeights::generate (+ rescale, fp16) in device layout (fp16 bits):
    embedding [V,d], positional [S,d], layers [L, layer_elems] packed as
    Wqkv^T [3d,d] | Wproj^T [d,d] | W1^T [f,d] | W2^T [d,f]."""
    cfg = ModelConfig(**cfg.__dict__).validate()
    d, f, V, L = cfg.hidden_dim, cfg.ffn_dim, cfg.vocab_size, cfg.num_layers
    le = 4 * d * d + 2 * d * f
    emb = np.zeros((V, d), np.uint16)
    pos = np.zeros((max_seq, d), np.uint16)
    layers = np.zeros((L, le), np.uint16)
    c = cfg.to_c()
    check(lib().hc_generate_weights(C.byref(c), seed, max_seq, int(rescale), ptr(emb, C.c_uint16),
                                    ptr(pos, C.c_uint16), ptr(layers, C.c_uint16)))
    return {"embedding": emb, "positional": pos, "layers": layers}


def unpack_layer(cfg: ModelConfig, packed: np.ndarray) -> Dict[str, np.ndarray]:
    """Split one packed layer into reference-layout [in x out] matrices."""
    d, f = cfg.hidden_dim, cfg.ffn_dim
    o = 0
    wqkv = packed[o:o + 3 * d * d].reshape(3 * d, d); o += 3 * d * d
    wproj = packed[o:o + d * d].reshape(d, d); o += d * d
    w1 = packed[o:o + f * d].reshape(f, d); o += f * d
    w2 = packed[o:o + d * f].reshape(d, f)
    return {"w_q": wqkv[:d].T, "w_k": wqkv[d:2 * d].T, "w_v": wqkv[2 * d:].T, "w_proj": wproj.T,
            "w_ffn1": w1.T, "w_ffn2": w2.T}


# ----------------------------------------------------------------- cache ---
@dataclass
class BlockTableEntry:
    kind: BlockKind
    location: Location
    pbn: int
    filled_tokens: int = 0


@dataclass
class BlockTable:
    request_id: str
    prompt_len: int
    entries: List[BlockTableEntry] = field(default_factory=list)

    def context_len(self) -> int:
        return sum(e.filled_tokens for e in self.entries)

    def blocks_by_kind(self) -> Tuple[int, int]:
        a = sum(1 for e in self.entries if e.kind == BlockKind.ACT)
        return a, len(self.entries) - a


@dataclass
class PoolCaps:
    kv_host: int = 0
    kv_gpu: int = 0
    act_host: int = 0
    act_gpu: int = 0


def _kind(k) -> int:
    if isinstance(k, str):
        return 1 if k.upper() == "ACT" else 0
    return int(k)


def _loc(l) -> int:
    if isinstance(l, str):
        return 1 if l.lower() == "gpu" else 0
    return int(l)


class HybridCache:
    """cache.hpp:49-95 — bit-exact block bookkeeping (C++ host code)."""

    def __init__(self, tokens_per_block: int, caps: Optional[PoolCaps] = None, kv_on_gpu: bool = False,
                 *, _borrowed: Optional[C.c_void_p] = None, _owner=None):
        self._owner = _owner
        if _borrowed is not None:
            self._h, self._own = _borrowed, False
            return
        caps = caps or PoolCaps()
        h = C.c_void_p()
        check(lib().hc_cache_create(tokens_per_block, caps.kv_host, caps.kv_gpu, caps.act_host, caps.act_gpu,
                                    int(kv_on_gpu), C.byref(h)))
        self._h, self._own = h, True

    def __del__(self):
        if getattr(self, "_own", False) and self._h:
            lib().hc_cache_destroy(self._h)
            self._h = None

    def create_request(self, rid: str, prompt_len: int) -> None:
        check(lib().hc_cache_create_request(self._h, rid.encode(), prompt_len))

    def append_block(self, rid: str, kind) -> BlockTableEntry:
        loc, pbn = C.c_int(), C.c_int()
        check(lib().hc_cache_append_block(self._h, rid.encode(), _kind(kind), C.byref(loc), C.byref(pbn)))
        return BlockTableEntry(BlockKind(_kind(kind)), Location(loc.value), pbn.value, 0)

    def fill_token(self, rid: str) -> None:
        check(lib().hc_cache_fill_token(self._h, rid.encode()))

    def free_request(self, rid: str) -> None:
        check(lib().hc_cache_free_request(self._h, rid.encode()))

    def blocks_by_kind(self, rid: str) -> Tuple[int, int]:
        a, k = C.c_long(), C.c_long()
        check(lib().hc_cache_blocks_by_kind(self._h, rid.encode(), C.byref(a), C.byref(k)))
        return a.value, k.value

    def context_len(self, rid: str) -> int:
        n = C.c_int()
        check(lib().hc_cache_context_len(self._h, rid.encode(), C.byref(n)))
        return n.value

    def table(self, rid: str) -> BlockTable:
        n = C.c_int()
        check(lib().hc_cache_table(self._h, rid.encode(), None, None, None, None, 0, C.byref(n)))
        k, lo, p, f = (np.zeros(n.value, np.int32) for _ in range(4))
        check(lib().hc_cache_table(self._h, rid.encode(), ptr(k, C.c_int), ptr(lo, C.c_int), ptr(p, C.c_int),
                                   ptr(f, C.c_int), n.value, C.byref(n)))
        doc = json.loads(self.dump_json())
        plen = next(r["prompt_len"] for r in doc["requests"] if r["id"] == rid)
        return BlockTable(rid, plen, [BlockTableEntry(BlockKind(int(a)), Location(int(b)), int(c), int(d))
                                      for a, b, c, d in zip(k, lo, p, f)])

    def free_blocks(self, kind, loc) -> int:
        out = C.c_long()
        check(lib().hc_cache_free_blocks(self._h, _kind(kind), _loc(loc), C.byref(out)))
        return out.value

    def capacity(self, kind, loc) -> int:
        out = C.c_long()
        check(lib().hc_cache_capacity(self._h, _kind(kind), _loc(loc), C.byref(out)))
        return out.value

    def dump_json(self) -> str:
        need = C.c_long()
        check(lib().hc_cache_dump_json(self._h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        check(lib().hc_cache_dump_json(self._h, buf, need.value, C.byref(need)))
        return buf.value.decode()

    @staticmethod
    def bytes_of(kind, cfg: ModelConfig) -> int:
        out = C.c_uint64()
        check(lib().hc_bytes_of(_kind(kind), cfg.hidden_dim, cfg.tokens_per_block, cfg.bytes_per_scalar,
                                C.byref(out)))
        return out.value


# --------------------------------------------------------------- planner ---
@dataclass
class HostAllocation:
    """plan.hpp:17-25"""
    act_host: int = 0
    kv_host: int = 0
    act_init: int = 0
    kv_init: int = 0
    act_remain: int = 0
    kv_remain: int = 0


def next_block_kind(act_req: int, kv_req: int, allocation: HostAllocation) -> BlockKind:
    """plan.cpp:154-164 — the hybrid-ratio setting."""
    k = C.c_int()
    check(lib().hc_next_block_kind(act_req, kv_req, allocation.act_host, allocation.kv_host, C.byref(k)))
    return BlockKind(k.value)


@dataclass
class LinearTimeModel:
    slope: float = 0.0
    intercept: float = 0.0
    r_squared: float = 0.0
    intercept_clamped: bool = False


def _darr(x):
    a = np.ascontiguousarray(x, dtype=np.float64)
    return a, ptr(a, C.c_double)


def fit_linear(samples: Sequence[Tuple[float, float]]) -> LinearTimeModel:
    """timing.cpp:38-73"""
    xs, xp = _darr([s[0] for s in samples])
    ys, yp = _darr([s[1] for s in samples])
    out, op = _darr(np.zeros(4))
    check(lib().hc_fit_linear(xp, yp, len(xs), op))
    return LinearTimeModel(out[0], out[1], out[2], bool(out[3]))


@dataclass
class TimingBundle:
    t_kv_gen: LinearTimeModel
    t_load_kv: LinearTimeModel
    t_load_w: float = 0.0
    s_weight_layer: int = 0
    s_weight_total: int = 0

    def arr5(self):
        return _darr([self.t_kv_gen.slope, self.t_kv_gen.intercept, self.t_load_kv.slope,
                      self.t_load_kv.intercept, self.t_load_w])


@dataclass
class MemoryBudget:
    m_host: float = 0.0
    s_weight: float = 0.0
    s_kv_block: float = 0.0
    s_act_block: float = 0.0

    def arr4(self):
        return _darr([self.m_host, self.s_weight, self.s_kv_block, self.s_act_block])


def bundle_from_samples(kv_gen: Sequence[Tuple[float, float]], load_kv: Sequence[Tuple[float, float]],
                        link_bytes_per_s: float, cfg: ModelConfig) -> TimingBundle:
    """timing.cpp:172-183, fed by measured B200 samples."""
    kn, knp = _darr([s[0] for s in kv_gen])
    ks, ksp = _darr([s[1] for s in kv_gen])
    ln, lnp = _darr([s[0] for s in load_kv])
    ls, lsp = _darr([s[1] for s in load_kv])
    out, op = _darr(np.zeros(11))
    c = cfg.to_c()
    check(lib().hc_bundle_from_samples(knp, ksp, len(kn), lnp, lsp, len(ln), link_bytes_per_s, C.byref(c), op))
    return TimingBundle(LinearTimeModel(out[0], out[1], out[2], bool(out[3])),
                        LinearTimeModel(out[4], out[5], out[6], bool(out[7])), out[8], int(out[9]), int(out[10]))


def budget_for(host_mem: float, cfg: ModelConfig, bundle: TimingBundle) -> MemoryBudget:
    out, op = _darr(np.zeros(4))
    c = cfg.to_c()
    check(lib().hc_budget_for(host_mem, C.byref(c), float(bundle.s_weight_total), op))
    return MemoryBudget(*out)


def initial_cache_allocation(bundle: TimingBundle, tpb: int, act_gpu: int) -> Tuple[int, int]:
    b, bp = bundle.arr5()
    out = (C.c_long * 2)()
    check(lib().hc_initial_cache_allocation(bp, tpb, act_gpu, out))
    return out[0], out[1]


def alloc_remaining(bundle: TimingBundle, mem: MemoryBudget, tpb: int, act_init: int, kv_init: int):
    b, bp = bundle.arr5()
    m, mp = mem.arr4()
    out = (C.c_long * 2)()
    check(lib().hc_alloc_remaining(bp, mp, tpb, act_init, kv_init, out))
    return out[0], out[1]


def plan_hbm_residency(cfg: ModelConfig, requests: int, blocks_per_request: int, hbm_bytes: float):
    """B200 extension of Alg. 1 (csrc/host/plan.hpp): (r, PoolCaps) for a cache placed in
    HBM first — the smallest ACT share whose blocks fit, the rest in pinned host memory."""
    c = cfg.to_c()
    r = C.c_double()
    out = (C.c_long * 4)()
    check(lib().hc_plan_hbm_residency(C.byref(c), requests, blocks_per_request, float(hbm_bytes), C.byref(r), out))
    return r.value, PoolCaps(kv_host=out[3], kv_gpu=out[1], act_host=out[2], act_gpu=out[0])


def plan_hbm_tiers(cfg: ModelConfig, requests: int, blocks_per_request: int, hbm_bytes: float,
                   bundle: TimingBundle, host_bytes: float = 0.0, weights_streamed: bool = False):
    """Balanced three-tier plan (csrc/host/plan.hpp): (r, PoolCaps, (t_comp, t_link) per layer).
    host_bytes bounds the pinned host tiers (0 = unbounded); weights_streamed adds
    the per-layer weight stream (bundle.t_load_w) to the link side."""
    c = cfg.to_c()
    b, bp = bundle.arr5()
    r = C.c_double()
    out = (C.c_long * 4)()
    t, tp = _darr(np.zeros(2))
    check(lib().hc_plan_hbm_tiers(C.byref(c), requests, blocks_per_request, float(hbm_bytes), float(host_bytes), bp,
                                  int(weights_streamed), C.byref(r), out, tp))
    return r.value, PoolCaps(kv_host=out[3], kv_gpu=out[1], act_host=out[2], act_gpu=out[0]), tuple(t.tolist())


def plan_host_min_step(cfg: ModelConfig, requests: int, blocks_per_request: int, bundle: TimingBundle,
                       host_bytes: float = 0.0):
    """Host-only plan minimising the predicted step (csrc/host/plan.hpp): Alg. 1's
    cost model plus the ACT blocks' own link time. Returns (r, PoolCaps with the
    host tiers, (t_comp, t_link) per layer)."""
    c = cfg.to_c()
    b, bp = bundle.arr5()
    r = C.c_double()
    out = (C.c_long * 2)()
    t, tp = _darr(np.zeros(2))
    check(lib().hc_plan_host_min_step(C.byref(c), requests, blocks_per_request, float(host_bytes), bp, C.byref(r),
                                      out, tp))
    return r.value, PoolCaps(act_host=out[0], kv_host=out[1]), tuple(t.tolist())


def plan_host_allocation(bundle: TimingBundle, mem: MemoryBudget, tpb: int, act_gpu: int) -> HostAllocation:
    """plan.cpp:106-152 (paper Alg. 1 + frontier polish)."""
    b, bp = bundle.arr5()
    m, mp = mem.arr4()
    out = (C.c_long * 6)()
    check(lib().hc_plan_host_allocation(bp, mp, tpb, act_gpu, out))
    return HostAllocation(*list(out))


def planned_t_pcie(bundle: TimingBundle, tpb: int, a: HostAllocation) -> float:
    b, bp = bundle.arr5()
    out, op = _darr(np.zeros(2))
    check(lib().hc_planned_times(bp, tpb, a.act_host, a.kv_host, 0, op))
    return float(out[0])


def planned_t_computation(bundle: TimingBundle, tpb: int, a: HostAllocation, act_gpu: int) -> float:
    b, bp = bundle.arr5()
    out, op = _darr(np.zeros(2))
    check(lib().hc_planned_times(bp, tpb, a.act_host, a.kv_host, act_gpu, op))
    return float(out[1])


@dataclass
class MiniBatch:
    ids: List[str]
    act_mb: int = 0
    kv_mb: int = 0


def form_minibatches(requests: Sequence[Tuple[str, int, int]], act_max: int, kv_max: int, bundle: TimingBundle,
                     tpb: int) -> List[MiniBatch]:
    """form_minibatches (minibatch.cpp:36-83): requests = [(id, act_blocks, kv_blocks)]."""
    n = len(requests)
    ids = (C.c_char_p * max(n, 1))(*[r[0].encode() for r in requests])
    act = (C.c_long * max(n, 1))(*[r[1] for r in requests])
    kv = (C.c_long * max(n, 1))(*[r[2] for r in requests])
    order = (C.c_int * max(n, 1))()
    bof = (C.c_int * max(n, 1))()
    nb = C.c_int()
    b, bp = bundle.arr5()
    check(lib().hc_form_minibatches(n, ids, act, kv, act_max, kv_max, bp, tpb, order, bof, C.byref(nb)))
    out = [MiniBatch([]) for _ in range(nb.value)]
    for k in range(n):
        i = order[k]
        mb = out[bof[i]]
        mb.ids.append(requests[i][0])
        mb.act_mb += requests[i][1]
        mb.kv_mb += requests[i][2]
    return out


def cost_fb(act_mb: int, kv_mb: int, bundle: TimingBundle, tpb: int) -> Tuple[float, float]:
    """(balance, F_b) of minibatch.cpp:10-23."""
    b, bp = bundle.arr5()
    out, op = _darr(np.zeros(2))
    check(lib().hc_cost_fb(act_mb, kv_mb, bp, tpb, op))
    return float(out[0]), float(out[1])


def default_packer(gpu_mem_bytes: float, cfg: ModelConfig) -> Tuple[int, int]:
    """default_packer (sim.cpp:122-132) -> (act_max, kv_max)."""
    out = (C.c_long * 2)()
    c = cfg.to_c()
    check(lib().hc_default_packer(gpu_mem_bytes, C.byref(c), out))
    return out[0], out[1]


FLOP_KINDS = {"kv_gen": 0, "qkv_gen": 1, "attention": 2, "proj_ffn": 3, "token_recompute": 4, "full_layer": 5}


def flop_count(kind, cfg: ModelConfig, n_tokens: int, k: int = 0) -> float:
    out = C.c_double()
    c = cfg.to_c()
    check(lib().hc_flop_count(FLOP_KINDS.get(kind, kind) if isinstance(kind, str) else int(kind), C.byref(c),
                              n_tokens, k, C.byref(out)))
    return out.value


def weight_bytes(cfg: ModelConfig) -> Tuple[int, int]:
    out = (C.c_uint64 * 2)()
    c = cfg.to_c()
    check(lib().hc_weight_bytes(C.byref(c), out))
    return out[0], out[1]


# ---------------------------------------------------------------- engine ---
MODES = {"hybrid": 0, "kv_only": 1, "act_only": 2, "token_recompute": 3}
# decoder-layer variants (csrc/host/model.hpp Arch): the reference's (no bias /
# LayerNorm / residual) and OPT's pre-LN layer with biases, residuals, final LN
ARCHS = {"reference": 0, "opt": 1}
OPT_EXTRAS = ("b_q", "b_k", "b_v", "b_o", "b_1", "b_2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")


def _ids(ids: Sequence[str]):
    arr = (C.c_char_p * len(ids))(*[s.encode() for s in ids])
    return arr


class TensorParallel:
    """Rank handle of a collective group (csrc/tp.hpp). As `Engine(tp=...)`:
    the optional head-sharded variant — rank g of N owns heads
    [gH/N, (g+1)H/N) and the ACT/host blocks with pbn % N == g; every rank's
    Engine gets the same request ids and tokens. As `Engine(weight_share=...)`:
    batch-partitioned ranks sharing one weight stream."""

    def __init__(self, handle, owner=None, is_group=False, rank=0, size=1):
        self._h = handle
        self._owner = owner          # keeps a local group alive while members exist
        self._is_group = is_group
        self.rank, self.size = rank, size

    @staticmethod
    def _nccl_provider() -> None:
        """libhybridcache dlopens "libnccl.so.2" and reuses a copy already in
        the process. torch links its own (newer) NCCL under the same soname,
        so load torch first: if the system NCCL were loaded first, a later
        `import torch` would bind to it and fail (missing symbols)."""
        try:
            import torch  # noqa: F401
        except ImportError:
            pass

    @staticmethod
    def nccl_unique_ids() -> bytes:
        """Two ncclUniqueIds (compute channel | copy channel), 256 bytes; made on
        rank 0 and broadcast to the others by the caller."""
        TensorParallel._nccl_provider()
        a, b = C.create_string_buffer(128), C.create_string_buffer(128)
        check(lib().hc_tp_nccl_unique_id(a))
        check(lib().hc_tp_nccl_unique_id(b))
        return a.raw + b.raw

    @classmethod
    def nccl(cls, ids: bytes, rank: int, size: int, device: int = 0) -> "TensorParallel":
        TensorParallel._nccl_provider()
        h = C.c_void_p()
        check(lib().hc_tp_create_nccl(ids[:128], ids[128:256], rank, size, device, C.byref(h)))
        return cls(h, rank=rank, size=size)

    @classmethod
    def emulated(cls, rank: int, size: int) -> "TensorParallel":
        """Timing stand-in for one rank of a size-N group on one GPU: the rank's
        shard shapes, streams and bytes, collectives skipped (outputs are NOT
        meaningful)."""
        h = C.c_void_p()
        check(lib().hc_tp_create_emulated(rank, size, C.byref(h)))
        return cls(h, rank=rank, size=size)

    @classmethod
    def local_group(cls, size: int) -> List["TensorParallel"]:
        """size ranks in this process (drive each rank's engine from its own thread)."""
        g = C.c_void_p()
        check(lib().hc_tp_create_local_group(size, C.byref(g)))
        group = cls(g, is_group=True, size=size)
        out = []
        for r in range(size):
            h = C.c_void_p()
            check(lib().hc_tp_local_member(g, r, C.byref(h)))
            out.append(cls(h, owner=group, rank=r, size=size))
        return out

    def __del__(self):
        if getattr(self, "_h", None) and (self._is_group or self._owner is None):
            try:
                lib().hc_tp_destroy(self._h, int(self._is_group))
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self._h = None


class Engine:
    """B200 decode engine over the hybrid KV/ACT cache (csrc/engine.hpp).

    weights: None -> DecoderWeights::generate(cfg, seed, max_seq) drawn in the
    library (rescale=True applies the depth-stable rescale); or a dict of fp64
    reference-layout tensors {"embedding", "positional", "layers": [{w_q..}]}.
    """

    def __init__(self, cfg: ModelConfig, *, seed: int = 42, max_seq: int = 0, rescale: bool = True,
                 weights: Optional[dict] = None, max_batch: int = 1, weights_on_device: bool = True,
                 caps: Optional[PoolCaps] = None, kv_on_gpu: bool = False, host_layers: int = 0,
                 mode: str = "hybrid", allocation: Optional[HostAllocation] = None, scaled: bool = True,
                 max_prefill_tokens: int = 0, device: int = 0, weight_layers: int = 0,
                 recompute_ratio: float = 0.0, arch: str = "reference", tp: Optional[TensorParallel] = None,
                 weight_share: Optional[TensorParallel] = None):
        """tp: head-sharded tensor parallelism. weight_share: a group (same
        constructors as tp) of batch-partitioned ranks streaming ONE copy of the
        weights between them — each rank's host link carries 1/N of every
        layer, an NVLink all-gather completes it (streamed weights only; every
        rank must issue the same decode_step sequence)."""
        self.cfg = ModelConfig(**cfg.__dict__).validate()
        caps = caps or PoolCaps()
        alloc = allocation or HostAllocation(1, 1)
        if mode not in MODES:
            raise InputError(f"unknown mode: {mode}")
        if arch not in ARCHS:
            raise InputError(f"unknown arch: {arch}")
        self.arch = arch
        self.opts = EngineOptionsC(max_batch, max_seq, int(weights_on_device), caps.kv_host, caps.kv_gpu,
                                   caps.act_host, caps.act_gpu, int(kv_on_gpu), host_layers, MODES[mode],
                                   alloc.act_host, alloc.kv_host, int(scaled), max_prefill_tokens, device,
                                   weight_layers, recompute_ratio, ARCHS[arch], tp._h if tp else None,
                                   weight_share._h if weight_share else None)
        self._tp = tp
        self._weight_share = weight_share
        self.max_batch = max_batch
        h = C.c_void_p()
        c = self.cfg.to_c()
        if weights is None:
            if max_seq < 1:
                raise InputError("DecoderWeights: max_seq must be >= 1")
            check(lib().hc_engine_create(C.byref(c), seed, max_seq, int(rescale), C.byref(self.opts), C.byref(h)))
        else:
            emb = np.ascontiguousarray(weights["embedding"], np.float64)
            pos = np.ascontiguousarray(weights["positional"], np.float64)
            keep = []
            ptrs = (C.POINTER(C.c_double) * (6 * self.cfg.num_layers))()
            names = ("w_q", "w_k", "w_v", "w_proj", "w_ffn1", "w_ffn2")
            for l, lw in enumerate(weights["layers"]):
                for j, nme in enumerate(names):
                    a = np.ascontiguousarray(lw[nme], np.float64)
                    keep.append(a)
                    ptrs[6 * l + j] = ptr(a, C.c_double)
            if arch == "opt":
                ex = (C.POINTER(C.c_double) * (10 * self.cfg.num_layers))()
                for l, lx in enumerate(weights["extras"]):
                    for j, nme in enumerate(OPT_EXTRAS):
                        a = np.ascontiguousarray(lx[nme], np.float64)
                        keep.append(a)
                        ex[10 * l + j] = ptr(a, C.c_double)
                lnf = np.ascontiguousarray(np.concatenate([weights["final_ln"]["gamma"],
                                                          weights["final_ln"]["beta"]]), np.float64)
                check(lib().hc_engine_create_from_f64_opt(C.byref(c), pos.shape[0], ptr(emb, C.c_double),
                                                          ptr(pos, C.c_double), ptrs, ex, ptr(lnf, C.c_double),
                                                          C.byref(self.opts), C.byref(h)))
            else:
                check(lib().hc_engine_create_from_f64(C.byref(c), pos.shape[0], ptr(emb, C.c_double),
                                                      ptr(pos, C.c_double), ptrs, C.byref(self.opts), C.byref(h)))
        self._h = h
        w_max_seq = max_seq if weights is None else np.asarray(weights["positional"]).shape[0]
        self._max_seq = min(max_seq, w_max_seq) if max_seq > 0 else w_max_seq
        ch = C.c_void_p()
        check(lib().hc_engine_cache(self._h, C.byref(ch)))
        self.cache = HybridCache(self.cfg.tokens_per_block, _borrowed=ch, _owner=self)
        self._last_n = 0

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().hc_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def prefill(self, ids: Sequence[str], prompts: Sequence[Sequence[int]]) -> None:
        if len(ids) != len(prompts):
            raise InputError("prefill: ids and prompts differ in length")
        offs = np.zeros(len(ids) + 1, np.int32)
        offs[1:] = np.cumsum([len(p) for p in prompts])
        toks = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in prompts])
                                    if len(prompts) else np.zeros(0, np.int32), dtype=np.int32)
        check(lib().hc_engine_prefill(self._h, len(ids), _ids(ids), ptr(offs, C.c_int), ptr(toks, C.c_int)))

    def admit_synthetic(self, ids: Sequence[str], prompt_lens: Sequence[int], seed: int = 1) -> None:
        lens = np.ascontiguousarray(prompt_lens, np.int32)
        check(lib().hc_engine_admit_synthetic(self._h, len(ids), _ids(ids), ptr(lens, C.c_int), seed))

    def set_minibatching(self, act_max: int, kv_max: int, bundle: Optional["TimingBundle"] = None) -> None:
        """Mini-batched decode (paper §4.3.3; sim.cpp:258-358): staging slots of
        act_max ACT / kv_max KV blocks, each step packed by form_minibatches
        (minibatch.cpp:36-83) on pre-growth block counts priced by `bundle`.
        act_max = kv_max = 0 returns to whole-batch steps."""
        b, bp = (bundle.arr5() if bundle is not None else _darr(np.zeros(5)))
        check(lib().hc_engine_set_minibatching(self._h, act_max, kv_max, bp))

    def set_fused_recompute(self, on: bool) -> bool:
        """Recompute fused with decode attention (default on where the heads'
        width is a multiple of 128): the recompute GEMM's epilogue reduces each
        recomputed block to flash-decoding partials against the step's queries
        instead of writing K|V into the paged layout. Returns the path in use."""
        a = C.c_int(0)
        check(lib().hc_engine_set_fused_recompute(self._h, int(bool(on)), C.byref(a)))
        return bool(a.value)

    def fused_recompute(self) -> bool:
        a = C.c_int(0)
        check(lib().hc_engine_set_fused_recompute(self._h, -1, C.byref(a)))
        return bool(a.value)

    def fill_pools(self, seed: int = 1) -> None:
        """Pattern-fill every pool slot (benchmark setup, before a real prefill)."""
        check(lib().hc_engine_fill_pools(self._h, seed))

    def advance_synthetic(self, ids: Sequence[str], n_tokens: int) -> None:
        """Grow each request by n_tokens in decode order, bookkeeping only."""
        check(lib().hc_engine_advance_synthetic(self._h, len(ids), _ids(ids), n_tokens))

    def decode_step(self, ids: Sequence[str], tokens: Sequence[int], *, want_x: bool = True,
                    want_logits: bool = False, want_argmax: bool = False, out: Optional[dict] = None) -> dict:
        n = len(ids)
        toks = np.ascontiguousarray(tokens, np.int32)
        if toks.shape != (n,):
            raise InputError(f"decode_step: {toks.size} tokens for {n} requests")
        res = out if out is not None else {}

        def buf(key, shape, dtype):  # reuse the caller's array only when it fits exactly
            a = res.get(key)
            if not (isinstance(a, np.ndarray) and a.shape == shape and a.dtype == dtype and a.flags.c_contiguous
                    and a.flags.writeable):
                res[key] = np.zeros(shape, dtype)

        if want_x:
            buf("x", (n, self.cfg.hidden_dim), np.uint16)
        if want_logits:
            buf("logits", (n, self.cfg.vocab_size), np.float32)
        if want_argmax:
            buf("argmax", (n,), np.int32)
        check(lib().hc_engine_decode_step(
            self._h, n, _ids(ids), ptr(toks, C.c_int),
            ptr(res["x"], C.c_uint16) if want_x else None,
            ptr(res["logits"], C.c_float) if want_logits else None,
            ptr(res["argmax"], C.c_int) if want_argmax else None))
        self._last_n = n
        return res

    def free_request(self, rid: str) -> None:
        check(lib().hc_engine_free_request(self._h, rid.encode()))

    def configure_cache(self, caps: PoolCaps, *, mode: str = "hybrid", allocation: Optional[HostAllocation] = None,
                        kv_on_gpu: bool = False, host_layers: int = 0, recompute_ratio: float = 0.0) -> None:
        """Drop all requests and rebuild pools / ratio setting (weights kept)."""
        if mode not in MODES:
            raise InputError(f"unknown mode: {mode}")
        a = allocation or HostAllocation(1, 1)
        check(lib().hc_engine_configure_cache(self._h, caps.kv_host, caps.kv_gpu, caps.act_host, caps.act_gpu,
                                              int(kv_on_gpu), MODES[mode], a.act_host, a.kv_host, host_layers,
                                              float(recompute_ratio)))

    def forward_trace(self, ids: Sequence[int]) -> dict:
        """GPU forward_prompt (decoder.cpp:144-157): layer inputs, K, V per layer
        and the output, as fp16 bits."""
        n, L, d = len(ids), self.cfg.num_layers, self.cfg.hidden_dim
        t = np.ascontiguousarray(ids, np.int32)
        res = {k: np.zeros((L, n, d), np.uint16) for k in ("layer_inputs", "k", "v")}
        res["output"] = np.zeros((n, d), np.uint16)
        check(lib().hc_engine_forward_trace(self._h, ptr(t, C.c_int), n, ptr(res["layer_inputs"], C.c_uint16),
                                            ptr(res["k"], C.c_uint16), ptr(res["v"], C.c_uint16),
                                            ptr(res["output"], C.c_uint16)))
        return res

    def layer_forward(self, layer: int, x_bits: np.ndarray) -> dict:
        """One layer of forward_prompt on given fp16 input rows (teacher forcing)."""
        x = np.ascontiguousarray(x_bits, np.uint16)
        n, d = x.shape
        res = {k: np.zeros((n, d), np.uint16) for k in ("k", "v", "output")}
        check(lib().hc_engine_layer_forward(self._h, layer, ptr(x, C.c_uint16), n, ptr(res["k"], C.c_uint16),
                                            ptr(res["v"], C.c_uint16), ptr(res["output"], C.c_uint16)))
        return res

    def token_recompute_kv(self, ids: Sequence[int], layer: int):
        """token_recompute_kv (decoder.cpp:131-142) on the GPU."""
        if layer < 0 or layer >= self.cfg.num_layers:
            raise InputError(f"layer index out of range: {layer}")
        tr = self.forward_trace(ids)
        return tr["k"][layer], tr["v"][layer]

    def read_block(self, kind, loc, pbn: int, layer: int) -> np.ndarray:
        d, tpb, H = self.cfg.hidden_dim, self.cfg.tokens_per_block, self.cfg.num_heads
        if _kind(kind) == 0:  # a tensor-parallel rank holds its own heads of every KV block
            out = np.zeros((2, H // (self._tp.size if self._tp else 1), tpb, d // H), np.uint16)
        else:
            out = np.zeros((tpb, d), np.uint16)
        check(lib().hc_engine_read_block(self._h, _kind(kind), _loc(loc), pbn, layer, ptr(out, C.c_uint16)))
        return out

    def read_weights(self, layer: int) -> np.ndarray:
        """Engine-held fp16 weights: packed layer (layer >= 0), -1 embedding, -2 positional."""
        d, f = self.cfg.hidden_dim, self.cfg.ffn_dim
        if layer == -1:
            out = np.zeros((self.cfg.vocab_size, d), np.uint16)
        elif layer == -2:
            out = np.zeros((self._max_seq, d), np.uint16)
        elif layer == -3:
            out = np.zeros(2 * d, np.uint16)
        else:
            n = self._tp.size if self._tp else 1
            out = np.zeros((4 * d * d + 2 * d * f) // n + ((3 * d + f) // n + 6 * d if self.arch == "opt" else 0),
                           np.uint16)
        check(lib().hc_engine_read_weights(self._h, layer, ptr(out, C.c_uint16)))
        return out

    def capture_inputs(self, on: bool = True) -> None:
        check(lib().hc_engine_capture_inputs(self._h, int(on)))

    def captured_inputs(self) -> np.ndarray:
        out = np.zeros((self.cfg.num_layers, self._last_n, self.cfg.hidden_dim), np.uint16)
        check(lib().hc_engine_captured_inputs(self._h, ptr(out, C.c_uint16), out.size))
        return out

    def last_stats(self) -> dict:
        out, op = _darr(np.zeros(17))
        check(lib().hc_engine_last_stats(self._h, op))
        keys = ("step_ms", "h2d_bytes", "d2h_bytes", "recompute_rows", "recompute_ms", "attn_ms", "gemm_ms",
                "launches", "copy_ms", "recompute_launches", "store_ms", "minibatches", "h2d_weights", "h2d_kv",
                "h2d_act", "d2h_kv", "d2h_act")
        return dict(zip(keys, out.tolist()))

    def set_profile(self, on: bool = True) -> None:
        check(lib().hc_engine_set_profile(self._h, int(on)))

    def set_graphs(self, on: bool = True) -> None:
        """CUDA-graph replay of decode steps (default on)."""
        check(lib().hc_engine_set_graphs(self._h, int(on)))

    def trace(self) -> dict:
        """Events of the last profiled step (reference trace.json schema)."""
        need = C.c_long()
        check(lib().hc_engine_trace_json(self._h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        check(lib().hc_engine_trace_json(self._h, buf, need.value, C.byref(need)))
        return json.loads(buf.value.decode()) if buf.value else {"events": []}

    def time_kv_gen(self, n_tokens: int, reps: int = 5) -> float:
        s = C.c_double()
        check(lib().hc_engine_time_kv_gen(self._h, n_tokens, reps, C.byref(s)))
        return s.value

    def time_load_kv(self, n_tokens: int, reps: int = 5) -> float:
        s = C.c_double()
        check(lib().hc_engine_time_load_kv(self._h, n_tokens, reps, C.byref(s)))
        return s.value
