"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A restatement of the reference ("hybridsim", /root/reference/proj) for the
KV-activation hybrid-caching decode path, used ONLY by tests/, by
``__graft_entry__.smoke()`` as the checker, and by ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs. The product library never
imports it and fails loudly when its CUDA extension is missing.

Pinning: every function here is checked in ``tests/test_oracle.py`` against
(a) the golden fixtures in ``tests/golden/`` that were produced by running the
UNMODIFIED reference (``oracle/_ref/libhybridsim_ref.so``, built by
``oracle/Makefile`` from the reference's own sources) and (b) the reference's
own known-answer tests (test_decoder.cpp, test_cache.cpp, test_plan.cpp,
acceptance.cpp). Integer/bookkeeping functions are bit-exact restatements;
the fp64 decoder numerics agree with the reference to ~1e-13 (numpy's BLAS
summation order differs from the reference's k-outer loop, matrix.cpp:11-21).

Layout conventions are the reference's: matrices are row-major ``A @ W`` with
W stored [in x out] (model.hpp:38-45).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


class InputError(ValueError):
    """errors.hpp:9-11"""


class CapacityError(RuntimeError):
    """errors.hpp:14-16"""


class ConfigError(RuntimeError):
    """errors.hpp:19-21"""


# --------------------------------------------------------------------------
# RNG — rng.hpp:10-49 (SplitMix64 is counter based: draw i uses seed+(i+1)*G)
# --------------------------------------------------------------------------
def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def splitmix_block(seed: int, n: int, start: int = 0) -> np.ndarray:
    """Draws start..start+n-1 of SplitMix64(seed).next() (rng.hpp:14-19)."""
    with np.errstate(over="ignore"):
        idx = np.arange(start + 1, start + n + 1, dtype=np.uint64)
        z = np.uint64(seed & MASK64) + idx * np.uint64(GOLDEN)
        return _mix(z)


class SplitMix64:
    """Scalar stream, rng.hpp:10-43."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + GOLDEN) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform01(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.uniform01()

    def normal(self, mean: float, std: float) -> float:
        u1 = self.uniform01()
        u2 = self.uniform01()
        if u1 <= 0.0:
            u1 = 2.0 ** -53
        r = math.sqrt(-2.0 * math.log(u1))
        return mean + std * r * math.cos(2.0 * 3.14159265358979323846 * u2)

    def uniform_int(self, lo: int, hi: int) -> int:
        return lo + self.next() % (hi - lo + 1)


def mix_seed(seed: int, tag: int) -> int:
    """rng.hpp:46-49"""
    return SplitMix64((seed ^ ((GOLDEN * (tag + 1)) & MASK64)) & MASK64).next()


def seeded_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """model.cpp:82-87: U(-0.1, 0.1), row-major draw order."""
    u = (splitmix_block(seed, rows * cols) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    lo, hi = -0.1, 0.1
    return (lo + (hi - lo) * u).reshape(rows, cols)


# --------------------------------------------------------------------------
# Model config + weights — model.hpp:15-58, model.cpp:8-117
# --------------------------------------------------------------------------
@dataclass
class ModelConfig:
    name: str = "custom"
    num_layers: int = 1
    hidden_dim: int = 64
    num_heads: int = 1
    ffn_dim: int = 0
    vocab_size: int = 256
    tokens_per_block: int = 16
    bytes_per_scalar: int = 2
    seed: int = 0

    def validate(self) -> "ModelConfig":
        if self.ffn_dim == 0:
            self.ffn_dim = 4 * self.hidden_dim
        if min(self.num_layers, self.hidden_dim, self.num_heads, self.vocab_size,
               self.tokens_per_block, self.bytes_per_scalar) < 1:
            raise InputError("ModelConfig: all counts must be >= 1")
        if self.hidden_dim % self.num_heads:
            raise InputError("ModelConfig: hidden_dim must be divisible by num_heads")
        if self.ffn_dim < self.hidden_dim:
            raise InputError("ModelConfig: ffn_dim must be >= hidden_dim")
        return self

    @property
    def head_dim(self) -> int:
        return self.hidden_dim // self.num_heads


PRESETS = {"opt-6.7b": (32, 4096, 32), "opt-13b": (40, 5120, 40),
           "opt-30b": (48, 7168, 56), "opt-66b": (64, 9216, 72)}


def preset(name: str) -> ModelConfig:
    """model.cpp:37-43"""
    if name not in PRESETS:
        raise InputError("unknown model preset: " + name)
    layers, d, h = PRESETS[name]
    return ModelConfig(name, layers, d, h, 4 * d, 50272, 16, 2)


WEIGHT_NAMES = ("w_q", "w_k", "w_v", "w_proj", "w_ffn1", "w_ffn2")


@dataclass
class DecoderWeights:
    config: ModelConfig
    max_seq: int
    embedding: np.ndarray
    positional: np.ndarray
    layers: List[Dict[str, np.ndarray]] = field(default_factory=list)
    # OPT decoder-layer variant only (extension, see forward_prompt_opt)
    extras: Optional[List[Dict[str, np.ndarray]]] = None
    final_ln: Optional[Dict[str, np.ndarray]] = None


def generate_weights(cfg: ModelConfig, seed: int, max_seq: int) -> DecoderWeights:
    """DecoderWeights::generate, model.cpp:94-117 (tags model.cpp:90)."""
    cfg = ModelConfig(**cfg.__dict__).validate()
    if max_seq < 1:
        raise InputError("DecoderWeights: max_seq must be >= 1")
    d, f = cfg.hidden_dim, cfg.ffn_dim
    w = DecoderWeights(cfg, max_seq,
                       seeded_matrix(cfg.vocab_size, d, mix_seed(seed, 0)),
                       seeded_matrix(max_seq, d, mix_seed(seed, 1)))
    shapes = ((d, d), (d, d), (d, d), (d, d), (d, f), (f, d))
    for l in range(cfg.num_layers):
        base = 100 + 8 * l
        w.layers.append({n: seeded_matrix(r, c, mix_seed(seed, base + i))
                         for i, (n, (r, c)) in enumerate(zip(WEIGHT_NAMES, shapes))})
    return w


def rescale_factors(cfg: ModelConfig) -> Dict[str, float]:
    """Deterministic per-tensor rescale of the reference draws.

    The reference init (no LayerNorm / residual) grows the
    activation RMS ~10x per layer; this keeps it O(0.07) over 48 layers.
    Factors are computed as 10*sqrt(x) in IEEE double, identically in the
    product's C++ host code (csrc/host/model.cpp)."""
    d, f = float(cfg.hidden_dim), float(cfg.ffn_dim)
    s_attn = 10.0 * math.sqrt(3.0 / d)
    s_f1 = 10.0 * math.sqrt(3.0 * math.sqrt(2.0) / d)
    s_f2 = 10.0 * math.sqrt(3.0 * math.sqrt(2.0) / f)
    return {"w_q": s_attn, "w_k": s_attn, "w_v": s_attn, "w_proj": s_attn,
            "w_ffn1": s_f1, "w_ffn2": s_f2}


def f16_round(x: np.ndarray) -> np.ndarray:
    """fp64 -> fp32 (RNE) -> IEEE binary16 (RNE), returned as fp64. Same rule as
    the product's host conversion (csrc/host/model.cpp: to_f16) and the GPU
    draw (weights_gen.cu: __float2half_rn)."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    return f.astype(np.float16).astype(np.float64)


def to_f16_bits(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float32).astype(np.float16).view(np.uint16)


def f16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(b, dtype=np.uint16).view(np.float16).astype(np.float64)


def prepare_weights(w: DecoderWeights, rescale: bool = True, f16: bool = True) -> DecoderWeights:
    """Rescale then round every tensor to fp16 (values kept in fp64) so the
    oracle consumes exactly the numbers the GPU consumes."""
    fac = rescale_factors(w.config) if rescale else {n: 1.0 for n in WEIGHT_NAMES}
    rnd = f16_round if f16 else (lambda a: a)
    out = DecoderWeights(w.config, w.max_seq, rnd(w.embedding), rnd(w.positional))
    for lw in w.layers:
        out.layers.append({n: rnd(lw[n] * fac[n]) for n in WEIGHT_NAMES})
    return out


# --------------------------------------------------------------------------
# Decoder numerics — decoder.cpp:15-174 (fp64)
# --------------------------------------------------------------------------
def attention_rows(q: np.ndarray, k: np.ndarray, v: np.ndarray, ctx: Sequence[int],
                   num_heads: int, scaled: bool = True) -> np.ndarray:
    """attention_row, decoder.cpp:15-43, for each query row i over rows [0, ctx[i])."""
    n, d = q.shape
    hd = d // num_heads
    scale = 1.0 / math.sqrt(hd) if scaled else 1.0
    out = np.zeros((n, d))
    for i in range(n):
        c = ctx[i]
        for h in range(num_heads):
            sl = slice(h * hd, (h + 1) * hd)
            logits = (k[:c, sl] @ q[i, sl]) * scale
            w = np.exp(logits - logits.max())
            w = w / w.sum()
            out[i, sl] = w @ v[:c, sl]
    return out


def embed(ids: Sequence[int], w: DecoderWeights, start_pos: int = 0) -> np.ndarray:
    """embed / embed_one, decoder.cpp:65-95."""
    ids = list(ids)
    if start_pos + len(ids) > w.max_seq:
        raise InputError("embed: sequence longer than max_seq")
    for t in ids:
        if t < 0 or t >= w.config.vocab_size:
            raise InputError(f"embed: token id out of range: {t}")
    pos = np.arange(start_pos, start_pos + len(ids))
    return w.embedding[np.asarray(ids, dtype=np.int64)] + w.positional[pos]


def qkv_generate(a: np.ndarray, layer: int, w: DecoderWeights):
    """decoder.cpp:97-103"""
    lw = w.layers[layer]
    return a @ lw["w_q"], a @ lw["w_k"], a @ lw["w_v"]


def project_ffn(att: np.ndarray, layer: int, w: DecoderWeights) -> np.ndarray:
    """decoder.cpp:113-121"""
    lw = w.layers[layer]
    h = np.maximum((att @ lw["w_proj"]) @ lw["w_ffn1"], 0.0)
    return h @ lw["w_ffn2"]


def recompute_kv_from_activation(a_c: np.ndarray, layer: int, w: DecoderWeights):
    """decoder.cpp:123-129 (paper Eq. 7; no bias)."""
    if layer < 0 or layer >= w.config.num_layers:
        raise InputError(f"layer index out of range: {layer}")
    if a_c.shape[1] != w.config.hidden_dim:
        raise InputError("recompute_kv_from_activation: width != hidden_dim")
    lw = w.layers[layer]
    return a_c @ lw["w_k"], a_c @ lw["w_v"]


@dataclass
class ForwardTrace:
    layer_inputs: List[np.ndarray]
    k: List[np.ndarray]
    v: List[np.ndarray]
    output: np.ndarray


def forward_prompt(ids: Sequence[int], w: DecoderWeights, scaled: bool = True) -> ForwardTrace:
    """decoder.cpp:144-157: causal prefill capturing A^l and K,V per layer."""
    a = embed(ids, w)
    n = a.shape[0]
    ins, ks, vs = [], [], []
    for l in range(w.config.num_layers):
        ins.append(a)
        q, k, v = qkv_generate(a, l, w)
        att = attention_rows(q, k, v, [t + 1 for t in range(n)], w.config.num_heads, scaled)
        ks.append(k)
        vs.append(v)
        a = project_ffn(att, l, w)
    return ForwardTrace(ins, ks, vs, a)


def token_recompute_kv(ids: Sequence[int], w: DecoderWeights, target_layer: int,
                       scaled: bool = True):
    """decoder.cpp:131-142"""
    if target_layer < 0 or target_layer >= w.config.num_layers:
        raise InputError(f"layer index out of range: {target_layer}")
    a = embed(ids, w)
    n = a.shape[0]
    for l in range(target_layer):
        q, k, v = qkv_generate(a, l, w)
        a = project_ffn(attention_rows(q, k, v, [t + 1 for t in range(n)], w.config.num_heads,
                                       scaled), l, w)
    _, k, v = qkv_generate(a, target_layer, w)
    return k, v


@dataclass
class StepResult:
    output: np.ndarray          # [1 x d]
    new_k: List[np.ndarray]     # per layer [1 x d]
    new_v: List[np.ndarray]
    layer_inputs: List[np.ndarray]  # decode-time X per layer (extension, §8 A8)


def generation_step(token: int, pos: int, ctx_k: Sequence[np.ndarray],
                    ctx_v: Sequence[np.ndarray], w: DecoderWeights,
                    scaled: bool = True) -> StepResult:
    """decoder.cpp:159-174. Also returns decode-time layer inputs, which the
    reference computes but does not expose (decoder.hpp:56-59); they equal
    forward_prompt(prefix+token).layer_inputs[l][pos]."""
    if len(ctx_k) != w.config.num_layers:
        raise InputError("generation_step: context must cover every layer")
    x = embed([token], w, start_pos=pos)
    nk, nv, ins = [], [], []
    for l in range(w.config.num_layers):
        ins.append(x)
        q, k, v = qkv_generate(x, l, w)
        fk = np.concatenate([ctx_k[l], k]) if ctx_k[l].shape[0] else k
        fv = np.concatenate([ctx_v[l], v]) if ctx_v[l].shape[0] else v
        att = attention_rows(q, fk, fv, [fk.shape[0]], w.config.num_heads, scaled)
        x = project_ffn(att, l, w)
        nk.append(k)
        nv.append(v)
    return StepResult(x, nk, nv, ins)


def logits_tied(x: np.ndarray, w: DecoderWeights) -> np.ndarray:
    """Extension (parity unpinned by the reference, which has no LM head —
    decoder.hpp:56-59): tied head x @ E^T, as OPT does."""
    return x @ w.embedding.T


# --------------------------------------------------------------------------
# OPT decoder-layer variant — an EXTENSION (bias,
# LayerNorm, residual). The reference's layer has none of these
# (decoder.cpp:97-129), so this restatement is parity-unpinned
# by reference tests; it is the checker for the product's kArchOpt
# (csrc/host/model.hpp). Extras use the reference's RNG (rng.hpp:10-49) on
# tags the reference leaves free: 100+8l+6 biases, 100+8l+7 LayerNorms,
# 2 the final LayerNorm.
# --------------------------------------------------------------------------
OPT_EXTRAS = ("b_q", "b_k", "b_v", "b_o", "b_1", "b_2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")
LN_EPS = 1e-5


def generate_opt_extras(cfg: ModelConfig, seed: int):
    """Per-layer biases + LayerNorm parameters and the final LayerNorm
    (gamma = 1 + u, beta = u, biases = u; u ~ U(-0.1, 0.1))."""
    d, f = cfg.hidden_dim, cfg.ffn_dim
    layers = []
    for l in range(cfg.num_layers):
        base = 100 + 8 * l
        b = seeded_matrix(1, 5 * d + f, mix_seed(seed, base + 6)).ravel()
        u = seeded_matrix(1, 4 * d, mix_seed(seed, base + 7)).ravel()
        layers.append({"b_q": b[:d], "b_k": b[d:2 * d], "b_v": b[2 * d:3 * d], "b_o": b[3 * d:4 * d],
                       "b_1": b[4 * d:4 * d + f], "b_2": b[4 * d + f:],
                       "ln1_g": 1.0 + u[:d], "ln1_b": u[d:2 * d], "ln2_g": 1.0 + u[2 * d:3 * d], "ln2_b": u[3 * d:]})
    u = seeded_matrix(1, 2 * d, mix_seed(seed, 2)).ravel()
    return layers, {"gamma": 1.0 + u[:d], "beta": u[d:]}


def with_opt_extras(w: DecoderWeights, seed: int, f16: bool = True) -> DecoderWeights:
    """w plus the OPT extras, fp16-rounded like the GPU's copies."""
    rnd = f16_round if f16 else (lambda a: a)
    ex, lnf = generate_opt_extras(w.config, seed)
    return DecoderWeights(w.config, w.max_seq, w.embedding, w.positional, w.layers,
                          [{k: rnd(v) for k, v in e.items()} for e in ex], {k: rnd(v) for k, v in lnf.items()})


def layer_norm(x: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float = LN_EPS) -> np.ndarray:
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


@dataclass
class OptTrace:
    layer_inputs: List[np.ndarray]   # residual stream x entering layer l
    act: List[np.ndarray]            # LN1(x): the ACT-cache payload
    k: List[np.ndarray]
    v: List[np.ndarray]
    output: np.ndarray               # LN_f(x_L): the model output


def forward_prompt_opt(ids: Sequence[int], w: DecoderWeights, scaled: bool = True) -> OptTrace:
    """OPT pre-LN decoder over a prompt: x^ = LN1(x); q,k,v = x^ W + b;
    x' = x + attn W_o + b_o; x_next = x' + relu(LN2(x') W1 + b1) W2 + b2;
    output LN_f(x_L). Recompute from the ACT payload is K|V = x^ [W_k|W_v] +
    [b_k|b_v] — Eq. 7 with OPT's bias."""
    if w.extras is None or w.final_ln is None:
        raise InputError("forward_prompt_opt: weights carry no OPT extras")
    x = embed(ids, w)
    n = x.shape[0]
    ins, acts, ks, vs = [], [], [], []
    for l in range(w.config.num_layers):
        lw, e = w.layers[l], w.extras[l]
        ins.append(x)
        xa = layer_norm(x, e["ln1_g"], e["ln1_b"])
        acts.append(xa)
        q, k, v = xa @ lw["w_q"] + e["b_q"], xa @ lw["w_k"] + e["b_k"], xa @ lw["w_v"] + e["b_v"]
        ks.append(k)
        vs.append(v)
        att = attention_rows(q, k, v, [t + 1 for t in range(n)], w.config.num_heads, scaled)
        x1 = x + att @ lw["w_proj"] + e["b_o"]
        h = np.maximum(layer_norm(x1, e["ln2_g"], e["ln2_b"]) @ lw["w_ffn1"] + e["b_1"], 0.0)
        x = x1 + h @ lw["w_ffn2"] + e["b_2"]
    return OptTrace(ins, acts, ks, vs, layer_norm(x, w.final_ln["gamma"], w.final_ln["beta"]))


# --------------------------------------------------------------------------
# FLOP model — flops.cpp:7-37
# --------------------------------------------------------------------------
KVGEN, QKVGEN, ATTENTION, PROJFFN, TOKEN_RECOMPUTE, FULL_LAYER = range(6)


def flop_count(kind: int, cfg: ModelConfig, n: int, k: int = 0) -> float:
    if n < 0:
        raise InputError("flop_count: negative token count")
    n, d, f = float(n), float(cfg.hidden_dim), float(cfg.ffn_dim)
    if kind == KVGEN:
        return 2.0 * (2.0 * n * d * d)
    if kind == QKVGEN:
        return 2.0 * (3.0 * n * d * d)
    if kind == ATTENTION:
        return 2.0 * d * n * (n + 1.0)
    if kind == PROJFFN:
        return 2.0 * (n * d * d + 2.0 * n * d * f)
    if kind == FULL_LAYER:
        return (flop_count(QKVGEN, cfg, int(n)) + flop_count(ATTENTION, cfg, int(n))
                + flop_count(PROJFFN, cfg, int(n)))
    if kind == TOKEN_RECOMPUTE:
        if k < 0 or k >= cfg.num_layers:
            raise InputError("flop_count: layer index out of range")
        return float(k) * flop_count(FULL_LAYER, cfg, int(n)) + flop_count(QKVGEN, cfg, int(n))
    raise InputError("flop_count: unknown op kind")


def attention_step_flops(cfg: ModelConfig, ctx: int) -> float:
    return 4.0 * float(cfg.hidden_dim) * float(ctx)


# --------------------------------------------------------------------------
# Hybrid cache block tables — cache.hpp:15-95, cache.cpp:35-166 (bit-exact)
# --------------------------------------------------------------------------
KV, ACT = "KV", "ACT"
HOST, GPU = "host", "gpu"


@dataclass
class BlockTableEntry:
    kind: str
    location: str
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
        a = sum(1 for e in self.entries if e.kind == ACT)
        return a, len(self.entries) - a


class HybridCache:
    """Four (kind x location) pools, LIFO free lists handing out pbn 0 first."""

    def __init__(self, tokens_per_block: int, kv_host: int = 0, kv_gpu: int = 0,
                 act_host: int = 0, act_gpu: int = 0, kv_on_gpu: bool = False):
        if tokens_per_block < 1:
            raise InputError("HybridCache: tokens_per_block must be >= 1")
        caps = {(KV, HOST): kv_host, (KV, GPU): kv_gpu, (ACT, HOST): act_host, (ACT, GPU): act_gpu}
        if min(caps.values()) < 0:
            raise InputError("HybridCache: negative pool capacity")
        self.tpb = tokens_per_block
        self.kv_on_gpu = kv_on_gpu
        self.caps = caps
        self.free = {k: list(range(c - 1, -1, -1)) for k, c in caps.items()}
        self.tables: Dict[str, BlockTable] = {}
        self.order: List[str] = []

    def _table(self, rid: str) -> BlockTable:
        if rid not in self.tables:
            raise InputError("unknown request id: " + rid)
        return self.tables[rid]

    def table(self, rid: str) -> BlockTable:
        return self._table(rid)

    def create_request(self, rid: str, prompt_len: int) -> BlockTable:
        if prompt_len < 0:
            raise InputError("create_request: negative prompt length")
        if rid in self.tables:
            raise InputError("duplicate request id: " + rid)
        self.tables[rid] = BlockTable(rid, prompt_len)
        self.order.append(rid)
        return self.tables[rid]

    def append_block(self, rid: str, kind: str) -> BlockTableEntry:
        t = self._table(rid)
        if t.entries and t.entries[-1].filled_tokens < self.tpb:
            raise InputError("append_block: last block not yet full")
        if kind == ACT:
            order = [GPU, HOST]
        else:
            order = [GPU, HOST] if self.kv_on_gpu else [HOST]
        for loc in order:
            if self.free[(kind, loc)]:
                pbn = self.free[(kind, loc)].pop()
                e = BlockTableEntry(kind, loc, pbn, 0)
                t.entries.append(e)
                return e
        raise CapacityError(f"append_block: {kind} pools exhausted")

    def fill_token(self, rid: str) -> None:
        t = self._table(rid)
        if not t.entries:
            raise InputError("fill_token: no blocks; append_block first")
        if t.entries[-1].filled_tokens >= self.tpb:
            raise InputError("fill_token: last block full; append_block first")
        t.entries[-1].filled_tokens += 1

    def blocks_by_kind(self, rid: str) -> Tuple[int, int]:
        return self._table(rid).blocks_by_kind()

    def free_request(self, rid: str) -> None:
        t = self._table(rid)
        for e in t.entries:
            self.free[(e.kind, e.location)].append(e.pbn)
        del self.tables[rid]
        self.order.remove(rid)

    def free_blocks(self, kind: str, loc: str) -> int:
        return len(self.free[(kind, loc)])

    def capacity(self, kind: str, loc: str) -> int:
        return self.caps[(kind, loc)]

    def dump_json(self) -> dict:
        reqs = []
        for rid in self.order:
            t = self.tables[rid]
            reqs.append({"id": t.request_id, "prompt_len": t.prompt_len,
                         "context_len": t.context_len(),
                         "entries": [{"kind": e.kind, "location": e.location, "pbn": e.pbn,
                                      "filled": e.filled_tokens} for e in t.entries]})
        return {"tokens_per_block": self.tpb, "requests": reqs}


def bytes_of(kind: str, cfg: ModelConfig) -> int:
    """cache.cpp:142-147 (per layer)."""
    per_token = cfg.hidden_dim * cfg.bytes_per_scalar
    return cfg.tokens_per_block * (2 if kind == KV else 1) * per_token


# --------------------------------------------------------------------------
# Ratio policy + planner — plan.cpp, timing.cpp (bit-exact IEEE restatement)
# --------------------------------------------------------------------------
@dataclass
class HostAllocation:
    act_host: int = 0
    kv_host: int = 0
    act_init: int = 0
    kv_init: int = 0
    act_remain: int = 0
    kv_remain: int = 0


def next_block_kind(act_req: int, kv_req: int, alloc: HostAllocation) -> str:
    """plan.cpp:154-164: minimise |share - target|, ties -> ACT."""
    if alloc.act_host + alloc.kv_host <= 0:
        raise InputError("next_block_kind: allocation has no blocks")
    if act_req < 0 or kv_req < 0:
        raise InputError("next_block_kind: negative block count")
    target = float(alloc.act_host) / float(alloc.act_host + alloc.kv_host)
    total = float(act_req + kv_req + 1)
    err_act = abs(float(act_req + 1) / total - target)
    err_kv = abs(float(act_req) / total - target)
    return ACT if err_act <= err_kv else KV


@dataclass
class LinearTimeModel:
    slope: float = 0.0
    intercept: float = 0.0
    r_squared: float = 0.0
    intercept_clamped: bool = False


def fit_linear(samples: Sequence[Tuple[float, float]]) -> LinearTimeModel:
    """timing.cpp:38-73 (OLS; negative intercept clamped to 0)."""
    n = len(samples)
    if n < 2:
        raise InputError("fit_linear: need at least two samples")
    if len({s[0] for s in samples}) < 2:
        raise InputError("fit_linear: need at least two distinct n_tokens values")
    sx = sy = 0.0
    for x, y in samples:
        sx += x
        sy += y
    mx, my = sx / n, sy / n
    sxx = sxy = 0.0
    for x, y in samples:
        sxx += (x - mx) * (x - mx)
        sxy += (x - mx) * (y - my)
    m = LinearTimeModel(sxy / sxx, 0.0)
    m.intercept = my - m.slope * mx
    if m.intercept < 0:
        m.intercept, m.intercept_clamped = 0.0, True
    ss_res = ss_tot = 0.0
    for x, y in samples:
        fit = m.slope * x + m.intercept
        ss_res += (y - fit) * (y - fit)
        ss_tot += (y - my) * (y - my)
    m.r_squared = (1.0 if ss_res == 0.0 else 0.0) if ss_tot == 0.0 else 1.0 - ss_res / ss_tot
    return m


def eval_model(m: LinearTimeModel, n: float) -> float:
    if n < 0:
        raise InputError("eval: negative token count")
    return m.slope * n + m.intercept


def invert(m: LinearTimeModel, seconds: float) -> int:
    """timing.cpp:108-116"""
    if m.slope <= 0:
        raise InputError("invert: model is not invertible (slope <= 0)")
    if seconds < 0:
        raise InputError("invert: negative time budget")
    n = int(math.floor((seconds - m.intercept) / m.slope))
    if n < 0:
        return 0
    while n > 0 and eval_model(m, float(n)) > seconds:
        n -= 1
    return n


def weight_bytes(cfg: ModelConfig) -> Tuple[int, int]:
    """timing.cpp:118-127 -> (per_layer, total)"""
    d, f, bps = cfg.hidden_dim, cfg.ffn_dim, cfg.bytes_per_scalar
    per = (4 * d * d + 2 * d * f) * bps
    return per, per * cfg.num_layers + cfg.vocab_size * d * bps


@dataclass
class TimingBundle:
    t_kv_gen: LinearTimeModel
    t_load_kv: LinearTimeModel
    t_load_w: float = 0.0
    s_weight_layer: int = 0
    s_weight_total: int = 0


def bundle_from_samples(kv_gen, load_kv, pcie_bandwidth: float, cfg: ModelConfig) -> TimingBundle:
    """timing.cpp:172-183"""
    per, total = weight_bytes(cfg)
    return TimingBundle(fit_linear(kv_gen), fit_linear(load_kv), float(per) / pcie_bandwidth, per, total)


@dataclass
class MemoryBudget:
    m_host: float = 0.0
    s_weight: float = 0.0
    s_kv_block: float = 0.0
    s_act_block: float = 0.0


def budget_for(host_mem: float, cfg: ModelConfig, bundle: TimingBundle) -> MemoryBudget:
    """plan.cpp:41-51"""
    return MemoryBudget(host_mem, float(bundle.s_weight_total),
                        float(bytes_of(KV, cfg)) * cfg.num_layers,
                        float(bytes_of(ACT, cfg)) * cfg.num_layers)


def _fit_blocks(avail: float, block: float) -> int:
    if avail <= 0 or block <= 0:
        return 0
    n = int(math.floor(avail / block))
    while n > 0 and float(n) * block > avail:
        n -= 1
    while float(n + 1) * block <= avail:
        n += 1
    return n


def initial_cache_allocation(b: TimingBundle, tpb: int, act_gpu: int) -> Tuple[int, int]:
    """plan.cpp:53-69"""
    if tpb < 1:
        raise InputError("initial_cache_allocation: bad block size")
    if act_gpu < 0:
        raise InputError("initial_cache_allocation: negative ACT_GPU")
    budget = b.t_load_w - eval_model(b.t_kv_gen, float(act_gpu) * tpb)
    a = k = 0
    if budget >= 0:
        if b.t_kv_gen.slope > 0:
            a = invert(b.t_kv_gen, budget) // tpb
    else:
        if b.t_load_kv.slope > 0:
            k = invert(b.t_load_kv, -budget) // tpb
    return a, k


def alloc_remaining(b: TimingBundle, mem: MemoryBudget, tpb: int, act_init: int,
                    kv_init: int) -> Tuple[int, int]:
    """plan.cpp:71-104"""
    if mem.s_kv_block <= 0 or mem.s_act_block <= 0:
        raise InputError("alloc_remaining: block sizes must be positive")
    occupied = mem.s_act_block * float(act_init) + mem.s_kv_block * float(kv_init)
    remaining = mem.m_host - mem.s_weight - occupied
    if remaining < 0:
        raise CapacityError("alloc_remaining: host memory cannot hold weights plus initial blocks")
    bb = float(tpb)
    sa, sk = b.t_kv_gen.slope * bb, b.t_load_kv.slope * bb
    ia, ik = b.t_kv_gen.intercept, b.t_load_kv.intercept
    denom = sa * mem.s_kv_block + sk * mem.s_act_block
    if denom <= 0:
        return 0, int(math.floor(remaining / mem.s_kv_block))
    x_exact = (sk * remaining + mem.s_kv_block * (ik - ia)) / denom
    if x_exact < 0:
        return 0, _fit_blocks(remaining, mem.s_kv_block)
    y_exact = (remaining - mem.s_act_block * x_exact) / mem.s_kv_block
    if y_exact < 0:
        return _fit_blocks(remaining, mem.s_act_block), 0
    x = int(math.floor(x_exact + 1e-9 * (1.0 + abs(x_exact))))
    return x, _fit_blocks(remaining - mem.s_act_block * float(x), mem.s_kv_block)


def planned_t_pcie(b: TimingBundle, tpb: int, a: HostAllocation) -> float:
    return b.t_load_w + eval_model(b.t_load_kv, float(a.kv_host) * tpb)


def planned_t_computation(b: TimingBundle, tpb: int, a: HostAllocation, act_gpu: int) -> float:
    return eval_model(b.t_kv_gen, float(a.act_host + act_gpu) * tpb)


def plan_host_allocation(b: TimingBundle, mem: MemoryBudget, tpb: int, act_gpu: int) -> HostAllocation:
    """plan.cpp:106-152 (two-step + binary-search polish on the frontier)."""
    a = HostAllocation()
    a.act_init, a.kv_init = initial_cache_allocation(b, tpb, act_gpu)
    a.act_remain, a.kv_remain = alloc_remaining(b, mem, tpb, a.act_init, a.kv_init)
    a.act_host, a.kv_host = a.act_init + a.act_remain, a.kv_init + a.kv_remain
    avail = mem.m_host - mem.s_weight

    def frontier_kv(x):
        return _fit_blocks(avail - mem.s_act_block * float(x), mem.s_kv_block)

    def gap(x):
        c = HostAllocation(x, frontier_kv(x))
        return planned_t_pcie(b, tpb, c) - planned_t_computation(b, tpb, c, act_gpu)

    x_max = _fit_blocks(avail, mem.s_act_block)
    if gap(0) <= 0:
        best = 0
    elif gap(x_max) >= 0:
        best = x_max
    else:
        lo, hi = 0, x_max
        while hi - lo > 1:
            mid = lo + (hi - lo) // 2
            if gap(mid) > 0:
                lo = mid
            else:
                hi = mid
        best = lo if abs(gap(lo)) <= abs(gap(hi)) else hi
    a.act_host, a.kv_host = best, frontier_kv(best)
    a.act_remain, a.kv_remain = a.act_host - a.act_init, a.kv_host - a.kv_init
    return a


# --------------------------------------------------------------------------
# Mini-batch packer — minibatch.cpp:10-83 (greedy) and 148-170 (brute force)
# --------------------------------------------------------------------------
def balance(act_mb: int, kv_mb: int, b: TimingBundle, tpb: int) -> float:
    if act_mb < 0 or kv_mb < 0:
        raise InputError("balance: negative block count")
    num = eval_model(b.t_kv_gen, float(act_mb) * tpb)
    den = eval_model(b.t_load_kv, float(kv_mb) * tpb)
    if num == 0.0 and den == 0.0:
        return 1.0
    if den == 0.0:
        return math.inf
    return num / den


def cost_fb(act_mb: int, kv_mb: int, b: TimingBundle, tpb: int) -> float:
    x = balance(act_mb, kv_mb, b, tpb)
    if x == 0.0:
        return math.inf
    return max(x, 1.0 / x)


def form_minibatches(requests, act_max: int, kv_max: int, b: TimingBundle, tpb: int):
    """requests: [(id, act_blocks, kv_blocks)] -> [[ids], ...] (minibatch.cpp:36-83)."""
    if act_max < 1 or kv_max < 1:
        raise InputError("form_minibatches: capacities must be >= 1")
    for rid, a, k in requests:
        if a < 0 or k < 0:
            raise InputError("form_minibatches: negative block count for request " + rid)
        if a > act_max or k > kv_max:
            raise InputError("request too large for GPU buffer capacities: " + rid)
    order = sorted(requests, key=lambda r: (-(r[1] + r[2]), r[0]))
    used = [False] * len(order)
    left = len(order)
    out = []
    while left:
        ids, am, km, fb = [], 0, 0, math.inf
        changed = True
        while changed:
            changed = False
            for i, (rid, a, k) in enumerate(order):
                if used[i] or am + a > act_max or km + k > kv_max:
                    continue
                after = cost_fb(am + a, km + k, b, tpb)
                if ids and after > fb:
                    continue
                ids.append(rid)
                am, km, fb = am + a, km + k, after
                used[i] = True
                left -= 1
                changed = True
        out.append(ids)
    return out


# --------------------------------------------------------------------------
# Block-kind assignment in the simulator's call order — sim.cpp:150-223,308-310
# --------------------------------------------------------------------------
HYBRID, KV_ONLY, ACT_ONLY, TOKEN_RECOMPUTE_MODE = "hybrid", "kv_only", "act_only", "token_recompute"


def mode_allocation(mode: str, alloc: HostAllocation, act_gpu: int) -> Tuple[HostAllocation, int]:
    """Byte-neutral pool conversion for forced modes, sim.cpp:150-167."""
    a = HostAllocation(**alloc.__dict__)
    if mode in (KV_ONLY, TOKEN_RECOMPUTE_MODE):
        a.kv_host += a.act_host // 2
        a.act_host = 0
        act_gpu = 0
    elif mode == ACT_ONLY:
        a.act_host += 2 * a.kv_host
        a.kv_host = 0
    return a, act_gpu


class BlockAssigner:
    """The simulator's ``add_token`` (sim.cpp:194-220) over a HybridCache built
    the way simulate() builds it (sim.cpp:181)."""

    def __init__(self, tpb: int, mode: str, alloc: HostAllocation, act_gpu: int = 0,
                 recompute_ratio: float = 0.0):
        self.mode = mode
        self.alloc, act_gpu = mode_allocation(mode, alloc, act_gpu)
        self.cache = HybridCache(tpb, self.alloc.kv_host, 0, self.alloc.act_host, act_gpu)
        self.rc: Dict[str, int] = {}
        self.ratio = recompute_ratio

    def add_request(self, rid: str, prompt_len: int) -> None:
        self.cache.create_request(rid, prompt_len)
        self.rc[rid] = 0

    def add_token(self, rid: str) -> Optional[BlockTableEntry]:
        c = self.cache
        if self.mode == TOKEN_RECOMPUTE_MODE:
            cached = c.table(rid).context_len()
            total = float(self.rc[rid] + cached + 1)
            err_rc = abs((self.rc[rid] + 1) / total - self.ratio)
            err_kv = abs(self.rc[rid] / total - self.ratio)
            if err_rc <= err_kv:
                self.rc[rid] += 1
                return None
        t = c.table(rid)
        if t.context_len() % c.tpb == 0:
            kind = KV
            if self.mode == HYBRID:
                a, k = t.blocks_by_kind()
                kind = next_block_kind(a, k, self.alloc)
            elif self.mode == ACT_ONLY:
                kind = ACT
            c.append_block(rid, kind)
        c.fill_token(rid)
        return c.table(rid).entries[-1]


def assign_batch(tpb: int, prompt_lens: Sequence[int], gen_lens: Sequence[int], mode: str,
                 alloc: HostAllocation, act_gpu: int = 0, decode_iters: Optional[int] = None,
                 recompute_ratio: float = 0.0) -> BlockAssigner:
    """Prompt tokens request by request (sim.cpp:222-223), then one token per
    active request per iteration (sim.cpp:261-264, 308-310)."""
    ba = BlockAssigner(tpb, mode, alloc, act_gpu, recompute_ratio)
    ids = [f"r{i}" for i in range(len(prompt_lens))]
    for rid, p in zip(ids, prompt_lens):
        ba.add_request(rid, p)
    for rid, p in zip(ids, prompt_lens):
        for _ in range(p):
            ba.add_token(rid)
    iters = max(gen_lens) if decode_iters is None else decode_iters
    for it in range(iters):
        for rid, g in zip(ids, gen_lens):
            if it < g:
                ba.add_token(rid)
    return ba


def dumps(obj) -> str:
    """nlohmann::json::dump() formatting (compact, keys sorted)."""
    return json.dumps(obj, separators=(",", ":"), sort_keys=True)
