"""End-to-end parity of the B200 engine (prefill + batched decode over the
hybrid cache) with the CPU oracle, through the C ABI.

Oracle side: hybridsim_oracle (fp64 restatement of decoder.cpp, pinned to the
reference in test_oracle.py) on the SAME bf16-rounded weights.
Tolerance (north_star): max|got - ref| / max|ref| <= 1e-2 per tensor for
decode outputs, recomputed K/V and logits; greedy tokens must match where the
oracle's top-2 logit margin exceeds the bf16 noise floor.
Block tables must match the oracle bit-exactly (dump_json string equality).
"""
import json

import numpy as np
import pytest

import hybridsim_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-2
TOL_OPT = 1e-2  # OPT layer variant (not in the reference): fp16 LayerNorm outputs, see the fuzz test


def rel(got, ref):
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def f64(bits):
    return O.f16_bits_to_f64(np.asarray(bits))


def small_cfg(L=3, d=256, H=2, f=512, V=512, tpb=16):
    return O.ModelConfig(num_layers=L, hidden_dim=d, num_heads=H, ffn_dim=f, vocab_size=V,
                         tokens_per_block=tpb).validate()


def oracle_weights(cfg, seed=42, max_seq=128):
    return O.prepare_weights(O.generate_weights(cfg, seed, max_seq))


def as_engine_weights(w):
    return {"embedding": w.embedding, "positional": w.positional, "layers": w.layers}


def make_engine(cfg, w, fused=None, **kw):
    """fused: None = the engine's default (recompute fused with attention where
    the heads' width is a multiple of 128), True / False = force the path."""
    from paper_2501_01792_b200.api import Engine, ModelConfig
    mc = ModelConfig(num_layers=cfg.num_layers, hidden_dim=cfg.hidden_dim, num_heads=cfg.num_heads,
                     ffn_dim=cfg.ffn_dim, vocab_size=cfg.vocab_size, tokens_per_block=cfg.tokens_per_block)
    eng = Engine(mc, weights=as_engine_weights(w), **kw)
    if fused is not None:
        assert eng.set_fused_recompute(fused) == fused
    return eng


def run_case(cfg, w, prompts, decode_tokens, **engine_kw):
    """Prefill + len(decode_tokens[0]) teacher-forced decode steps; returns the
    engine outputs per step and the oracle outputs per step."""
    from paper_2501_01792_b200.api import PoolCaps
    n = len(prompts)
    ids = [f"r{i}" for i in range(n)]
    eng = make_engine(cfg, w, max_batch=n, **engine_kw)
    eng.prefill(ids, prompts)
    got, want = [], []
    seqs = [list(p) for p in prompts]
    for s in range(len(decode_tokens[0])):
        toks = [decode_tokens[b][s] for b in range(n)]
        res = eng.decode_step(ids, toks, want_x=True, want_logits=True, want_argmax=True)
        got.append(res)
        ref_x, ref_logits = [], []
        for b in range(n):
            seqs[b].append(toks[b])
            tr = O.forward_prompt(seqs[b], w)
            x = tr.output[-1:]
            ref_x.append(x[0])
            ref_logits.append(O.logits_tied(x, w)[0])
        want.append({"x": np.array(ref_x), "logits": np.array(ref_logits)})
    return eng, ids, got, want


def check_outputs(got, want):
    for g, r in zip(got, want):
        assert rel(f64(g["x"]), r["x"]) <= TOL
        assert rel(g["logits"], r["logits"]) <= TOL
        for b in range(len(g["argmax"])):
            top2 = np.sort(r["logits"][b])[-2:]
            if top2[1] - top2[0] > 2e-2 * np.abs(r["logits"][b]).max():
                assert g["argmax"][b] == int(np.argmax(r["logits"][b]))


def test_engine_resident_act_only_matches_oracle(native):
    """Config-2 shape in miniature: ACT-only cache in HBM, resident weights."""
    from paper_2501_01792_b200.api import PoolCaps
    cfg = small_cfg()
    w = oracle_weights(cfg)
    rng = np.random.default_rng(0)
    prompts = [rng.integers(0, cfg.vocab_size, 37).tolist(), rng.integers(0, cfg.vocab_size, 50).tolist()]
    dec = [rng.integers(0, cfg.vocab_size, 4).tolist() for _ in prompts]
    eng, ids, got, want = run_case(cfg, w, prompts, dec, caps=PoolCaps(act_gpu=16), mode="act_only")
    check_outputs(got, want)
    st = eng.last_stats()
    assert st["h2d_bytes"] == 0 and st["launches"] > 0


@pytest.mark.parametrize("weights_on_device,fused", [(True, True), (False, True), (True, False), (False, False)])
def test_engine_hybrid_offloaded_matches_oracle(native, weights_on_device, fused):
    """Hybrid 1:1 ratio, ACT blocks split GPU/host, KV on host, weights streamed
    or resident, recompute fused with the attention or writing K|V: outputs
    match the oracle and block tables match bit-exactly."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=4, d=256, H=4, f=768)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(1)
    lens = [33, 64, 17]
    prompts = [rng.integers(0, cfg.vocab_size, n).tolist() for n in lens]
    dec = [rng.integers(0, cfg.vocab_size, 5).tolist() for _ in prompts]
    alloc = HostAllocation(20, 20)
    caps = PoolCaps(kv_host=20, act_host=20, act_gpu=3)
    eng, ids, got, want = run_case(cfg, w, prompts, dec, caps=caps, allocation=alloc, mode="hybrid",
                                   weights_on_device=weights_on_device, fused=fused)
    assert eng.fused_recompute() == fused
    check_outputs(got, want)
    # block tables: the oracle's add_token replay in the same call order
    ba = O.BlockAssigner(cfg.tokens_per_block, O.HYBRID, O.HostAllocation(20, 20), act_gpu=3)
    for i, n in enumerate(lens):
        ba.add_request(ids[i], n)
        for _ in range(n):
            ba.add_token(ids[i])
    for _ in range(5):
        for i in range(len(lens)):
            ba.add_token(ids[i])
    assert eng.cache.dump_json() == O.dumps(ba.cache.dump_json())
    st = eng.last_stats()
    assert st["h2d_bytes"] > 0


def test_engine_cache_writers_match_oracle(native):
    """ACT writer (layer inputs X) and KV blocks hold the oracle's X / K / V
    rows after prefill + decode (north-star (1))."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=2, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(2)
    prompt = rng.integers(0, cfg.vocab_size, 29).tolist()
    dec = rng.integers(0, cfg.vocab_size, 3).tolist()
    eng = make_engine(cfg, w, max_batch=1, caps=PoolCaps(kv_host=8, act_host=8, act_gpu=1),
                      allocation=HostAllocation(1, 1))
    eng.prefill(["a"], [prompt])
    for t in dec:
        eng.decode_step(["a"], [t])
    seq = prompt + dec
    tr = O.forward_prompt(seq, w)
    table = eng.cache.table("a")
    assert table.context_len() == len(seq)
    tpb, d, H = cfg.tokens_per_block, cfg.hidden_dim, cfg.num_heads
    row = 0
    for e in table.entries:
        for l in range(cfg.num_layers):
            blk = f64(eng.read_block(e.kind, e.location, e.pbn, l))
            n = e.filled_tokens
            if int(e.kind) == 1:  # ACT: X rows
                assert rel(blk[:n], tr.layer_inputs[l][row:row + n]) <= TOL
            else:
                k = blk[0].transpose(1, 0, 2).reshape(tpb, d)[:n]
                v = blk[1].transpose(1, 0, 2).reshape(tpb, d)[:n]
                assert rel(k, tr.k[l][row:row + n]) <= TOL
                assert rel(v, tr.v[l][row:row + n]) <= TOL
        row += e.filled_tokens


def test_engine_modes_agree(native):
    """kv_only / act_only / hybrid assemble the same context (the reference's
    4-way equivalence, verify.cpp:54-85, at bf16 tolerance)."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=3, d=256, H=2, f=512)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(3)
    prompts = [rng.integers(0, cfg.vocab_size, 45).tolist()]
    toks = [int(rng.integers(0, cfg.vocab_size))]
    outs = {}
    for mode in ("kv_only", "act_only", "hybrid"):
        eng = make_engine(cfg, w, max_batch=1, caps=PoolCaps(kv_host=16, act_host=16, act_gpu=2), mode=mode,
                          allocation=HostAllocation(3, 5))
        eng.prefill(["r"], prompts)
        outs[mode] = f64(eng.decode_step(["r"], toks)["x"])
        eng.close()
    assert rel(outs["act_only"], outs["kv_only"]) <= TOL
    assert rel(outs["hybrid"], outs["kv_only"]) <= TOL


@pytest.mark.parametrize("ratio", [0.5, 1.0])
def test_engine_token_recompute_mode_matches_oracle(native, ratio):
    """Token-recompute baseline (SimMode::TokenRecompute, sim.cpp:196-206): a
    block-aligned prompt prefix is kept as ids only and re-run through every
    layer each step; decode outputs still equal the oracle."""
    from paper_2501_01792_b200.api import PoolCaps
    cfg = small_cfg(L=3, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(6)
    lens = [40, 27]
    prompts = [rng.integers(0, cfg.vocab_size, n).tolist() for n in lens]
    dec = [rng.integers(0, cfg.vocab_size, 3).tolist() for _ in prompts]
    eng, ids, got, want = run_case(cfg, w, prompts, dec, caps=PoolCaps(kv_host=16, kv_gpu=0),
                                   mode="token_recompute", recompute_ratio=ratio)
    check_outputs(got, want)
    from paper_2501_01792_b200 import _native
    import ctypes
    for rid, n in zip(ids, lens):
        rc = (int(ratio * n) // cfg.tokens_per_block) * cfg.tokens_per_block
        assert eng.cache.context_len(rid) == n - rc + 3
    assert eng.last_stats()["recompute_rows"] > 0


def test_engine_greedy_generation_matches_oracle(native):
    """Greedy decode (tied LM head argmax) reproduces the oracle's tokens."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=2, d=256, H=2, f=512)
    w = oracle_weights(cfg, seed=7)
    rng = np.random.default_rng(4)
    prompt = rng.integers(0, cfg.vocab_size, 20).tolist()
    eng = make_engine(cfg, w, max_batch=1, caps=PoolCaps(kv_host=8, act_host=8), allocation=HostAllocation(1, 2))
    eng.prefill(["g"], [prompt])
    seq = list(prompt)
    tok = int(rng.integers(0, cfg.vocab_size))
    for _ in range(6):
        res = eng.decode_step(["g"], [tok], want_logits=True, want_argmax=True)
        seq.append(tok)
        ref = O.logits_tied(O.forward_prompt(seq, w).output[-1:], w)[0]
        top2 = np.sort(ref)[-2:]
        assert rel(res["logits"][0], ref) <= TOL
        if top2[1] - top2[0] > 2e-2 * np.abs(ref).max():
            assert int(res["argmax"][0]) == int(np.argmax(ref))
        tok = int(np.argmax(ref))  # follow the oracle's greedy path


def test_engine_decode_time_layer_inputs(native):
    """Decode-time X per layer equals forward_prompt(prefix+token).layer_inputs
    row pos."""
    from paper_2501_01792_b200.api import PoolCaps
    cfg = small_cfg(L=3)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(5)
    prompt = rng.integers(0, cfg.vocab_size, 30).tolist()
    tok = int(rng.integers(0, cfg.vocab_size))
    eng = make_engine(cfg, w, max_batch=1, caps=PoolCaps(act_gpu=4), mode="act_only")
    eng.prefill(["x"], [prompt])
    eng.capture_inputs(True)
    eng.decode_step(["x"], [tok])
    cap = f64(eng.captured_inputs())
    tr = O.forward_prompt(prompt + [tok], w)
    for l in range(cfg.num_layers):
        assert rel(cap[l, 0], tr.layer_inputs[l][-1]) <= TOL


def test_engine_errors(native):
    from paper_2501_01792_b200 import CapacityError, InputError
    from paper_2501_01792_b200.api import PoolCaps
    cfg = small_cfg(L=1)
    w = oracle_weights(cfg, max_seq=64)
    eng = make_engine(cfg, w, max_batch=2, caps=PoolCaps(act_gpu=2), mode="act_only")
    with pytest.raises(InputError):
        eng.prefill(["a"], [[cfg.vocab_size]])           # token id out of range
    with pytest.raises(InputError):
        eng.decode_step(["nope"], [1])                    # unknown request
    eng.prefill(["a"], [[1] * 32])                        # fills both ACT blocks
    with pytest.raises(CapacityError):
        eng.decode_step(["a"], [1])                       # pools exhausted
    with pytest.raises(InputError):
        eng.prefill(["b"], [[1] * 65])                    # longer than max_seq


@pytest.mark.parametrize("weights_on_device", [True, False])
def test_engine_chunked_offloaded_prefill_matches_oracle(native, weights_on_device):
    """Offloaded prefill pipeline (layer-outer over request chunks; host blocks
    staged in HBM and stored by D2H runs on the store stream): every block of
    every layer holds the oracle's X / K / V rows, the stats count exactly the
    streamed weights and stored blocks, and decode over the result matches."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=3, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(11)
    lens = [29, 40, 8, 51, 16]
    prompts = [rng.integers(0, cfg.vocab_size, n).tolist() for n in lens]
    ids = [f"p{i}" for i in range(len(lens))]
    eng = make_engine(cfg, w, max_batch=len(lens), caps=PoolCaps(kv_host=24, act_host=24, act_gpu=2),
                      allocation=HostAllocation(2, 3), mode="hybrid", weights_on_device=weights_on_device,
                      max_prefill_tokens=60)
    eng.prefill(ids, prompts)
    st = eng.last_stats()
    tpb, d = cfg.tokens_per_block, cfg.hidden_dim
    n_host = {0: 0, 1: 0}
    for rid, p in zip(ids, prompts):
        tr = O.forward_prompt(p, w)
        row = 0
        for e in eng.cache.table(rid).entries:
            if int(e.location) == 0:
                n_host[int(e.kind)] += 1
            n = e.filled_tokens
            for l in range(cfg.num_layers):
                blk = f64(eng.read_block(e.kind, e.location, e.pbn, l))
                if int(e.kind) == 1:
                    assert rel(blk[:n], tr.layer_inputs[l][row:row + n]) <= TOL
                else:
                    k = blk[0].transpose(1, 0, 2).reshape(tpb, d)[:n]
                    v = blk[1].transpose(1, 0, 2).reshape(tpb, d)[:n]
                    assert rel(k, tr.k[l][row:row + n]) <= TOL
                    assert rel(v, tr.v[l][row:row + n]) <= TOL
            row += n
    assert n_host[0] > 0 and n_host[1] > 0
    L = cfg.num_layers
    assert st["d2h_bytes"] == L * 2 * tpb * (n_host[0] * 2 * d + n_host[1] * d)
    layer_bytes = 2 * (4 * d * d + 2 * d * cfg.ffn_dim)
    assert st["h2d_bytes"] == (0 if weights_on_device else L * layer_bytes)
    assert st["step_ms"] > 0
    toks = rng.integers(0, cfg.vocab_size, len(lens)).tolist()
    res = eng.decode_step(ids, toks, want_x=True)
    for b, p in enumerate(prompts):
        ref = O.forward_prompt(p + [toks[b]], w).output[-1]
        assert rel(f64(res["x"][b]), ref) <= TOL


# ---------------------------------------------------------------- OPT arch ---
def opt_weights(cfg, seed=42, max_seq=128):
    return O.with_opt_extras(oracle_weights(cfg, seed, max_seq), seed)


def make_opt_engine(cfg, w, **kw):
    from paper_2501_01792_b200.api import Engine, ModelConfig
    mc = ModelConfig(num_layers=cfg.num_layers, hidden_dim=cfg.hidden_dim, num_heads=cfg.num_heads,
                     ffn_dim=cfg.ffn_dim, vocab_size=cfg.vocab_size, tokens_per_block=cfg.tokens_per_block)
    wd = dict(as_engine_weights(w), extras=w.extras, final_ln=w.final_ln)
    return Engine(mc, weights=wd, arch="opt", **kw)


@pytest.mark.parametrize("weights_on_device", [True, False])
def test_engine_opt_arch_matches_oracle(native, weights_on_device):
    """OPT decoder-layer variant (biases, pre-LN, residuals, final LN; §8(f)
    rank 4): hybrid offloaded prefill + batched decode equal the oracle's
    forward_prompt_opt; ACT blocks hold LN1(x), KV blocks x^ W + b, and the
    recompute (with [b_k|b_v] in the GEMM epilogue) reproduces them."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=3, d=256, H=2, f=512, tpb=8)
    w = opt_weights(cfg)
    rng = np.random.default_rng(21)
    lens = [29, 40, 13]
    prompts = [rng.integers(0, cfg.vocab_size, n).tolist() for n in lens]
    ids = [f"o{i}" for i in range(len(lens))]
    eng = make_opt_engine(cfg, w, max_batch=len(lens), caps=PoolCaps(kv_host=24, act_host=24, act_gpu=2),
                          allocation=HostAllocation(1, 1), mode="hybrid", weights_on_device=weights_on_device,
                          max_prefill_tokens=50)
    eng.prefill(ids, prompts)
    tpb, d = cfg.tokens_per_block, cfg.hidden_dim
    for rid, p in zip(ids, prompts):
        tr = O.forward_prompt_opt(p, w)
        row = 0
        for e in eng.cache.table(rid).entries:
            n = e.filled_tokens
            for l in range(cfg.num_layers):
                blk = f64(eng.read_block(e.kind, e.location, e.pbn, l))
                if int(e.kind) == 1:
                    assert rel(blk[:n], tr.act[l][row:row + n]) <= TOL
                else:
                    assert rel(blk[0].transpose(1, 0, 2).reshape(tpb, d)[:n], tr.k[l][row:row + n]) <= TOL
                    assert rel(blk[1].transpose(1, 0, 2).reshape(tpb, d)[:n], tr.v[l][row:row + n]) <= TOL
            row += n
    seqs = [list(p) for p in prompts]
    for s in range(3):
        toks = rng.integers(0, cfg.vocab_size, len(lens)).tolist()
        res = eng.decode_step(ids, toks, want_x=True, want_logits=True)
        for b in range(len(lens)):
            seqs[b].append(toks[b])
            out = O.forward_prompt_opt(seqs[b], w).output[-1:]
            assert rel(f64(res["x"][b]), out[0]) <= TOL
            assert rel(res["logits"][b], O.logits_tied(out, w)[0]) <= TOL


def test_engine_opt_arch_seeded_extras_and_trace(native):
    """Seeded OPT engine: extras drawn bit-exactly like the oracle's
    generate_opt_extras; forward_trace equals forward_prompt_opt."""
    from paper_2501_01792_b200.api import Engine, ModelConfig, PoolCaps
    cfg = small_cfg(L=2, d=256, H=4, f=512)
    mc = ModelConfig(num_layers=2, hidden_dim=256, num_heads=4, ffn_dim=512, vocab_size=cfg.vocab_size)
    eng = Engine(mc, seed=9, max_seq=64, rescale=True, arch="opt", caps=PoolCaps(act_gpu=8), mode="act_only")
    w = O.with_opt_extras(O.prepare_weights(O.generate_weights(cfg, 9, 64)), 9)
    d, f = 256, 512
    for l in range(2):
        got = eng.read_weights(l)[4 * d * d + 2 * d * f:]
        e = w.extras[l]
        want = np.concatenate([e[k] for k in O.OPT_EXTRAS])
        assert np.array_equal(got, O.to_f16_bits(want))
    assert np.array_equal(eng.read_weights(-3),
                          O.to_f16_bits(np.concatenate([w.final_ln["gamma"], w.final_ln["beta"]])))
    ids = np.random.default_rng(3).integers(0, cfg.vocab_size, 37).tolist()
    tr = eng.forward_trace(ids)
    ref = O.forward_prompt_opt(ids, w)
    assert rel(f64(tr["output"]), ref.output) <= TOL
    for l in range(2):
        assert rel(f64(tr["k"][l]), ref.k[l]) <= TOL
        assert rel(f64(tr["layer_inputs"][l]), ref.layer_inputs[l]) <= TOL


def test_engine_opt_arch_token_recompute(native):
    """Token-recompute baseline on the OPT variant (prefix rebuilt through LN,
    biases and residuals every step)."""
    from paper_2501_01792_b200.api import PoolCaps
    cfg = small_cfg(L=2, d=256, H=2, f=512, tpb=8)
    w = opt_weights(cfg)
    rng = np.random.default_rng(22)
    prompts = [rng.integers(0, cfg.vocab_size, 33).tolist(), rng.integers(0, cfg.vocab_size, 20).tolist()]
    eng = make_opt_engine(cfg, w, max_batch=2, caps=PoolCaps(kv_host=16), mode="token_recompute",
                          recompute_ratio=0.5)
    eng.prefill(["a", "b"], prompts)
    toks = rng.integers(0, cfg.vocab_size, 2).tolist()
    res = eng.decode_step(["a", "b"], toks, want_x=True)
    for b in range(2):
        assert rel(f64(res["x"][b]), O.forward_prompt_opt(prompts[b] + [toks[b]], w).output[-1]) <= TOL


# ------------------------------------------------- tensor parallel (heads) ---
def _run_ranks(fns):
    """Run one callable per tensor-parallel rank concurrently (the in-process
    group rendezvouses inside prefill / decode_step)."""
    import threading
    res, errs = [None] * len(fns), []

    def wrap(i):
        try:
            res[i] = fns[i]()
        except Exception as e:  # noqa: BLE001 — surfaced below
            errs.append(e)

    ts = [threading.Thread(target=wrap, args=(i,), daemon=True) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    if any(t.is_alive() for t in ts):  # a rank stuck in a collective: fail, do not hang the session
        raise TimeoutError("a rank did not finish (collective sequence mismatch?)")
    if errs:
        raise errs[0]
    return res


@pytest.mark.parametrize("tpn,arch,weights_on_device", [(2, "reference", False), (2, "opt", True),
                                                        (4, "reference", True), (4, "opt", False)])
def test_engine_tensor_parallel_matches_oracle(native, tpn, arch, weights_on_device):
    """Head-sharded variant (§8(e)): rank g holds heads [gH/N, (g+1)H/N), a 1/N
    FFN slice and the ACT/host blocks with pbn % N == g (streamed by it, then
    all-gathered); proj / FFN2 partial sums are all-reduced. Every rank's
    decode output equals the oracle, KV blocks hold the rank's heads of the
    oracle's K/V, and ACT blocks sit on their owner rank."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps, TensorParallel
    cfg = small_cfg(L=3, d=256, H=4, f=512, tpb=8)
    w = oracle_weights(cfg) if arch == "reference" else opt_weights(cfg)
    rng = np.random.default_rng(31 + tpn)
    lens = [29, 40, 13]
    prompts = [rng.integers(0, cfg.vocab_size, n).tolist() for n in lens]
    steps = [rng.integers(0, cfg.vocab_size, len(lens)).tolist() for _ in range(3)]
    ids = [f"t{i}" for i in range(len(lens))]
    group = TensorParallel.local_group(tpn)
    kw = dict(max_batch=len(lens), caps=PoolCaps(kv_host=24, act_host=24, act_gpu=2), allocation=HostAllocation(1, 1),
              mode="hybrid", weights_on_device=weights_on_device, max_prefill_tokens=50)
    engs = [(make_opt_engine if arch == "opt" else make_engine)(cfg, w, tp=group[r], **kw) for r in range(tpn)]

    def rank_fn(eng):
        def run():
            eng.prefill(ids, prompts)
            return [eng.decode_step(ids, t, want_x=True, want_logits=True) for t in steps]
        return run

    outs = _run_ranks([rank_fn(e) for e in engs])
    fwd = O.forward_prompt_opt if arch == "opt" else O.forward_prompt
    seqs = [list(p) for p in prompts]
    for s, t in enumerate(steps):
        for b in range(len(lens)):
            seqs[b].append(t[b])
            ref = fwd(seqs[b], w).output[-1:]
            for r in range(tpn):
                assert rel(f64(outs[r][s]["x"][b]), ref[0]) <= TOL
                assert rel(outs[r][s]["logits"][b], O.logits_tied(ref, w)[0]) <= TOL
    # cache contents: KV blocks = the rank's heads; ACT/host blocks on their owner only
    tpb, d, H = cfg.tokens_per_block, cfg.hidden_dim, cfg.num_heads
    hd, Hg = d // H, H // tpn
    for rid, p in zip(ids, prompts):
        tr = fwd(p, w)
        row = 0
        for e in engs[0].cache.table(rid).entries:
            n = min(e.filled_tokens, len(p) - row)
            if n <= 0:
                break
            for r, eng in enumerate(engs):
                heads = slice(r * Hg * hd, (r + 1) * Hg * hd)
                if int(e.kind) == 0:
                    blk = f64(eng.read_block(e.kind, e.location, e.pbn, 1))
                    k = blk[0].transpose(1, 0, 2).reshape(tpb, Hg * hd)[:n]
                    assert rel(k, tr.k[1][row:row + n, heads]) <= TOL
                elif int(e.location) == 0:  # ACT/host: owner rank pbn % N
                    if e.pbn % tpn == r:
                        blk = f64(eng.read_block(e.kind, e.location, e.pbn, 1))
                        want = tr.act[1] if arch == "opt" else tr.layer_inputs[1]
                        assert rel(blk[:n], want[row:row + n]) <= TOL
                    else:
                        with pytest.raises(Exception):
                            eng.read_block(e.kind, e.location, e.pbn, 1)
            row += e.filled_tokens
    # every rank streamed 1/N of the weights
    st = [e.last_stats() for e in engs]
    if not weights_on_device:
        full = 2 * (4 * d * d + 2 * d * cfg.ffn_dim) * cfg.num_layers
        assert all(abs(x["h2d_bytes"] - full / tpn) < full / tpn * 0.5 for x in st)


def test_engine_tensor_parallel_seeded_shards(native):
    """Seeded weights drawn unsharded on the GPU and cut per rank equal the
    matching slices of a single-GPU engine's weights (bit-exact)."""
    from paper_2501_01792_b200.api import Engine, ModelConfig, PoolCaps, TensorParallel
    mc = ModelConfig(num_layers=2, hidden_dim=256, num_heads=4, ffn_dim=512, vocab_size=512)
    full = Engine(mc, seed=5, max_seq=32, caps=PoolCaps(act_gpu=4), mode="act_only", arch="opt")
    group = TensorParallel.local_group(2)
    d, f, dg, fg = 256, 512, 128, 256
    for r in range(2):
        eng = Engine(mc, seed=5, max_seq=32, caps=PoolCaps(act_gpu=4), mode="act_only", arch="opt", tp=group[r],
                     weights_on_device=bool(r))
        for l in range(2):
            F = full.read_weights(l)
            o = 0
            wqkv = F[:3 * d * d].reshape(3, d, d)[:, r * dg:(r + 1) * dg]
            wproj = F[3 * d * d:4 * d * d].reshape(d, d)[:, r * dg:(r + 1) * dg]
            w1 = F[4 * d * d:4 * d * d + f * d].reshape(f, d)[r * fg:(r + 1) * fg]
            w2 = F[4 * d * d + f * d:4 * d * d + 2 * f * d].reshape(d, f)[:, r * fg:(r + 1) * fg]
            ex = F[4 * d * d + 2 * f * d:]
            bqkv = ex[:3 * d].reshape(3, d)[:, r * dg:(r + 1) * dg]
            want = np.concatenate([wqkv.ravel(), wproj.ravel(), w1.ravel(), w2.ravel(), bqkv.ravel(),
                                   ex[3 * d:4 * d], ex[4 * d + r * fg:4 * d + (r + 1) * fg], ex[4 * d + f:]])
            got = eng.read_weights(l)[:want.size]
            assert np.array_equal(got, want), (r, l)
            o += 1
        eng.close()


def test_cpp_caller_decodes(native):
    """examples/decode_demo: a reference-style C++ program linking only the C
    ABI runs prefill + 4 greedy batched decode steps, dumps the block table
    and sees the reference's InputError for an unknown request."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "examples", "decode_demo")
    assert os.path.exists(exe), "examples/decode_demo not built"
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "decode_demo ok" in out.stdout and '"requests"' in out.stdout


@pytest.mark.parametrize("weights_on_device", [True, False])
def test_engine_graph_replay_matches_eager(native, weights_on_device):
    """Decode steps replayed as CUDA graphs (keyed by launch structure, data in
    the uploaded metadata) give bit-identical outputs, stats and block tables
    to eager launches — across block boundaries (new graphs) and reuse."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=3, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(41)
    prompts = [rng.integers(0, cfg.vocab_size, n).tolist() for n in (21, 30)]
    steps = [rng.integers(0, cfg.vocab_size, 2).tolist() for _ in range(12)]
    outs = {}
    for graphs in (False, True):
        eng = make_engine(cfg, w, max_batch=2, caps=PoolCaps(kv_host=16, act_host=16, act_gpu=2),
                          allocation=HostAllocation(1, 1), weights_on_device=weights_on_device)
        eng.set_graphs(graphs)
        eng.prefill(["a", "b"], prompts)
        res = []
        for t in steps:
            r = eng.decode_step(["a", "b"], t, want_x=True, want_logits=True, want_argmax=True)
            st = eng.last_stats()
            res.append((r["x"].copy(), r["logits"].copy(), r["argmax"].copy(), st["h2d_bytes"], st["launches"]))
        outs[graphs] = (res, eng.cache.dump_json())
        eng.close()
    for (a, b) in zip(outs[False][0], outs[True][0]):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
        assert a[3] == b[3] and a[4] == b[4]
    assert outs[False][1] == outs[True][1]


def test_engine_tp_nccl_group_of_one(native):
    """The NCCL path of the head-sharded variant on the box: libnccl is
    dlopen'ed (torch's copy), a 1-rank communicator pair is created, and an
    engine driven through it matches the oracle (collectives degenerate)."""
    import torch  # noqa: F401  (NCCL provider first)
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps, TensorParallel
    cfg = small_cfg(L=2, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg)
    tp = TensorParallel.nccl(TensorParallel.nccl_unique_ids(), 0, 1, 0)
    eng = make_engine(cfg, w, max_batch=1, caps=PoolCaps(kv_host=8, act_host=8), allocation=HostAllocation(1, 1),
                      tp=tp)
    prompt = np.random.default_rng(3).integers(0, cfg.vocab_size, 19).tolist()
    eng.prefill(["n"], [prompt])
    x = f64(eng.decode_step(["n"], [5])["x"][0])
    assert rel(x, O.forward_prompt(prompt + [5], w).output[-1]) <= TOL
    eng.close()


def test_engine_long_greedy_generation_matches_oracle(native):
    """48 greedy steps for 3 requests of different lengths (hybrid host pools,
    streamed weights, CUDA-graph replay across 6+ block boundaries): every
    step's logits match the oracle and the greedy path is followed."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=2, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg, seed=13, max_seq=128)
    rng = np.random.default_rng(51)
    prompts = [rng.integers(0, cfg.vocab_size, n).tolist() for n in (9, 30, 17)]
    ids = ["g0", "g1", "g2"]
    eng = make_engine(cfg, w, max_batch=3, caps=PoolCaps(kv_host=40, act_host=40, act_gpu=3),
                      allocation=HostAllocation(2, 3), weights_on_device=False)
    eng.prefill(ids, prompts)
    seqs = [list(p) for p in prompts]
    toks = [int(rng.integers(0, cfg.vocab_size)) for _ in ids]
    for step in range(48):
        res = eng.decode_step(ids, toks, want_logits=True, want_argmax=True)
        nxt = []
        for b in range(3):
            seqs[b].append(toks[b])
            ref = O.logits_tied(O.forward_prompt(seqs[b], w).output[-1:], w)[0]
            assert rel(res["logits"][b], ref) <= TOL, (step, b)
            top2 = np.sort(ref)[-2:]
            if top2[1] - top2[0] > 2e-2 * np.abs(ref).max():
                assert int(res["argmax"][b]) == int(np.argmax(ref)), (step, b)
            nxt.append(int(np.argmax(ref)))  # follow the oracle's greedy path
        toks = nxt
    assert [eng.cache.context_len(i) for i in ids] == [len(s) for s in seqs]


def test_engine_hbm_resident_kv_and_act_matches_oracle(native):
    """The HBM-resident layout of the bench's hbm_resident variant: KV and ACT
    blocks placed on the GPU first (kv_on_gpu, cache.cpp:64-91) with a small
    KV/host overflow, weights resident — decode outputs equal the oracle and
    the block table equals the reference allocator's."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=3, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(61)
    lens = [25, 40]
    prompts = [rng.integers(0, cfg.vocab_size, n).tolist() for n in lens]
    dec = [rng.integers(0, cfg.vocab_size, 4).tolist() for _ in prompts]
    caps = PoolCaps(kv_host=3, kv_gpu=3, act_gpu=6)
    eng, ids, got, want = run_case(cfg, w, prompts, dec, caps=caps, allocation=HostAllocation(1, 1), mode="hybrid",
                                   kv_on_gpu=True)
    check_outputs(got, want)
    ba = O.BlockAssigner(cfg.tokens_per_block, O.HYBRID, O.HostAllocation(1, 1), act_gpu=6)
    ba.cache = O.HybridCache(cfg.tokens_per_block, kv_host=3, kv_gpu=3, act_host=0, act_gpu=6, kv_on_gpu=True)
    for i, n in enumerate(lens):
        ba.add_request(ids[i], n)
        for _ in range(n):
            ba.add_token(ids[i])
    for _ in range(4):
        for i in range(len(lens)):
            ba.add_token(ids[i])
    assert eng.cache.dump_json() == O.dumps(ba.cache.dump_json())
    locs = {(int(e.kind), int(e.location)) for rid in ids for e in eng.cache.table(rid).entries}
    assert (0, 1) in locs and (1, 1) in locs  # KV/gpu and ACT/gpu blocks both used


def test_engine_empty_prompt_and_partial_batches(native):
    """Edge cases the reference allows: an empty prompt (embed of 0 tokens is
    valid, decoder.cpp:83-95) and decode steps over changing subsets of the
    admitted requests (batch composition changes between graph replays)."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=2, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(71)
    prompts = {"e": [], "a": rng.integers(0, cfg.vocab_size, 13).tolist(), "b": rng.integers(0, cfg.vocab_size, 8).tolist()}
    eng = make_engine(cfg, w, max_batch=3, caps=PoolCaps(kv_host=16, act_host=16, act_gpu=2),
                      allocation=HostAllocation(1, 1))
    eng.prefill(list(prompts), list(prompts.values()))
    seqs = {k: list(v) for k, v in prompts.items()}
    for step, batch in enumerate([["e", "a", "b"], ["a"], ["e", "b"], ["b", "a", "e"], ["e"]]):
        toks = rng.integers(0, cfg.vocab_size, len(batch)).tolist()
        res = eng.decode_step(batch, toks, want_x=True)
        for i, rid in enumerate(batch):
            seqs[rid].append(toks[i])
            ref = O.forward_prompt(seqs[rid], w).output[-1]
            assert rel(f64(res["x"][i]), ref) <= TOL, (step, rid)
    for rid, s in seqs.items():
        assert eng.cache.context_len(rid) == len(s)


def test_engine_failed_configure_cache_is_recoverable(native):
    """A configure_cache whose pools cannot be allocated (here: a KV/gpu pool
    far beyond HBM) raises, leaves the engine refusing work with ConfigError
    instead of touching missing pools, and a later configure_cache with sane
    capacities restores a working engine."""
    from paper_2501_01792_b200 import ConfigError, HcError
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=2, d=256, H=2, f=512, tpb=16)
    w = oracle_weights(cfg)
    eng = make_engine(cfg, w, max_batch=1, caps=PoolCaps(kv_host=8, act_host=8), allocation=HostAllocation(1, 1))
    with pytest.raises(HcError):
        eng.configure_cache(PoolCaps(kv_gpu=1 << 26), mode="kv_only", kv_on_gpu=True)  # ~ 40 TB of KV blocks
    with pytest.raises(ConfigError):
        eng.prefill(["a"], [[1, 2, 3]])
    with pytest.raises(ConfigError):
        eng.decode_step(["a"], [1])
    eng.configure_cache(PoolCaps(kv_host=8, act_host=8), mode="hybrid", allocation=HostAllocation(1, 1))
    prompt = [5, 6, 7, 8, 9]
    eng.prefill(["a"], [prompt])
    res = eng.decode_step(["a"], [11], want_x=True)
    assert rel(f64(res["x"][0]), O.forward_prompt(prompt + [11], w).output[-1]) <= TOL


@pytest.mark.parametrize("n", [2, 3])
def test_engine_shared_weight_stream_matches_oracle(native, n):
    """Batch-partitioned ranks sharing ONE weight stream (Engine(weight_share=)):
    each rank serves its own requests, copies 1/N of every layer's weights over
    its host link and all-gathers the rest. Outputs equal the oracle, graph
    replay is off, and each rank's weight bytes are 1/N of a full stream."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps, TensorParallel
    cfg = small_cfg(L=3, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(97 + n)
    group = TensorParallel.local_group(n)
    kw = dict(max_batch=2, caps=PoolCaps(kv_host=16, act_host=16, act_gpu=1), allocation=HostAllocation(1, 1),
              mode="hybrid", weights_on_device=False)
    engs = [make_engine(cfg, w, weight_share=group[r], **kw) for r in range(n)]
    prompts = [[rng.integers(0, cfg.vocab_size, int(rng.integers(5, 30))).tolist() for _ in range(2)]
               for _ in range(n)]
    steps = [[rng.integers(0, cfg.vocab_size, 2).tolist() for _ in range(4)] for _ in range(n)]

    def rank_fn(r):
        def run():
            ids = [f"r{r}_{i}" for i in range(2)]
            engs[r].prefill(ids, prompts[r])
            return [engs[r].decode_step(ids, t, want_x=True) for t in steps[r]], engs[r].last_stats()
        return run

    outs = _run_ranks([rank_fn(r) for r in range(n)])
    for r in range(n):
        seqs = [list(p) for p in prompts[r]]
        for s, t in enumerate(steps[r]):
            for b in range(2):
                seqs[b].append(t[b])
                ref = O.forward_prompt(seqs[b], w).output[-1]
                assert rel(f64(outs[r][0][s]["x"][b]), ref) <= TOL, (r, s, b)
    full_w = 2 * (4 * cfg.hidden_dim ** 2 + 2 * cfg.hidden_dim * cfg.ffn_dim) * cfg.num_layers
    for r in range(n):
        st = outs[r][1]
        kv_act = st["h2d_bytes"] - full_w / n
        assert -full_w * 0.05 <= kv_act < full_w, (r, st["h2d_bytes"], full_w / n)  # weights ~ 1/N of a stream


def test_engine_shared_weight_stream_uneven_and_failing_ranks(native):
    """Ranks sharing a weight stream issue the same collectives every step even
    when their own work differs: a rank with an empty batch still streams and
    gathers every layer, a rank admitting requests in between (prefill) keeps
    the sequence, and a step one rank rejects (bad token id) fails on every
    rank before the first all-gather — after which all ranks keep decoding."""
    from paper_2501_01792_b200 import InputError
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps, TensorParallel
    cfg = small_cfg(L=3, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg)
    group = TensorParallel.local_group(2)
    kw = dict(max_batch=2, caps=PoolCaps(kv_host=16, act_host=16, act_gpu=1), allocation=HostAllocation(1, 1),
              mode="hybrid", weights_on_device=False)
    engs = [make_engine(cfg, w, weight_share=group[r], **kw) for r in range(2)]
    rng = np.random.default_rng(5)
    prompt = rng.integers(0, cfg.vocab_size, 13).tolist()

    def rank_fn(r):
        def run():
            e, got, errs = engs[r], [], []
            if r == 0:
                e.prefill(["a"], [prompt])
            for step in range(4):
                if r == 1 and step == 2:
                    e.prefill(["b"], [prompt])  # admits between steps: no collectives, sequence intact
                ids = ["a"] if r == 0 else (["b"] if step >= 2 else [])
                toks = [7] if ids else []
                if step == 1:
                    toks = [7] if r == 0 else []
                    if r == 0:
                        toks = [cfg.vocab_size + 5]  # rank 0 rejects this step ...
                try:  # every rank calls decode_step every step, even with nothing to decode
                    x = e.decode_step(ids, toks, want_x=True)["x"].copy()
                    got.append(x if ids else None)
                except InputError as ex:
                    errs.append((step, str(ex)))
            return got, errs
        return run

    outs = _run_ranks([rank_fn(r) for r in range(2)])
    for r in range(2):
        assert [s for s, _ in outs[r][1]] == [1], outs[r][1]  # ... and every rank raised at step 1
    assert "token id out of range" in outs[0][1][0][1] and "rejected" in outs[1][1][0][1]
    seq = list(prompt)
    for x in outs[0][0]:
        seq.append(7)
        assert rel(f64(x[0]), O.forward_prompt(seq, w).output[-1]) <= TOL
    seq = list(prompt)
    assert outs[1][0][0] is None
    for x in outs[1][0][1:]:
        seq.append(7)
        assert rel(f64(x[0]), O.forward_prompt(seq, w).output[-1]) <= TOL


def test_engine_shared_weight_stream_rejects_tp_and_resident(native):
    from paper_2501_01792_b200 import ConfigError
    from paper_2501_01792_b200.api import TensorParallel
    cfg = small_cfg(L=1)
    w = oracle_weights(cfg, max_seq=64)
    g = TensorParallel.local_group(2)
    with pytest.raises(ConfigError):
        make_engine(cfg, w, weight_share=g[0], weights_on_device=True)
    t = TensorParallel.local_group(2)
    with pytest.raises(ConfigError):
        make_engine(cfg, w, weight_share=g[0], tp=t[0], weights_on_device=False)


def test_engine_capacity_error_leaves_batch_untouched(native):
    """A decode step whose new blocks do not fit raises CapacityError before
    any context grows (the reference's append leaves the table untouched,
    cache.cpp:91, 98): after freeing a request the survivors decode on and
    still match the oracle, and their tables equal a run that never failed."""
    from paper_2501_01792_b200 import CapacityError
    from paper_2501_01792_b200.api import PoolCaps
    cfg = small_cfg(L=2, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(5)
    # three requests at a block boundary, pools with room for exactly two more ACT blocks
    prompts = {r: rng.integers(0, cfg.vocab_size, 16).tolist() for r in ("a", "b", "c")}
    eng = make_engine(cfg, w, max_batch=3, caps=PoolCaps(act_gpu=8), mode="act_only")
    eng.prefill(list(prompts), list(prompts.values()))
    before = eng.cache.dump_json()
    with pytest.raises(CapacityError):
        eng.decode_step(["a", "b", "c"], [1, 2, 3])
    assert eng.cache.dump_json() == before                 # nothing half-applied
    eng.free_request("c")
    seqs = {k: list(v) for k, v in prompts.items() if k != "c"}
    for step in range(3):
        toks = rng.integers(0, cfg.vocab_size, 2).tolist()
        res = eng.decode_step(["a", "b"], toks, want_x=True)
        for i, rid in enumerate(["a", "b"]):
            seqs[rid].append(toks[i])
            assert rel(f64(res["x"][i]), O.forward_prompt(seqs[rid], w).output[-1]) <= TOL, (step, rid)
    for rid, s in seqs.items():
        assert eng.cache.context_len(rid) == len(s)


def test_engine_prefill_capacity_error_admits_none(native):
    """A prefill whose prompts do not all fit raises CapacityError and admits
    none of them (the pools are as before); a smaller prefill then works."""
    from paper_2501_01792_b200 import CapacityError
    from paper_2501_01792_b200.api import PoolCaps
    cfg = small_cfg(L=2, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg)
    rng = np.random.default_rng(6)
    eng = make_engine(cfg, w, max_batch=3, caps=PoolCaps(act_gpu=5), mode="act_only")
    before = eng.cache.dump_json()
    big = [rng.integers(0, cfg.vocab_size, 12).tolist() for _ in range(3)]   # 3 x 2 blocks > 5
    with pytest.raises(CapacityError):
        eng.prefill(["a", "b", "c"], big)
    assert eng.cache.dump_json() == before
    eng.prefill(["a", "b"], big[:2])
    res = eng.decode_step(["a", "b"], [7, 8], want_x=True)
    for i in range(2):
        assert rel(f64(res["x"][i]), O.forward_prompt(big[i] + [7 + i], w).output[-1]) <= TOL


@pytest.mark.parametrize("seed,mode,arch", [(1, "hybrid", "reference"), (2, "hybrid", "reference"),
                                             (3, "kv_only", "reference"), (4, "act_only", "reference"),
                                             (5, "hybrid", "opt")])
def test_engine_fuzz_against_oracle(native, seed, mode, arch):
    """Randomised serving session on small pools (the end-to-end analogue of the
    reference's cache fuzz, test_cache.cpp:143-217): admit prompts (empty
    included), decode random subsets, free requests, hit pool exhaustion.
    Every decode output equals the oracle's forward over the request's tokens,
    every CapacityError leaves the block tables unchanged, and the tables stay
    consistent with the token counts."""
    from paper_2501_01792_b200 import CapacityError
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=2, d=256, H=2, f=512, tpb=8)
    w = opt_weights(cfg, max_seq=96) if arch == "opt" else oracle_weights(cfg, max_seq=96)
    fwd = O.forward_prompt_opt if arch == "opt" else O.forward_prompt
    # the OPT variant rounds three LayerNorm outputs per layer (and the final LN) to fp16
    # — the reference decoder has none; the bar is the same 1e-2
    tol = TOL_OPT if arch == "opt" else TOL
    rng = np.random.default_rng(1000 + seed)
    caps = PoolCaps(kv_host=14, act_host=10, act_gpu=3) if mode == "hybrid" else (
        PoolCaps(kv_host=20) if mode == "kv_only" else PoolCaps(act_host=12, act_gpu=6))
    eng = (make_opt_engine if arch == "opt" else make_engine)(cfg, w, max_batch=4, max_seq=96, caps=caps, mode=mode,
                      allocation=HostAllocation(int(rng.integers(1, 4)), int(rng.integers(1, 4))),
                      weights_on_device=bool(seed % 2))
    seqs, next_id, checked, exhausted = {}, 0, 0, 0
    for op in range(70):
        live = list(seqs)
        r = rng.random()
        if (r < 0.25 and len(live) < 4) or not live:
            n_new = int(rng.integers(1, min(2, 4 - len(live)) + 1))
            ids = [f"q{next_id + i}" for i in range(n_new)]
            prompts = [rng.integers(0, cfg.vocab_size, int(rng.integers(0, 30))).tolist() for _ in ids]
            before = eng.cache.dump_json()
            try:
                eng.prefill(ids, prompts)
            except CapacityError:
                assert eng.cache.dump_json() == before
                exhausted += 1
                continue
            next_id += n_new
            seqs.update({i: list(p) for i, p in zip(ids, prompts)})
        elif r < 0.35:
            victim = live[int(rng.integers(0, len(live)))]
            eng.free_request(victim)
            del seqs[victim]
        else:
            batch = [x for x in live if rng.random() < 0.7] or live[:1]
            batch = [x for x in batch if len(seqs[x]) < 90]
            if not batch:
                continue
            toks = rng.integers(0, cfg.vocab_size, len(batch)).tolist()
            before = eng.cache.dump_json()
            try:
                res = eng.decode_step(batch, toks, want_x=True)
            except CapacityError:
                assert eng.cache.dump_json() == before
                exhausted += 1
                continue
            for i, rid in enumerate(batch):
                seqs[rid].append(toks[i])
                ref = fwd(seqs[rid], w).output[-1]
                assert rel(f64(res["x"][i]), ref) <= tol, (op, rid, len(seqs[rid]))
                checked += 1
        for rid, s in seqs.items():
            assert eng.cache.context_len(rid) == len(s)
    assert checked > 40


@pytest.mark.parametrize("tpn,seed", [(2, 11), (2, 12)])
def test_engine_tensor_parallel_fuzz(native, tpn, seed):
    """The serving fuzz on the head-sharded variant: every rank runs the same
    randomised session (same ids, tokens, frees, pool exhaustion) in its own
    thread; all ranks' outputs equal the oracle and their block tables agree."""
    from paper_2501_01792_b200 import CapacityError
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps, TensorParallel
    cfg = small_cfg(L=2, d=256, H=4, f=512, tpb=8)
    w = oracle_weights(cfg, max_seq=96)
    group = TensorParallel.local_group(tpn)
    engs = [make_engine(cfg, w, max_batch=3, max_seq=96, caps=PoolCaps(kv_host=12, act_host=10, act_gpu=2),
                        mode="hybrid", allocation=HostAllocation(1, 1), weights_on_device=bool(seed % 2),
                        tp=group[r]) for r in range(tpn)]

    def session(r):
        def run():
            rng = np.random.default_rng(seed)
            eng, seqs, next_id, outs = engs[r], {}, 0, []
            for op in range(40):
                live = list(seqs)
                u = rng.random()
                if (u < 0.3 and len(live) < 3) or not live:
                    ids = [f"t{next_id}"]
                    prompts = [rng.integers(0, cfg.vocab_size, int(rng.integers(0, 25))).tolist()]
                    try:
                        eng.prefill(ids, prompts)
                    except CapacityError:
                        continue
                    next_id += 1
                    seqs[ids[0]] = list(prompts[0])
                elif u < 0.4:
                    victim = live[int(rng.integers(0, len(live)))]
                    eng.free_request(victim)
                    del seqs[victim]
                else:
                    batch = [x for x in live if len(seqs[x]) < 90]
                    if not batch:
                        continue
                    toks = rng.integers(0, cfg.vocab_size, len(batch)).tolist()
                    try:
                        res = eng.decode_step(batch, toks, want_x=True)
                    except CapacityError:
                        continue
                    for i, rid in enumerate(batch):
                        seqs[rid].append(toks[i])
                        outs.append((rid, list(seqs[rid]), f64(res["x"][i])))
            return outs, eng.cache.dump_json()
        return run

    results = _run_ranks([session(r) for r in range(tpn)])
    assert all(res[1] == results[0][1] for res in results)  # identical bookkeeping on every rank
    assert len(results[0][0]) > 20
    for outs, _ in results:
        for rid, seq, x in outs:
            assert rel(x, O.forward_prompt(seq, w).output[-1]) <= TOL, (rid, len(seq))


@pytest.mark.parametrize("B,tpb,mode,fused", [(200, 16, "hybrid", True), (64, 32, "act_only", True),
                                              (96, 4, "kv_only", True), (48, 64, "hybrid", True),
                                              (40, 4, "act_only", True), (40, 8, "hybrid", True),
                                              (200, 16, "hybrid", False), (48, 64, "hybrid", False)])
def test_engine_large_batches_and_block_sizes(native, B, tpb, mode, fused):
    """Edge sizes the reference allows: hundreds of requests in one decode
    step (grid = B x heads, staging sized for every host block) and block
    sizes other than 16 (tokens_per_block is a model parameter, model.hpp:22):
    outputs equal the oracle for every request."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=2, d=256, H=2, f=512, tpb=tpb)
    w = oracle_weights(cfg, max_seq=64)
    rng = np.random.default_rng(B + tpb)
    lens = rng.integers(1, 40, B).tolist()
    per = max(-(-(n + 3) // tpb) for n in lens) + 1
    caps = PoolCaps(kv_host=B * per, act_host=B * per, act_gpu=B // 2)
    eng = make_engine(cfg, w, max_batch=B, max_seq=64, caps=caps, mode=mode, allocation=HostAllocation(1, 1),
                      weights_on_device=False, fused=fused)
    ids = [f"b{i}" for i in range(B)]
    prompts = [rng.integers(0, cfg.vocab_size, n).tolist() for n in lens]
    eng.prefill(ids, prompts)
    seqs = [list(p) for p in prompts]
    for step in range(3):
        toks = rng.integers(0, cfg.vocab_size, B).tolist()
        res = eng.decode_step(ids, toks, want_x=True)
        for b in range(0, B, 7 if B > 100 else 3):  # a spread of requests (oracle cost)
            seqs[b].append(toks[b])
            ref = O.forward_prompt(seqs[b], w).output[-1]
            assert rel(f64(res["x"][b]), ref) <= TOL, (step, b)
        for b in range(B):
            if b % (7 if B > 100 else 3):
                seqs[b].append(toks[b])


@pytest.mark.parametrize("hd,tpb,scaled", [(128, 16, True), (64, 16, True), (128, 4, True), (64, 8, False),
                                           (128, 32, False), (64, 64, True)])
def test_fused_recompute_attention_agrees_with_kv_paged_path(native, hd, tpb, scaled):
    """The fused recompute + attention path (kAttnPart partial records merged by
    decode_attention) against the kKvPaged path (K|V written to the paged
    layout, attention reads them): two engines, same weights, prompts and
    tokens, ACT blocks resident and streamed, ragged contexts (partially filled
    last blocks, 128-row tiles shared by several requests). The same f16 K|V
    meet the same queries, so the outputs agree to accumulation order, and both
    match the oracle."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    H = 4
    cfg = small_cfg(L=2, d=H * hd, H=H, f=512, tpb=tpb)
    w = oracle_weights(cfg, max_seq=160)
    rng = np.random.default_rng(hd + tpb)
    B = 9
    lens = rng.integers(1, 120, B).tolist()
    per = max(-(-(n + 4) // tpb) for n in lens) + 1
    caps = PoolCaps(kv_host=B * per, act_host=B * per, act_gpu=B * per // 3)
    engs = [make_engine(cfg, w, max_batch=B, max_seq=160, caps=caps, mode="hybrid", allocation=HostAllocation(3, 1),
                        weights_on_device=False, scaled=scaled, fused=f) for f in (True, False)]
    ids = [f"f{i}" for i in range(B)]
    prompts = [rng.integers(0, cfg.vocab_size, n).tolist() for n in lens]
    for e in engs:
        e.prefill(ids, prompts)
    seqs = [list(p) for p in prompts]
    for step in range(3):
        toks = rng.integers(0, cfg.vocab_size, B).tolist()
        fused, paged = (e.decode_step(ids, toks, want_x=True, want_logits=True) for e in engs)
        assert rel(f64(fused["x"]), f64(paged["x"])) <= 2e-3, step
        assert rel(fused["logits"], paged["logits"]) <= 2e-3, step
        for b in range(B):
            seqs[b].append(toks[b])
            ref = O.forward_prompt(seqs[b], w, scaled=scaled).output[-1]
            assert rel(f64(fused["x"][b]), ref) <= TOL, (step, b)
    assert engs[0].last_stats()["recompute_rows"] > 0


def test_engine_rejects_unsupported_block_size(native):
    """tokens_per_block outside the instantiated set fails at construction
    (InputError), not in the middle of a decode step."""
    from paper_2501_01792_b200 import InputError
    cfg = small_cfg(L=1, tpb=3)
    w = oracle_weights(cfg, max_seq=32)
    with pytest.raises(InputError):
        make_engine(cfg, w, max_batch=1)


def test_engine_reconfigure_across_modes(native):
    """One engine reconfigured through every cache mode and pool shape in turn
    (what the bench's sweeps do): each configuration's decode outputs equal
    the oracle — no graph, prefetch or pool state leaks across configure_cache."""
    from paper_2501_01792_b200.api import HostAllocation, PoolCaps
    cfg = small_cfg(L=2, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg, max_seq=64)
    rng = np.random.default_rng(77)
    eng = make_engine(cfg, w, max_batch=2, max_seq=64, weights_on_device=False,
                      caps=PoolCaps(kv_host=16), mode="kv_only")
    plans = [("kv_only", PoolCaps(kv_host=16), HostAllocation(0, 1), {}),
             ("hybrid", PoolCaps(kv_host=12, act_host=12, act_gpu=2), HostAllocation(1, 2), {}),
             ("act_only", PoolCaps(act_host=4, act_gpu=10), HostAllocation(1, 0), {}),
             ("hybrid", PoolCaps(kv_host=6, kv_gpu=6, act_gpu=8), HostAllocation(2, 1), {"kv_on_gpu": True}),
             ("token_recompute", PoolCaps(kv_host=16), HostAllocation(1, 1), {"recompute_ratio": 0.5}),
             ("hybrid", PoolCaps(kv_host=12, act_host=12), HostAllocation(1, 1), {"host_layers": 1})]
    for i, (mode, caps, alloc, kw) in enumerate(plans * 2):
        eng.configure_cache(caps, mode=mode, allocation=alloc, **kw)
        prompts = [rng.integers(0, cfg.vocab_size, int(rng.integers(5, 30))).tolist() for _ in range(2)]
        ids = [f"c{i}a", f"c{i}b"]
        eng.prefill(ids, prompts)
        seqs = [list(p) for p in prompts]
        for step in range(3):
            toks = rng.integers(0, cfg.vocab_size, 2).tolist()
            res = eng.decode_step(ids, toks, want_x=True)
            for b in range(2):
                seqs[b].append(toks[b])
                if kw.get("host_layers"):
                    continue  # folded host pools (a benchmark device): payloads alias across layers
                ref = O.forward_prompt(seqs[b], w).output[-1]
                assert rel(f64(res["x"][b]), ref) <= TOL, (i, mode, step, b)


@pytest.mark.parametrize("weights_on_device,graphs", [(False, True), (True, False)])
def test_engine_minibatched_decode_matches_oracle(native, weights_on_device, graphs):
    """Mini-batched decode (paper §4.3.3; sim.cpp:258-358): staging slots capped
    so every step splits into >= 2 (layer, mini-batch) units packed by
    form_minibatches on PRE-growth block counts (minibatch.cpp:36-83). Outputs
    equal the oracle; the block tables equal the oracle's add_token replay in
    the reference's mini-batch order (sim.cpp:294-310); the prefill writes its
    host blocks straight into the pinned pools (the staging is smaller)."""
    from paper_2501_01792_b200.api import HostAllocation, LinearTimeModel, PoolCaps, TimingBundle
    cfg = small_cfg(L=3, d=256, H=2, f=512, tpb=8)
    w = oracle_weights(cfg, seed=21, max_seq=96)
    rng = np.random.default_rng(77)
    lens = [23, 40, 9, 31, 17]
    prompts = [rng.integers(0, cfg.vocab_size, n).tolist() for n in lens]
    ids = [f"m{i}" for i in range(len(lens))]
    alloc = HostAllocation(3, 2)
    caps = PoolCaps(kv_host=40, act_host=40, act_gpu=2)
    eng = make_engine(cfg, w, max_batch=len(ids), caps=caps, allocation=alloc, mode="hybrid",
                      weights_on_device=weights_on_device)
    eng.set_graphs(graphs)
    bundle = TimingBundle(LinearTimeModel(1e-7, 1e-5), LinearTimeModel(5e-7, 0.0), 0.02)
    act_max, kv_max = 6, 5
    eng.set_minibatching(act_max, kv_max, bundle)
    eng.prefill(ids, prompts)
    ba = O.BlockAssigner(cfg.tokens_per_block, O.HYBRID, O.HostAllocation(3, 2), act_gpu=2)
    ba.cache = O.HybridCache(cfg.tokens_per_block, 40, 0, 40, 2)  # the engine's pools; (3, 2) is only the target
    for rid, n in zip(ids, lens):
        ba.add_request(rid, n)
        for _ in range(n):
            ba.add_token(rid)
    ob = O.TimingBundle(O.LinearTimeModel(1e-7, 1e-5), O.LinearTimeModel(5e-7, 0.0), 0.02)
    seqs = [list(p) for p in prompts]
    n_mb = []
    for step in range(5):
        toks = [int(t) for t in rng.integers(0, cfg.vocab_size, len(ids))]
        # the reference's order: pack on pre-growth counts, grow mini-batch by mini-batch
        reqs = [(rid, *ba.cache.table(rid).blocks_by_kind()) for rid in ids]
        for mb in O.form_minibatches(reqs, act_max, kv_max, ob, cfg.tokens_per_block):
            for rid in mb:
                ba.add_token(rid)
        res = eng.decode_step(ids, toks, want_x=True, want_logits=True, want_argmax=True)
        n_mb.append(eng.last_stats()["minibatches"])
        for b in range(len(ids)):
            seqs[b].append(toks[b])
            x = O.forward_prompt(seqs[b], w).output[-1:]
            assert rel(f64(res["x"][b]), x[0]) <= TOL, (step, b)
            assert rel(res["logits"][b], O.logits_tied(x, w)[0]) <= TOL, (step, b)
        assert eng.cache.dump_json() == O.dumps(ba.cache.dump_json()), step
    assert min(n_mb) >= 2, n_mb
    # a request larger than the staging: CapacityError, tables untouched
    from paper_2501_01792_b200 import CapacityError
    before = eng.cache.dump_json()
    eng.set_minibatching(1, 1, bundle)
    with pytest.raises(CapacityError):
        eng.decode_step(ids, toks)
    assert eng.cache.dump_json() == before
    eng.set_minibatching(0, 0)
    res = eng.decode_step(ids, toks, want_x=True)
    assert eng.last_stats()["minibatches"] == 1
    eng.close()


@pytest.mark.parametrize("env", [{"HC_WSTREAM": "0"}, {"HC_PREFILL_PTMEM": "0"}, {"HC_PREFILL_PTMEM": "2"}])
def test_engine_kernel_alternatives_match_oracle(native, env):
    """The A/B knobs' alternative kernels stay correct: decode-batch GEMMs on the
    tile kernel + split-K instead of wstream, prefill attention with P in smem
    (or in TMEM at head_dim 64 too). The knobs are read once per process, so the
    engine parity tests run again in a child process with the knob set."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_engine_gpu.py"),
                        "-k", "resident_act_only or hybrid_offloaded or opt_arch or large_batches"],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
