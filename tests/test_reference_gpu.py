"""GPU path vs vectors computed by the UNMODIFIED reference (tests/golden,
made by tests/golden/make_golden.py from oracle/_ref), plus the reference's
4-way context-assembly equivalence (verify.cpp:26-95) at bf16 tolerance over
seeded random models.

Weights: the engine draws DecoderWeights::generate itself (bit-exact with the
reference, tests/test_host_cpu.py) + the documented rescale + bf16; the
golden vectors were computed by the reference on exactly those bf16 values.
"""
import os

import numpy as np
import pytest

import hybridsim_oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-2


def rel(got, ref):
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def f64(bits):
    return O.f16_bits_to_f64(np.asarray(bits))


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "golden.npz"))


CASES = {"toy_rescaled": ((3, 256, 2, 512, 512, 16), 7, 40),
         "opt125m_shape": ((12, 768, 12, 3072, 50272, 16), 42, 160)}


def engine_for(tag, **kw):
    from paper_2501_01792_b200 import api
    (L, d, H, f, V, tpb), seed, max_seq = CASES[tag]
    cfg = api.ModelConfig(num_layers=L, hidden_dim=d, num_heads=H, ffn_dim=f, vocab_size=V, tokens_per_block=tpb)
    return api.Engine(cfg, seed=seed, max_seq=max_seq, rescale=True, **kw)


@pytest.mark.parametrize("tag", list(CASES))
def test_layer_forward_teacher_forced_matches_reference(gold, tag):
    """Each layer on the reference's own input X^l (bf16-rounded): K^l, V^l
    and X^{l+1} within 1e-2 of the reference (qkv_generate + attention_causal +
    project_ffn, decoder.cpp:150-153)."""
    eng = engine_for(tag, max_batch=1)
    X = gold[f"{tag}/layer_inputs"]
    L = X.shape[0]
    for l in range(L):
        r = eng.layer_forward(l, O.to_f16_bits(X[l]))
        nxt = X[l + 1] if l + 1 < L else gold[f"{tag}/output"]
        assert rel(f64(r["k"]), gold[f"{tag}/k"][l]) <= TOL, l
        assert rel(f64(r["v"]), gold[f"{tag}/v"][l]) <= TOL, l
        assert rel(f64(r["output"]), nxt) <= TOL, l


@pytest.mark.parametrize("tag", list(CASES))
def test_forward_trace_matches_reference(gold, tag):
    """forward_prompt (decoder.cpp:144-157) end to end: every layer's input X
    (the ACT checkpoints), K, V and the output vs the reference's fp64 values."""
    eng = engine_for(tag, max_batch=1)
    ids = gold[f"{tag}/ids"].tolist()
    tr = eng.forward_trace(ids)
    L = tr["k"].shape[0]
    for l in range(L):
        assert rel(f64(tr["layer_inputs"][l]), gold[f"{tag}/layer_inputs"][l]) <= TOL, l
        assert rel(f64(tr["k"][l]), gold[f"{tag}/k"][l]) <= TOL, l
        assert rel(f64(tr["v"][l]), gold[f"{tag}/v"][l]) <= TOL, l
    assert rel(f64(tr["output"]), gold[f"{tag}/output"]) <= TOL


@pytest.mark.parametrize("tag", list(CASES))
@pytest.mark.parametrize("mode", ["kv_only", "act_only", "hybrid"])
def test_decode_step_matches_reference_generation_step(gold, tag, mode):
    """Prefill the golden prompt, decode the golden token: output and the new
    token's K,V equal the reference's generation_step (decoder.cpp:159-174)."""
    from paper_2501_01792_b200 import api
    eng = engine_for(tag, max_batch=1, caps=api.PoolCaps(kv_host=4, act_host=4, act_gpu=1), mode=mode,
                     allocation=api.HostAllocation(1, 1), weights_on_device=(mode != "hybrid"))
    ids = gold[f"{tag}/ids"].tolist()
    tok = int(gold[f"{tag}/gen_token"][0])
    eng.prefill(["r"], [ids])
    res = eng.decode_step(["r"], [tok])
    assert rel(f64(res["x"]), gold[f"{tag}/gen_output"]) <= TOL
    # the new token's K,V were written into its block at every layer
    t = eng.cache.table("r")
    e = t.entries[-1]
    row = e.filled_tokens - 1
    L, d = gold[f"{tag}/gen_k"].shape
    H = eng.cfg.num_heads
    for l in range(L):
        blk = f64(eng.read_block(e.kind, e.location, e.pbn, l))
        if int(e.kind) == 0:
            k = blk[0, :, row, :].reshape(d)
            v = blk[1, :, row, :].reshape(d)
            assert rel(k, gold[f"{tag}/gen_k"][l]) <= TOL
            assert rel(v, gold[f"{tag}/gen_v"][l]) <= TOL


def test_token_recompute_kv_gpu():
    """token_recompute_kv (decoder.cpp:131-142) == forward capture at layer k."""
    from paper_2501_01792_b200 import api
    cfg = api.ModelConfig(num_layers=4, hidden_dim=256, num_heads=2, ffn_dim=512, vocab_size=256)
    eng = api.Engine(cfg, seed=31, max_seq=32, max_batch=1)
    ids = [2, 7, 1, 12, 0, 5, 11, 3]
    ocfg = O.ModelConfig(num_layers=4, hidden_dim=256, num_heads=2, ffn_dim=512, vocab_size=256).validate()
    w = O.prepare_weights(O.generate_weights(ocfg, 31, 32))
    for k in range(4):
        gk, gv = eng.token_recompute_kv(ids, k)
        ok, ov = O.token_recompute_kv(ids, w, k)
        assert rel(f64(gk), ok) <= TOL and rel(f64(gv), ov) <= TOL
    from paper_2501_01792_b200 import InputError
    with pytest.raises(InputError):
        eng.token_recompute_kv(ids, 4)


@pytest.mark.parametrize("seed,scaled", [(s, True) for s in range(25)] + [(3, False), (11, False)])
def test_equivalence_seeded_models(seed, scaled):
    """run_equivalence_case (verify.cpp:26-95) on the GPU over the reference's 25
    seeds (test_decoder.cpp:290-295) plus its unscaled-attention case
    (:296-298): a seeded random model, its context held as stored KV, as ACT
    checkpoints (recomputed), as token-recompute and as a block-wise mix; the
    decode output is the same for all (within the 16-bit tolerance) and
    equals the oracle. Shapes are the reference's draw mapped onto the
    engine's supported widths (head_dim 64/128, tokens_per_block 8/16)."""
    from paper_2501_01792_b200 import api
    rng = O.SplitMix64(O.mix_seed(seed, 0x657175))
    L = rng.uniform_int(1, 4)
    H = [1, 2, 4][rng.uniform_int(0, 2)]
    d = 128 * H if rng.uniform_int(0, 1) else 64 * H
    tpb = [8, 16][rng.uniform_int(0, 1)]
    P = rng.uniform_int(3, 60)
    cfg = api.ModelConfig(num_layers=L, hidden_dim=d, num_heads=H, ffn_dim=2 * d, vocab_size=64,
                          tokens_per_block=tpb)
    wseed = O.mix_seed(seed, 0x77)
    ids = [rng.uniform_int(0, 63) for _ in range(P)]
    tok = rng.uniform_int(0, 63)
    eng = api.Engine(cfg, seed=wseed, max_seq=P + 2, max_batch=1, scaled=scaled)
    outs, stats = {}, {}
    for mode, alloc, rc in (("kv_only", None, 0.0), ("act_only", None, 0.0), ("hybrid", api.HostAllocation(1, 1), 0.0),
                            ("token_recompute", None, 0.5)):
        eng.configure_cache(api.PoolCaps(kv_host=8, act_host=8, act_gpu=2), mode=mode, allocation=alloc,
                            recompute_ratio=rc)
        eng.prefill(["q"], [ids])
        eng.set_profile(True)
        outs[mode] = f64(eng.decode_step(["q"], [tok])["x"])
        stats[mode] = (eng.last_stats(), eng.cache.dump_json())
    ocfg = O.ModelConfig(num_layers=L, hidden_dim=d, num_heads=H, ffn_dim=2 * d, vocab_size=64).validate()
    w = O.prepare_weights(O.generate_weights(ocfg, wseed, P + 2))
    ref = O.forward_prompt(ids + [tok], w, scaled).output[-1:]
    for m, o in outs.items():
        assert rel(o, ref) <= TOL, (m, stats[m], (L, H, d, tpb, P))
    assert rel(outs["act_only"], outs["kv_only"]) <= TOL
    assert rel(outs["hybrid"], outs["kv_only"]) <= TOL
    assert rel(outs["token_recompute"], outs["kv_only"]) <= TOL


@pytest.mark.parametrize("on_device", [True, False])
def test_gpu_weight_generation_bit_exact(on_device):
    """DecoderWeights::generate drawn on the GPU (weights_gen.cu) equals the
    host generator (itself bit-exact with the reference draws) bit for bit."""
    from paper_2501_01792_b200 import api
    cfg = api.ModelConfig(num_layers=2, hidden_dim=256, num_heads=2, ffn_dim=768, vocab_size=320)
    host = api.generate_weights(cfg, 1234, 48, rescale=True)
    eng = api.Engine(cfg, seed=1234, max_seq=48, rescale=True, weights_on_device=on_device)
    assert np.array_equal(eng.read_weights(-1), host["embedding"])
    assert np.array_equal(eng.read_weights(-2), host["positional"])
    for l in range(2):
        assert np.array_equal(eng.read_weights(l), host["layers"][l])


def test_full_width_opt30b_layer_parity():
    """One OPT-30B-width layer (d 7168, 56 heads, f 28672) through the offloaded
    hybrid engine: prefill + 3 decode steps, and the cache blocks, within 1e-2 of
    the fp64 oracle (scripts/full_width_parity.py; ~30 s, ~10 GB host RAM)."""
    import importlib.util
    import os
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts", "full_width_parity.py")
    spec = importlib.util.spec_from_file_location("full_width_parity", p)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.main([])


@pytest.mark.parametrize("weights_on_device", [False, True])
def test_config1_greedy_matches_reference(gold, weights_on_device):
    """BASELINE configs[0] exactly: OPT-125M shape (12 layers, d 768, vocab
    50272), 4 requests, prompt 128, 32 greedy tokens, KV:ACT 0.5
    (HostAllocation{K, K}: ACT, KV, ACT, ... blocks in pinned host pools).
    Against the golden run of the UNMODIFIED reference (make_golden.py
    config1_case: forward_prompt + recompute_kv_from_activation +
    generation_step, tied head): every step's output x and full-vocabulary
    logits within 1e-2, every greedy token equal (the GPU's argmax is what is
    fed back), block tables equal the oracle's add_token replay."""
    from paper_2501_01792_b200 import api
    B, P, G, tpb = 4, 128, 32, 16
    prompts = gold["config1/prompts"]
    fed, toks, xs, margin = gold["config1/fed"], gold["config1/tokens"], gold["config1/x"], gold["config1/margin"]
    K = B * ((P + G + tpb - 1) // tpb)
    cfg = api.ModelConfig(num_layers=12, hidden_dim=768, num_heads=12, ffn_dim=3072, vocab_size=50272)
    eng = api.Engine(cfg, seed=42, max_seq=P + G + 1, rescale=True, max_batch=B, weights_on_device=weights_on_device,
                     caps=api.PoolCaps(kv_host=K, act_host=K), allocation=api.HostAllocation(K, K), mode="hybrid")
    E = f64(eng.read_weights(-1)).reshape(cfg.vocab_size, cfg.hidden_dim)
    ids = [f"c1r{b}" for b in range(B)]
    eng.prefill(ids, [p[:-1].tolist() for p in prompts])
    cur = [int(p[-1]) for p in prompts]
    worst = 0.0
    for s in range(G):
        assert cur == fed[s].tolist(), s  # the GPU's own greedy path is the reference's
        res = eng.decode_step(ids, cur, want_x=True, want_logits=True, want_argmax=True)
        for b in range(B):
            worst = max(worst, rel(f64(res["x"][b]), xs[s, b]))
            assert rel(f64(res["x"][b]), xs[s, b]) <= TOL, (s, b)
            assert rel(res["logits"][b], xs[s, b].astype(np.float64) @ E.T) <= TOL, (s, b)
        cur = [int(t) for t in res["argmax"]]
        assert cur == toks[s].tolist(), (s, cur, toks[s].tolist(), margin[s].tolist())
    # greedy path unambiguous: the smallest top-2 margin over the run is far above the error
    assert margin.min() > 10 * worst
    ba = O.BlockAssigner(tpb, O.HYBRID, O.HostAllocation(K, K), act_gpu=0)
    for rid in ids:
        ba.add_request(rid, P - 1)
        for _ in range(P - 1):
            ba.add_token(rid)
    for _ in range(G):
        for rid in ids:
            ba.add_token(rid)
    assert eng.cache.dump_json() == O.dumps(ba.cache.dump_json())
    eng.close()
