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


@pytest.mark.parametrize("seed", range(10))
def test_equivalence_seeded_models(seed):
    """run_equivalence_case (verify.cpp:26-95) on the GPU: a seeded random model,
    its context held as stored KV, as ACT checkpoints (recomputed), and as a
    block-wise mix; the decode output is the same for all (within bf16
    tolerance) and equals the oracle."""
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
    eng = api.Engine(cfg, seed=wseed, max_seq=P + 2, max_batch=1)
    outs, stats = {}, {}
    for mode, alloc in (("kv_only", None), ("act_only", None), ("hybrid", api.HostAllocation(1, 1))):
        eng.configure_cache(api.PoolCaps(kv_host=8, act_host=8, act_gpu=2), mode=mode, allocation=alloc)
        eng.prefill(["q"], [ids])
        eng.set_profile(True)
        outs[mode] = f64(eng.decode_step(["q"], [tok])["x"])
        stats[mode] = (eng.last_stats(), eng.cache.dump_json())
    ocfg = O.ModelConfig(num_layers=L, hidden_dim=d, num_heads=H, ffn_dim=2 * d, vocab_size=64).validate()
    w = O.prepare_weights(O.generate_weights(ocfg, wseed, P + 2))
    ref = O.forward_prompt(ids + [tok], w).output[-1:]
    for m, o in outs.items():
        assert rel(o, ref) <= TOL, (m, stats[m], (L, H, d, tpb, P))
    assert rel(outs["act_only"], outs["kv_only"]) <= TOL
    assert rel(outs["hybrid"], outs["kv_only"]) <= TOL


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
