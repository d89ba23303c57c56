"""The product's host logic (C++ behind the C ABI, no GPU needed) against the
reference's golden fixtures and the oracle: block tables and pbns bit-exact,
planner / fits bit-exact, weight generation bit-exact to the oracle's bf16."""
import json
import os

import numpy as np
import pytest

import hybridsim_oracle as O
from paper_2501_01792_b200 import CapacityError, ConfigError, InputError, api

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gjson():
    with open(os.path.join(GOLD, "golden.json")) as fh:
        return json.load(fh)


def replay(args):
    """The simulator's add_token order on the product's HybridCache."""
    a, k, g = args["act_host"], args["kv_host"], args["act_gpu"]
    mode = args["mode"]
    if mode == "kv_only":
        k += a // 2
        a, g = 0, 0
    elif mode == "act_only":
        a += 2 * k
        k = 0
    c = api.HybridCache(args["tpb"], api.PoolCaps(k, 0, a, g))
    alloc = api.HostAllocation(a, k)
    ids = [f"r{i}" for i in range(len(args["lens"]))]
    for rid, n in zip(ids, args["lens"]):
        c.create_request(rid, n)

    def add(rid):
        if c.context_len(rid) % args["tpb"] == 0:
            if mode == "hybrid":
                kind = api.next_block_kind(*c.blocks_by_kind(rid), alloc)
            else:
                kind = api.BlockKind.ACT if mode == "act_only" else api.BlockKind.KV
            c.append_block(rid, kind)
        c.fill_token(rid)

    for rid, n in zip(ids, args["lens"]):
        for _ in range(n):
            add(rid)
    for it in range(max(args["gens"])):
        for rid, gl in zip(ids, args["gens"]):
            if it < gl:
                add(rid)
    for rid in args.get("frees", []):
        c.free_request(rid)
    return c


def test_block_tables_bit_exact(gjson):
    for case in gjson["block_tables"]:
        c = replay(case["args"])
        assert c.dump_json() == O.dumps(case["dump"])
        # the same document parsed, entry by entry
        for req in case["dump"]["requests"]:
            t = c.table(req["id"])
            assert [(str(e.kind), str(e.location), e.pbn, e.filled_tokens) for e in t.entries] == \
                   [(e["kind"], e["location"], e["pbn"], e["filled"]) for e in req["entries"]]


def test_next_block_kind(gjson):
    for a, k, ah, kh, want in gjson["next_block_kind"]:
        assert str(api.next_block_kind(a, k, api.HostAllocation(ah, kh))) == want
    with pytest.raises(InputError):
        api.next_block_kind(0, 0, api.HostAllocation())
    with pytest.raises(InputError):
        api.next_block_kind(-1, 0, api.HostAllocation(1, 1))


def test_planner_bit_exact(gjson):
    for c in gjson["plan"]:
        b = api.TimingBundle(api.LinearTimeModel(c["bundle"][0], c["bundle"][1]),
                             api.LinearTimeModel(c["bundle"][2], c["bundle"][3]), c["bundle"][4])
        mem = api.MemoryBudget(*c["mem"])
        assert list(api.initial_cache_allocation(b, c["tpb"], c["act_gpu"])) == c["init"]
        if c["err"] is not None:
            with pytest.raises(CapacityError):
                api.plan_host_allocation(b, mem, c["tpb"], c["act_gpu"])
            continue
        a = api.plan_host_allocation(b, mem, c["tpb"], c["act_gpu"])
        assert [a.act_host, a.kv_host, a.act_init, a.kv_init, a.act_remain, a.kv_remain] == c["alloc"]


def test_planner_worked_examples():
    B = lambda ks, ki, ls, li, w: api.TimingBundle(api.LinearTimeModel(ks, ki), api.LinearTimeModel(ls, li), w)
    assert api.initial_cache_allocation(B(1e-5, 0, 4e-6, 0, 0.01), 16, 0) == (62, 0)
    assert api.initial_cache_allocation(B(1e-5, 0, 4e-6, 0, 0.01008), 16, 88) == (0, 62)
    assert api.alloc_remaining(B(2e-5, 0, 1e-5, 0, 0), api.MemoryBudget(500, 0, 2, 1), 16, 0, 0) == (100, 200)
    with pytest.raises(CapacityError):
        api.alloc_remaining(B(1e-5, 0, 1e-5, 0, 0), api.MemoryBudget(100, 90, 2, 1), 16, 20, 0)
    a = api.plan_host_allocation(B(1e-5, 0, 4e-6, 0, 0.01), api.MemoryBudget(1e6, 0, 4, 2), 16, 0)
    assert (a.act_init, a.kv_init) == (62, 0) and 2 * a.act_host + 4 * a.kv_host <= 1e6


def test_fit_linear_and_bundle(gjson):
    for c in gjson["fit_linear"]:
        m = api.fit_linear(list(zip(c["x"], c["y"])))
        assert [m.slope, m.intercept, m.r_squared, float(m.intercept_clamped)] == c["fit"]
    with pytest.raises(InputError):
        api.fit_linear([(1.0, 1.0)])
    cfg = api.ModelConfig.preset("opt-30b")
    b = api.bundle_from_samples([(64, 1e-4), (128, 2e-4)], [(64, 3e-5), (128, 6e-5)], 55e9, cfg)
    per, total = api.weight_bytes(cfg)
    assert b.s_weight_layer == per and b.t_load_w == per / 55e9
    assert abs(b.t_kv_gen.slope - 1e-4 / 64) < 1e-18


def test_flops_and_bytes(gjson):
    for kind, d, f, n, k, L, want in gjson["flops"]:
        cfg = api.ModelConfig(num_layers=L, hidden_dim=d, ffn_dim=f)
        assert api.flop_count(kind, cfg, n, k) == want
    for d, tpb, kv, act in gjson["bytes_of"]:
        cfg = api.ModelConfig(hidden_dim=d, tokens_per_block=tpb)
        assert (api.HybridCache.bytes_of("KV", cfg), api.HybridCache.bytes_of("ACT", cfg)) == (kv, act)


def test_cache_reference_unit_cases():
    """test_cache.cpp:35-141 on the product's cache."""
    c = api.HybridCache(16, api.PoolCaps(10, 0, 10, 2))
    c.create_request("r", 0)
    locs = []
    for kind in ("ACT", "ACT", "ACT", "KV"):
        e = c.append_block("r", kind)
        for _ in range(16):
            c.fill_token("r")
        locs.append(str(e.location))
    assert locs == ["gpu", "gpu", "host", "host"]
    with pytest.raises(InputError):
        c.create_request("r", 1)
    t = api.HybridCache(16, api.PoolCaps(1, 0, 0, 0))
    t.create_request("x", 0)
    with pytest.raises(InputError):
        t.fill_token("x")
    t.append_block("x", "KV")
    with pytest.raises(InputError):
        t.append_block("x", "KV")            # last block not full
    for _ in range(16):
        t.fill_token("x")
    with pytest.raises(InputError):
        t.fill_token("x")
    with pytest.raises(CapacityError):
        t.append_block("x", "KV")
    assert len(t.table("x").entries) == 1
    kv = api.HybridCache(16, api.PoolCaps(4, 1, 0, 0), kv_on_gpu=True)
    kv.create_request("k", 0)
    assert str(kv.append_block("k", "KV").location) == "gpu"
    f = api.HybridCache(16, api.PoolCaps(8, 0, 8, 4))
    f.create_request("r", 0)
    for kind in ["KV"] * 5 + ["ACT"] * 6:
        f.append_block("r", kind)
        for _ in range(16):
            f.fill_token("r")
    assert f.free_blocks("KV", "host") == 3
    f.free_request("r")
    assert (f.free_blocks("KV", "host"), f.free_blocks("ACT", "gpu"), f.free_blocks("ACT", "host")) == (8, 4, 8)
    with pytest.raises(InputError):
        f.free_request("r")
    with pytest.raises(InputError):
        api.HybridCache(0)


def test_cache_fuzz_against_oracle():
    """test_cache.cpp:143-201 style fuzz: every op on the product cache and the
    oracle cache gives identical results and identical tables."""
    rng = O.SplitMix64(2024)
    prod = api.HybridCache(8, api.PoolCaps(30, 0, 30, 10))
    orac = O.HybridCache(8, kv_host=30, act_host=30, act_gpu=10)
    live, nxt = [], 0
    for step in range(1500):
        op = rng.uniform_int(0, 3)
        res = []
        for c in (prod, orac):
            try:
                if op == 0:
                    c.create_request(f"q{nxt}", 0)
                    res.append("ok")
                elif live:
                    rid = live[rng.uniform_int(0, len(live) - 1) if c is prod else pick]
                    if op == 1:
                        kind = "ACT" if (kbit if c is orac else rng.uniform01() < 0.5) else "KV"
                        if c is prod:
                            kbit = kind == "ACT"
                        e = c.append_block(rid, kind)
                        res.append((str(e.location), e.pbn))
                    elif op == 2:
                        c.fill_token(rid)
                        res.append("ok")
                    else:
                        c.free_request(rid)
                        res.append("ok")
                else:
                    res.append("skip")
                if c is prod and live and op != 0:
                    pick = live.index(rid)
            except (CapacityError, InputError, O.CapacityError, O.InputError) as e:
                res.append(type(e).__name__)
                if c is prod and live and op != 0:
                    pick = live.index(rid)
        assert res[0] == res[1], (step, res)
        if op == 0:
            live.append(f"q{nxt}")
            nxt += 1
        elif live and op == 3 and res[0] == "ok":
            live.remove(rid)
    assert prod.dump_json() == O.dumps(orac.dump_json())


def test_generate_weights_bit_exact_to_oracle():
    """C++ generate + rescale + bf16 (device layout) == oracle's bf16 bits."""
    cfg = api.ModelConfig(num_layers=2, hidden_dim=64, num_heads=2, ffn_dim=128, vocab_size=96)
    w = api.generate_weights(cfg, 42, 24, rescale=True)
    ocfg = O.ModelConfig(num_layers=2, hidden_dim=64, num_heads=2, ffn_dim=128, vocab_size=96).validate()
    ow = O.prepare_weights(O.generate_weights(ocfg, 42, 24))
    assert np.array_equal(w["embedding"], O.to_f16_bits(ow.embedding))
    assert np.array_equal(w["positional"], O.to_f16_bits(ow.positional))
    for l in range(2):
        lay = api.unpack_layer(cfg.validate(), w["layers"][l])
        for n in O.WEIGHT_NAMES:
            assert np.array_equal(lay[n], O.to_f16_bits(ow.layers[l][n])), n


def test_model_config_validation():
    with pytest.raises(InputError):
        api.ModelConfig(hidden_dim=30, num_heads=4).validate()
    with pytest.raises(InputError):
        api.ModelConfig.preset("opt-1t")
    c = api.ModelConfig(hidden_dim=64).validate()
    assert c.ffn_dim == 256
    assert api.ModelConfig.preset("opt-66b").num_layers == 64


def _hbm_plan_restated(cfg, B, nb, hbm):
    """Python restatement of plan_hbm_residency (csrc/host/plan.hpp)."""
    import math
    from paper_2501_01792_b200 import api
    L = cfg.num_layers
    kv_one = api.HybridCache.bytes_of("KV", cfg)
    kv_all, act_all = kv_one * L, api.HybridCache.bytes_of("ACT", cfg) * L
    N = B * nb
    x_exact = (N * kv_all - hbm) / (kv_all - act_all - kv_one)
    x_fit = 0 if x_exact <= 0 else math.ceil(x_exact)
    r = 0.0 if x_fit == 0 else min(1.0, (x_fit + B) / N)
    act_need = 0 if r <= 0 else (N if r >= 1 else B * (math.ceil(r * nb) + 1))
    kv_need = 0 if r >= 1 else (N if r <= 0 else B * (math.ceil((1 - r) * nb) + 1))
    act_gpu = int(min(act_need, math.floor(hbm / (act_all + kv_one))))
    room = hbm - act_gpu * (act_all + kv_one) - 2.0 * kv_need * kv_one
    kv_gpu = int(max(0, min(kv_need, math.floor(room / (kv_all - 2 * kv_one)))))
    return r, (act_gpu, kv_gpu, act_need - act_gpu, kv_need - kv_gpu)


@pytest.mark.parametrize("model,B,nb,hbm_gb", [("opt-30b", 128, 65, 124.6), ("opt-13b", 64, 129, 150.0),
                                               ("opt-66b", 128, 65, 40.0), ("opt-6.7b", 8, 10, 500.0),
                                               ("opt-30b", 128, 65, 20.0)])
def test_plan_hbm_residency(model, B, nb, hbm_gb):
    """HBM-residency planner (B200 extension of Alg. 1): smallest ACT share
    whose blocks fit; 0 when all-KV fits; capacities cover the workload."""
    from paper_2501_01792_b200 import api
    cfg = api.ModelConfig.preset(model)
    r, caps = api.plan_hbm_residency(cfg, B, nb, hbm_gb * 1e9)
    r2, c2 = _hbm_plan_restated(cfg, B, nb, hbm_gb * 1e9)
    assert r == pytest.approx(r2, abs=1e-15)
    assert (caps.act_gpu, caps.kv_gpu, caps.act_host, caps.kv_host) == c2
    assert 0.0 <= r <= 1.0
    kv_one = api.HybridCache.bytes_of("KV", cfg)
    used = (caps.act_gpu * (api.HybridCache.bytes_of("ACT", cfg) * cfg.num_layers + kv_one) +
            caps.kv_gpu * kv_one * cfg.num_layers + 2 * caps.kv_host * kv_one)
    assert used <= hbm_gb * 1e9 * 1.0000001
    if hbm_gb >= 500:
        assert r == 0.0 and caps.kv_host == 0
    with pytest.raises(api.InputError):
        api.plan_hbm_residency(cfg, 0, nb, 1e9)


def _hbm_tiers_restated(cfg, B, nb, hbm, slope_gen, slope_load, host=0.0, t_w=0.0):
    """Python restatement of plan_hbm_tiers (csrc/host/plan.hpp), zero intercepts."""
    import math
    from paper_2501_01792_b200 import api
    L, tpb = cfg.num_layers, cfg.tokens_per_block
    kv_one, act_one = api.HybridCache.bytes_of("KV", cfg), api.HybridCache.bytes_of("ACT", cfg)
    kv_all, act_all = kv_one * L, act_one * L
    N = B * nb
    best = None
    for x in range(N + 1):
        rhs = hbm - x * (act_all + kv_one) - B * kv_one - 2.0 * (N - x + B) * kv_one - 2.0 * B * act_one
        if rhs < 0:
            break
        y = min(N - x, math.floor(rhs / (kv_all - 2 * kv_one)))
        z = N - x - max(y, 0)
        slack = B if 0 < x < N else 0
        if host > 0 and (z + slack) * kv_all + slack * act_all > host:
            continue
        t = max(slope_gen * x * tpb, t_w + slope_load * z * tpb)
        if best is None or t < best[0]:
            best = (t, x, max(y, 0), z)
    if best is None:
        return None
    t, x, y, z = best
    return x / N, (x, y, (B if 0 < x < N else 0), z + (B if 0 < x < N else 0))


@pytest.mark.parametrize("model,B,nb,hbm_gb,gen,load", [("opt-30b", 128, 65, 127.6, 1.3e-7, 5.2e-7),
                                                          ("opt-30b", 64, 65, 40.0, 1.3e-7, 5.2e-7),
                                                          ("opt-13b", 64, 129, 150.0, 8e-8, 3.7e-7),
                                                          ("opt-30b", 128, 65, 127.6, 1e-5, 5.2e-7)])
def test_plan_hbm_tiers(model, B, nb, hbm_gb, gen, load):
    """Balanced three-tier plan: matches the restatement; balances the two
    channels when both are in use; all-KV in HBM when it fits; falls back to
    capacity-bound KV streaming when recompute is expensive."""
    from paper_2501_01792_b200 import api
    cfg = api.ModelConfig.preset(model)
    kv = [(1024.0, 1024 * gen), (4096.0, 4096 * gen)]
    ld = [(1024.0, 1024 * load), (4096.0, 4096 * load)]
    bundle = api.bundle_from_samples(kv, ld, 55e9, cfg)
    r, caps, (tc, tl) = api.plan_hbm_tiers(cfg, B, nb, hbm_gb * 1e9, bundle)
    r2, c2 = _hbm_tiers_restated(cfg, B, nb, hbm_gb * 1e9, bundle.t_kv_gen.slope, bundle.t_load_kv.slope)
    assert r == pytest.approx(r2) and (caps.act_gpu, caps.kv_gpu, caps.act_host, caps.kv_host) == c2
    if model == "opt-13b":
        assert caps.act_gpu == 0 and caps.kv_host == 0          # all KV fits in HBM
    elif gen < 1e-6:
        assert caps.act_gpu > 0 and caps.kv_host > B            # both channels busy ...
        assert abs(tc - tl) <= max(tc, tl) * 0.02               # ... and balanced


@pytest.mark.parametrize("hbm_gb", [170.0, 120.0, 60.0])
def test_plan_hbm_tiers_streamed_weights(hbm_gb):
    """Weights left in pinned host memory (streamed every layer): the link side
    carries t_load_w too, so recompute is free up to the weight stream's time
    and the plan matches the restatement with that term."""
    from paper_2501_01792_b200 import api
    cfg = api.ModelConfig.preset("opt-30b")
    B, nb = 128, 73
    kv = [(1024.0, 1024 * 1.2e-7), (4096.0, 4096 * 1.2e-7)]
    ld = [(1024.0, 1024 * 5.2e-7), (4096.0, 4096 * 5.2e-7)]
    bundle = api.bundle_from_samples(kv, ld, 55e9, cfg)
    r, caps, (tc, tl) = api.plan_hbm_tiers(cfg, B, nb, hbm_gb * 1e9, bundle, weights_streamed=True)
    r2, c2 = _hbm_tiers_restated(cfg, B, nb, hbm_gb * 1e9, bundle.t_kv_gen.slope, bundle.t_load_kv.slope,
                                 t_w=bundle.t_load_w)
    assert r == pytest.approx(r2) and (caps.act_gpu, caps.kv_gpu, caps.act_host, caps.kv_host) == c2
    assert tl >= bundle.t_load_w
    r0, _, _ = api.plan_hbm_tiers(cfg, B, nb, hbm_gb * 1e9, bundle)
    assert r >= r0 - 1e-12  # a busier link shifts blocks to recompute: never less ACT



@pytest.mark.parametrize("host_gb", [224.0, 120.0, 60.0, 5.0])
def test_plan_hbm_tiers_host_budget(host_gb):
    """A pinned-host budget moves blocks from the KV host tier to recompute
    (ACT in HBM), matching the restatement; an impossible budget is a
    CapacityError."""
    from paper_2501_01792_b200 import api
    cfg = api.ModelConfig.preset("opt-66b")
    B, nb = 64, 132
    kv = [(1024.0, 1024 * 2.5e-7), (4096.0, 4096 * 2.5e-7)]
    ld = [(1024.0, 1024 * 1.2e-6), (4096.0, 4096 * 1.2e-6)]
    bundle = api.bundle_from_samples(kv, ld, 55e9, cfg)
    want = _hbm_tiers_restated(cfg, B, nb, 56e9, bundle.t_kv_gen.slope, bundle.t_load_kv.slope, host_gb * 1e9)
    if want is None:
        from paper_2501_01792_b200.errors import CapacityError
        with pytest.raises(CapacityError):
            api.plan_hbm_tiers(cfg, B, nb, 56e9, bundle, host_bytes=host_gb * 1e9)
        return
    r, caps, _ = api.plan_hbm_tiers(cfg, B, nb, 56e9, bundle, host_bytes=host_gb * 1e9)
    r2, c2 = want
    assert r == pytest.approx(r2) and (caps.act_gpu, caps.kv_gpu, caps.act_host, caps.kv_host) == c2
    kv_all = api.HybridCache.bytes_of("KV", cfg) * cfg.num_layers
    act_all = api.HybridCache.bytes_of("ACT", cfg) * cfg.num_layers
    assert caps.kv_host * kv_all + caps.act_host * act_all <= host_gb * 1e9
    r_free, _, _ = api.plan_hbm_tiers(cfg, B, nb, 56e9, bundle)
    assert r >= r_free


def _host_min_step_restated(cfg, B, nb, b, host=0.0):
    """Python restatement of plan_host_min_step (csrc/host/plan.hpp)."""
    from paper_2501_01792_b200 import api
    L, tpb = cfg.num_layers, cfg.tokens_per_block
    kv_one, act_one = api.HybridCache.bytes_of("KV", cfg), api.HybridCache.bytes_of("ACT", cfg)
    N = B * nb
    ev = lambda m, n: m.intercept + m.slope * n  # noqa: E731  (eval, timing.cpp:75-77)
    best = None
    for x in range(N + 1):
        slack = B if 0 < x < N else 0
        if host > 0 and ((N - x + slack) * kv_one + (x + slack) * act_one) * L > host:
            continue
        tc = ev(b.t_kv_gen, x * tpb) if x > 0 else 0.0
        tl = b.t_load_w + ev(b.t_load_kv, ((N - x) + x * act_one / kv_one) * tpb)
        if best is None or max(tc, tl) < best[0]:
            best = (max(tc, tl), x, slack, tc, tl)
    _, x, slack, tc, tl = best
    return x / N, x + slack, N - x + slack, tc, tl


@pytest.mark.parametrize("gen,host_gb", [(None, 0.0), (None, 140.0), (2.5e-6, 0.0), (1e-4, 0.0)])
def test_plan_host_min_step(gen, host_gb):
    """Host-only min-step planner (B200 extension): equals its restatement; on the
    committed B200 bundle at config 3 (OPT-30B, B 128, context 1152) the link
    dominates even at r = 1, so it picks pure ACT (the measured per-ratio sweep's
    fastest, 43.8 vs Alg. 1's 42.5 tok/s); with costly recompute it balances the
    two channels; with prohibitive recompute it keeps nearly all KV; a host budget that
    cannot hold all-KV pushes it towards ACT."""
    import json
    import os
    from paper_2501_01792_b200 import api
    bj = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "profiles",
                                     "planner_bundle_opt-30b.json")))
    cfg = api.ModelConfig.preset("opt-30b")
    b = api.TimingBundle(api.LinearTimeModel(gen if gen else bj["kv_gen"]["slope"], bj["kv_gen"]["intercept"]),
                         api.LinearTimeModel(bj["load_kv"]["slope"], bj["load_kv"]["intercept"]), bj["t_load_w"])
    B, nb = 128, 72  # 1152 tokens of context per request
    r, caps, (tc, tl) = api.plan_host_min_step(cfg, B, nb, b, host_gb * 1e9)
    r2, ah, kh, tc2, tl2 = _host_min_step_restated(cfg, B, nb, b, host_gb * 1e9)
    assert r == pytest.approx(r2) and (caps.act_host, caps.kv_host) == (ah, kh)
    assert (tc, tl) == pytest.approx((tc2, tl2))
    if gen is None and host_gb == 0:
        assert r == 1.0 and tc < tl
    elif gen == 2.5e-6:
        assert 0 < r < 1 and abs(tc - tl) <= max(tc, tl) * 0.01
    elif gen == 1e-4:  # recompute 190x dearer than streaming: only a sliver of ACT pays
        assert 0 < r < 0.01 and abs(tc - tl) <= 16 * gen * 1.01
    else:  # 140 GB cannot hold all-KV (194 GB): the budget binds
        kv_all = api.HybridCache.bytes_of("KV", cfg) * cfg.num_layers
        act_all = api.HybridCache.bytes_of("ACT", cfg) * cfg.num_layers
        assert caps.kv_host * kv_all + caps.act_host * act_all <= 140e9
    with pytest.raises(api.InputError):
        api.plan_host_min_step(cfg, 0, nb, b)
