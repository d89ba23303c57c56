"""Artifact compatibility: the bundle.json /
plan.json that bench.py --artifacts writes from B200 measurements load with
the UNMODIFIED reference's own parsers (TimingBundle::from_json,
HostAllocation::from_json), and the reference planner on that bundle
reproduces our planner's allocation bit-exactly."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import ref_lib as R

ART = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r01_artifacts")

pytestmark = pytest.mark.skipif(not R.available() or not os.path.exists(os.path.join(ART, "bundle.json")),
                                reason="needs oracle/_ref and committed artifacts")


def parse(bundle_txt, plan_txt):
    L = R.lib()
    L.ref_parse_artifacts.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_long)]
    out7 = (C.c_double * 7)()
    a6 = (C.c_long * 6)()
    rc = L.ref_parse_artifacts(bundle_txt.encode() if bundle_txt else None, plan_txt.encode() if plan_txt else None,
                               out7, a6)
    assert rc == 0, L.ref_last_error()
    return list(out7), list(a6)


def test_reference_loads_b200_bundle_and_plan():
    bundle_txt = open(os.path.join(ART, "bundle.json")).read()
    plan_txt = open(os.path.join(ART, "plan.json")).read()
    b, a = parse(bundle_txt, plan_txt)
    bj, pj = json.loads(bundle_txt), json.loads(plan_txt)
    assert b[0] == bj["kv_gen"]["slope"] and b[2] == bj["load_kv"]["slope"] and b[4] == bj["t_load_w"]
    assert a == [pj[k] for k in ("act_host", "kv_host", "act_init", "kv_init", "act_remain", "kv_remain")]


def test_reference_planner_agrees_on_b200_bundle():
    """Feed the measured bundle to the reference's plan_host_allocation and to
    ours: identical HostAllocation (both over the same memory budget)."""
    from paper_2501_01792_b200 import api
    bj = json.loads(open(os.path.join(ART, "bundle.json")).read())
    cfg = api.ModelConfig.preset("opt-30b")
    bundle = api.TimingBundle(api.LinearTimeModel(bj["kv_gen"]["slope"], bj["kv_gen"]["intercept"]),
                              api.LinearTimeModel(bj["load_kv"]["slope"], bj["load_kv"]["intercept"]),
                              bj["t_load_w"], bj["s_weight_layer"], bj["s_weight_total"])
    for host_gb in (200, 500, 882):
        mem = api.budget_for(host_gb * 1e9, cfg, bundle)
        ours = api.plan_host_allocation(bundle, mem, 16, 0)
        ref = R.plan_host_allocation([bundle.t_kv_gen.slope, bundle.t_kv_gen.intercept, bundle.t_load_kv.slope,
                                      bundle.t_load_kv.intercept, bundle.t_load_w],
                                     [mem.m_host, mem.s_weight, mem.s_kv_block, mem.s_act_block], 16, 0)
        assert [ours.act_host, ours.kv_host, ours.act_init, ours.kv_init, ours.act_remain, ours.kv_remain] == ref


def test_trace_schema():
    """trace.json carries the reference's SimEvent fields (sim.hpp:50-58)."""
    tr = json.loads(open(os.path.join(ART, "trace.json")).read())
    ev = tr["events"]
    assert ev and all(set(e) == {"name", "track", "start_us", "end_us", "iteration", "layer", "minibatch"} for e in ev)
    assert {e["track"] for e in ev} <= {"PCIe", "GPU", "PCIeUp"}
    assert all(e["end_us"] >= e["start_us"] for e in ev)
    layers = {e["layer"] for e in ev}
    assert len(layers) > 1


def test_reference_simulator_as_predictor():
    """The reference's simulate() (sim.cpp:134-633) runs on a B200-measured
    bundle (scripts/sim_vs_measured.py does it at config-3 scale and commits
    profiles/r01_sim_vs_measured.json); at toy scale its ordering matches the
    B200 measurements: ACT-only < hybrid < KV-only step time on a fast GPU."""
    import math
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    import sim_vs_measured as S
    cfg = {"num_layers": 2, "hidden_dim": 256, "num_heads": 2, "ffn_dim": 1024, "vocab_size": 512}
    bundle5 = [1.2e-10, 0.0, 5.2e-9, 0.0, 1.0e-4]   # recompute cheap, link slow (B200-like balance)
    B, P, G = 8, 64, 16
    nb = math.ceil((P + G) / 16)
    steps = {}
    for mode, r in (("kv_only", 0.0), ("hybrid", 0.5), ("act_only", 1.0)):
        a = 0 if mode == "kv_only" else B * (math.ceil(r * nb) + 1)
        k = 0 if mode == "act_only" else B * (math.ceil((1 - r) * nb) + 1)
        steps[mode] = S.simulate(cfg, bundle5, a, k, mode, B, P, G)["gen_s"]
    assert steps["act_only"] < steps["hybrid"] < steps["kv_only"]
    j = json.load(open(os.path.join(os.path.dirname(ART), "r01_sim_vs_measured.json")))
    planned = [r for r in j["rows"] if r["mode"] == "hybrid" and r["act_share_r"] > 0.9][0]
    gen = j["generation_e2e_measured"]
    measured_mean = (gen["step_ms_at_prompt"] + gen["step_ms_at_prompt_plus_gen"]) / 2
    assert abs(planned["sim_mean_step_ms"] / measured_mean - 1) < 0.05
