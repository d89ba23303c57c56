"""Predicted (the reference's own discrete-event simulator, sim.cpp:134-633,
driven by the B200-MEASURED timing bundle) vs achieved (bench.py on a B200)
decode throughput per KV:ACT ratio — SURVEY.md §8(a) A15: "sim becomes the
predictor to compare achieved vs modelled". Runs on CPU (oracle/_ref).

    python scripts/sim_vs_measured.py [profiles/r01_bench_opt30b_full.json]
"""
import ctypes as C
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import ref_lib as R  # noqa: E402  (test / analysis infrastructure)

MODES = {"hybrid": 0, "kv_only": 1, "act_only": 2, "token_recompute": 3}


def simulate(cfg, bundle5, act_host, kv_host, mode, B, P, G, rc=0.0):
    L = R.lib()
    L.ref_simulate.argtypes = [C.c_int] * 6 + [C.POINTER(C.c_double), C.c_long, C.c_long, C.c_long, C.c_int,
                                               C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                               C.POINTER(C.c_double)]
    b = (C.c_double * 5)(*bundle5)
    out = (C.c_double * 6)()
    rc_ = L.ref_simulate(cfg["num_layers"], cfg["hidden_dim"], cfg["num_heads"], cfg["ffn_dim"], cfg["vocab_size"],
                         16, b, act_host, kv_host, 0, MODES[mode], rc, B, P, G, 1, out)
    if rc_:
        raise RuntimeError(L.ref_last_error().decode())
    return dict(zip(("throughput", "makespan_s", "prefill_s", "gen_s", "pcie_busy", "gpu_busy"), list(out)))


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01_bench_opt30b_full.json")
    j = json.load(open(path))
    pl = j["planner"]
    bundle5 = [pl["t_kv_gen"]["slope_s_per_token"], pl["t_kv_gen"]["intercept_s"],
               pl["t_load_kv"]["slope_s_per_token"], pl["t_load_kv"]["intercept_s"], pl["t_load_w_s"]]
    cfg = {"num_layers": 48, "hidden_dim": 7168, "num_heads": 56, "ffn_dim": 28672, "vocab_size": 50272}
    B, P, G = j["config"]["batch_per_gpu"], j["config"]["seq_len"], j["config"]["gen_len"]
    nb = math.ceil((P + G) / 16)
    rows = []
    for m in j["per_ratio"]:
        if "error" in m:
            continue
        r = m["act_share_r"]
        mode = m["mode"]
        if mode == "token_recompute":
            pred = simulate(cfg, bundle5, 0, B * nb + B, mode, B, P, G, m.get("recompute_ratio", 0.5))
        else:
            a = 0 if mode == "kv_only" else B * (math.ceil(r * nb) + 1)
            k = 0 if mode == "act_only" else B * (math.ceil((1 - r) * nb) + 1)
            pred = simulate(cfg, bundle5, a, k, mode, B, P, G)
        step_pred = pred["gen_s"] / G  # mean decode iteration over the generation
        rows.append({"mode": mode, "act_share_r": r, "measured_tokens_per_s_at_P": m["tokens_per_s"],
                     "measured_step_ms_at_P": m["ms_per_step"], "sim_mean_step_ms": step_pred * 1e3,
                     "sim_decode_tokens_per_s": B / step_pred, "sim_pcie_busy": pred["pcie_busy"],
                     "sim_gpu_busy": pred["gpu_busy"], "sim_prefill_s": pred["prefill_s"]})
    gen = j.get("generation_e2e") or {}
    out = {"source": os.path.relpath(path, ROOT), "bundle5": bundle5,
           "note": "sim = the reference's simulate() with the B200-measured bundle (full-duplex stores, one "
                   "mini-batch); its mean step covers contexts P..P+G, the measured step is at context ~P "
                   "(the generation_e2e endpoints bracket the mean)",
           "generation_e2e_measured": gen, "rows": rows}
    dst = os.path.join(ROOT, "profiles", "r01_sim_vs_measured.json")
    json.dump(out, open(dst, "w"), indent=1)
    for rrow in rows:
        print(f"{rrow['mode']:16s} r={rrow['act_share_r']:.3f} measured@P {rrow['measured_step_ms_at_P']:8.1f} ms  "
              f"sim mean {rrow['sim_mean_step_ms']:8.1f} ms  (pcie {rrow['sim_pcie_busy']:.2f}, gpu {rrow['sim_gpu_busy']:.2f})")


if __name__ == "__main__":
    main()
