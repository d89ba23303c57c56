"""The reference CLI's sweep CSV (tools/main.cpp:281-305: mode, batch,
prompt_len, throughput, pcie_busy, gpu_busy, traffic by class, error) from
B200 MEASUREMENTS instead of the simulator: OPT-30B shape, weights + cache in
pinned host memory, gen 32 (the sweep's default, sim.hpp:110), modes hybrid
(the planner's r from the committed bundle) / kv_only / act_only, batch 32 /
64 / 128, prompt 512 / 1024. Per row: the real offloaded prefill of B random
prompts, the requests grown to the generation's mean context in decode order,
3 timed decode steps (+1 profiled for the busy fractions);
throughput = B*G / (prefill + G * step), traffic = prefill + G * per-step
bytes by class. Writes gpurun_out/sweep.csv.

    python scripts/sweep_csv.py [--model opt-30b] [--gen 32]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (pool sizing helpers)
from paper_2501_01792_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-30b")
    ap.add_argument("--gen", type=int, default=32)
    ap.add_argument("--batches", default="32,64,128")
    ap.add_argument("--prompts", default="512,1024")
    a = ap.parse_args()
    cfg = api.ModelConfig.preset(a.model)
    G, L, tpb = a.gen, cfg.num_layers, cfg.tokens_per_block
    batches = [int(x) for x in a.batches.split(",")]
    prompts = [int(x) for x in a.prompts.split(",")]
    Bmax, Pmax = max(batches), max(prompts)
    b7 = bench.read_bundle(os.path.join(ROOT, "profiles", f"planner_bundle_{a.model}.json"))

    def plan_fn(b5, m4, tpb_, ag):
        tb = api.TimingBundle(api.LinearTimeModel(b5[0], b5[1]), api.LinearTimeModel(b5[2], b5[3]), b5[4])
        return list(api.plan_host_allocation(tb, api.MemoryBudget(*m4), tpb_, ag).__dict__.values())

    w_layer, _ = api.weight_bytes(cfg)
    budget = max(16e9, bench.mem_available_bytes() - 40e9)
    Lw = L if L * w_layer <= 0.55 * budget else max(2, int(0.55 * budget // w_layer))
    eng = api.Engine(cfg, seed=42, max_seq=Pmax + G + 2, rescale=True, max_batch=Bmax, weights_on_device=False,
                     caps=api.PoolCaps(kv_host=16, act_host=16), weight_layers=Lw, mode="hybrid")
    rows = []
    for mode in ("hybrid", "kv_only", "act_only"):
        for B in batches:
            for P in prompts:
                err = ""
                try:
                    r = {"kv_only": 0.0, "act_only": 1.0}.get(mode)
                    if r is None:
                        r = bench.planned_ratio(b7, cfg, B * (P + G), plan_fn)[0]
                    md, alloc, caps = bench.pool_plan(cfg, B, P + G + 1, 0, r)
                    Lp = bench.host_layers_for(cfg, caps, budget, Lw * w_layer)
                    eng.configure_cache(caps, mode=md, allocation=alloc, host_layers=Lp)
                    ids = [f"s{i}" for i in range(B)]
                    eng.fill_pools(seed=7)
                    eng.set_profile(True)
                    eng.prefill(ids, [list(range(1, P + 1))] * B)
                    pre = eng.last_stats()
                    eng.advance_synthetic(ids, G // 2 - 3)
                    toks = [3] * B
                    eng.set_profile(False)
                    for _ in range(2):
                        eng.decode_step(ids, toks, want_x=False)
                    t = []
                    for _ in range(3):
                        eng.decode_step(ids, toks, want_x=False)
                        t.append(eng.last_stats()["step_ms"])
                    eng.set_profile(True)
                    eng.decode_step(ids, toks, want_x=False)
                    st = eng.last_stats()
                    eng.set_profile(False)
                    step = sum(t) / len(t) / 1e3
                    pre_s = pre["step_ms"] / 1e3
                    make = pre_s + G * step
                    gbusy = ((pre["gemm_ms"] + pre["attn_ms"]) + G * step * 1e3 *
                             (st["recompute_ms"] + st["attn_ms"] + st["gemm_ms"]) / st["step_ms"]) / (make * 1e3)
                    pbusy = (pre["copy_ms"] + G * step * 1e3 * st["copy_ms"] / st["step_ms"]) / (make * 1e3)
                    traffic = [pre["h2d_weights"] + G * st["h2d_weights"], pre["h2d_kv"] + G * st["h2d_kv"],
                               pre["h2d_act"] + G * st["h2d_act"], pre["d2h_kv"] + G * st["d2h_kv"],
                               pre["d2h_act"] + G * st["d2h_act"]]
                    rows.append((mode, B, P, B * G / make, pbusy, gbusy, *[int(x) for x in traffic], ""))
                    print(rows[-1][:6], flush=True)
                except Exception as e:  # noqa: BLE001 — a row that cannot run is reported, as the CLI does
                    err = str(e).replace(",", ";").replace("\n", " ")
                    rows.append((mode, B, P, None, None, None, None, None, None, None, None, err))
                    print(mode, B, P, "error", err, flush=True)
    eng.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", "sweep.csv")
    with open(path, "w") as fh:
        fh.write(f"# b200-measured {time.strftime('%Y-%m-%d')} model={a.model} gen={G} (scripts/sweep_csv.py)\n")
        fh.write("mode,batch,prompt_len,throughput_tok_s,pcie_busy,gpu_busy,traffic_weights,traffic_kv_load,"
                 "traffic_act_load,traffic_kv_store,traffic_act_store,error\n")
        for rw in rows:
            cells = []
            for v in rw:
                cells.append("" if v is None else (f"{v:.9g}" if isinstance(v, float) else str(v)))
            fh.write(",".join(cells) + "\n")
    print(path)


if __name__ == "__main__":
    main()
