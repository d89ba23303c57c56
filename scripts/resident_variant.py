"""Time bench.resident_variants() alone (the HBM-resident config-3 workload:
weights + KV/ACT blocks in HBM, planned ratio r_fit) — GEMM tuning experiments.

    python scripts/resident_variant.py [--model opt-30b] [--batch 128]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-30b")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--prompt", type=int, default=1024)
    ap.add_argument("--only-planned", action="store_true")
    a = ap.parse_args()
    import bench
    from paper_2501_01792_b200 import api
    cfg = api.ModelConfig.preset(a.model)
    clk = bench.ClockSampler(0)
    clk.start()
    res = bench.resident_variants(0, cfg, a.batch, a.prompt, "reference", only_planned=a.only_planned)
    res["clocks"] = clk.stop()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
