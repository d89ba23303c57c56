"""Offloaded prefill at OPT-30B width on the B200 (not a test): B requests of
P tokens through `layers` layers, weights streamed from pinned host memory,
hybrid KV/ACT blocks stored to pinned host pools. Prints the profiled split
(GEMMs / causal attention / weight H2D / block D2H) as one JSON line; also the
command profiled by ncu for prefill_flash_kernel.

    python scripts/prefill_profile.py [--batch 16] [--prompt 1024] [--layers 2] [--ratio 0.3333]
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-30b")
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--prompt", type=int, default=1024)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--ratio", type=float, default=1.0 / 3.0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--arch", default="reference", choices=["reference", "opt"])
    ap.add_argument("--heads", type=int, default=0, help="override num_heads (e.g. 2x the preset: head_dim 64)")
    a = ap.parse_args()
    from paper_2501_01792_b200 import api
    cfg = api.ModelConfig.preset(a.model)
    if a.heads:
        cfg.num_heads = a.heads
    cfg.num_layers = a.layers
    B, P, tpb = a.batch, a.prompt, cfg.tokens_per_block
    nb = math.ceil((P + 1) / tpb)
    act = math.ceil(a.ratio * nb) + 1
    kv = math.ceil((1 - a.ratio) * nb) + 1
    k = int(round(a.ratio * 1000))
    eng = api.Engine(cfg, seed=42, max_seq=P + 2, rescale=True, max_batch=B, weights_on_device=False,
                     caps=api.PoolCaps(kv_host=B * kv, act_host=B * act), mode="hybrid",
                     allocation=api.HostAllocation(k, 1000 - k), arch=a.arch)
    rng = np.random.default_rng(0)
    prompts = [rng.integers(0, cfg.vocab_size, P).tolist() for _ in range(B)]
    d, f, L = cfg.hidden_dim, cfg.ffn_dim, cfg.num_layers
    for rep in range(a.reps):
        ids = [f"r{rep}_{i}" for i in range(B)]
        eng.set_profile(True)
        eng.prefill(ids, prompts)
        eng.set_profile(False)
        st = eng.last_stats()
        for i in ids:
            eng.free_request(i)
    gemm = L * 2.0 * B * P * (4 * d * d + 2 * d * f)
    attn = L * B * 2.0 * d * P * (P + 1)
    print(json.dumps({"model": a.model, "arch": a.arch, "batch": B, "prompt": P, "layers": L, "prefill_ms": st["step_ms"],
                      "gemm_ms": st["gemm_ms"], "attn_ms": st["attn_ms"], "weight_h2d_ms": st["copy_ms"],
                      "block_d2h_ms": st["store_ms"], "gemm_tflops": gemm / st["gemm_ms"] / 1e9,
                      "attn_tflops_causal": attn / st["attn_ms"] / 1e9,
                      "d2h_gbs": st["d2h_bytes"] / st["store_ms"] / 1e6 if st["store_ms"] else None,
                      "h2d_gb": st["h2d_bytes"] / 1e9, "d2h_gb": st["d2h_bytes"] / 1e9}))
    eng.close()


if __name__ == "__main__":
    main()
