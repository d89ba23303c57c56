"""BASELINE configs[1] (OPT-6.7B shape, batch 64, prompt 512, ACT-only cache +
weights in HBM): warm-up steps, then ONE decode step between
cudaProfilerStart/Stop, for an ncu launch list of exactly one step
(graphs off so every kernel is its own launch):

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \\
        python scripts/config2_ncu.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2501_01792_b200 import api
    B, P = 64, 512
    cfg = api.ModelConfig.preset(sys.argv[1] if len(sys.argv) > 1 else "opt-6.7b")
    nb = -(-(P + 8) // cfg.tokens_per_block)
    eng = api.Engine(cfg, seed=42, max_seq=P + 9, max_batch=B, weights_on_device=True,
                     caps=api.PoolCaps(act_gpu=B * nb), mode="act_only")
    eng.set_graphs(False)
    ids = [f"c2r{i}" for i in range(B)]
    eng.admit_synthetic(ids, [P] * B, seed=5)
    toks = np.random.default_rng(2).integers(0, cfg.vocab_size, (4, B)).astype(np.int32)
    for s in range(3):
        eng.decode_step(ids, toks[s].tolist(), want_x=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    eng.decode_step(ids, toks[3].tolist(), want_x=False)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    st = eng.last_stats()
    print({k: st[k] for k in ("step_ms", "recompute_rows", "launches")})
    eng.close()


if __name__ == "__main__":
    main()
