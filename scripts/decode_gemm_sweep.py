"""Weight-streaming decode GEMM sweep on the B200 (not a test): time every
(BN, splits) for the four decode GEMMs of a model shape at batch M and print
GB/s of weight traffic; the planner's pick is marked with '*'.

    python scripts/decode_gemm_sweep.py [opt-30b|opt-6.7b] [M]
"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2501_01792_b200 import api, kernels  # noqa: E402


def timed(fn, reps=5):
    fn()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    return min(t)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "opt-30b"
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    cfg = api.ModelConfig.preset(name)
    d, f = cfg.hidden_dim, cfg.ffn_dim
    # the engine path times GEMMs on device; here we use the engine's profile
    # split on a 1-layer resident engine per setting of HC_GEMM_SPLITS
    import subprocess
    child = r"""
import sys, os
sys.path.insert(0, ROOT)
from paper_2501_01792_b200 import api
name, M = sys.argv[1], int(sys.argv[2])
cfg = api.ModelConfig.preset(name); cfg.num_layers = 2
eng = api.Engine(cfg, seed=1, max_seq=64, max_batch=M, weights_on_device=True,
                 caps=api.PoolCaps(act_gpu=M * 2), mode="act_only")
ids = [f"r{i}" for i in range(M)]
eng.admit_synthetic(ids, [16] * M, seed=3)
best = 1e9
for s in range(4):
    eng.set_profile(True)
    eng.decode_step(ids, [1] * M, want_x=False)
    st = eng.last_stats()
    best = min(best, st["gemm_ms"] / cfg.num_layers)
w = (4 * cfg.hidden_dim ** 2 + 2 * cfg.hidden_dim * cfg.ffn_dim) * 2
print(f"{best * 1e3:.1f} us/layer  {w / (best / 1e3) / 1e9:.0f} GB/s")
"""
    for s in ("auto", "1", "2", "3", "4", "6", "8"):
        env = dict(os.environ)
        if s != "auto":
            env["HC_GEMM_SPLITS"] = s
        out = subprocess.run([sys.executable, "-c", f"ROOT={ROOT!r}\n" + child, name, str(M)], env=env,
                             capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        print(f"splits={s:>4s}: {line}", flush=True)


if __name__ == "__main__":
    main()
