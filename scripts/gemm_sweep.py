"""Recompute-GEMM tuning sweep on the B200 (not a test; prints one line per
setting). OPT-30B width, one layer, n ACT tokens from the ACT staging pool:
time_kv_gen = CUDA-event time of gemm_tn_kernel<256, kKvPaged>.

    python scripts/gemm_sweep.py [n_tokens]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r"""
import sys, json
sys.path.insert(0, ROOT)
from paper_2501_01792_b200 import api
n = int(sys.argv[1]); dm = int(sys.argv[2])
cfg = api.ModelConfig.preset("opt-30b" if dm == 7168 else "opt-6.7b"); cfg.num_layers = 1
blocks = (n + 15) // 16 + 8
eng = api.Engine(cfg, seed=1, max_seq=64, max_batch=1, weights_on_device=True,
                 caps=api.PoolCaps(kv_host=16, act_host=blocks), mode="hybrid")
eng.admit_synthetic(["x"], [16], seed=3)
t = min(eng.time_kv_gen(n, reps=10) for _ in range(3))
print(json.dumps({"n": n, "d": dm, "ms": t * 1e3, "tflops": 4.0 * dm * dm * n / t / 1e12}))
"""


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 43264
    for dm in (7168, 4096):
        for g in (8, 16, 32, 48, 64):
            env = dict(os.environ, HC_GEMM_GROUP_M=str(g))
            out = subprocess.run([sys.executable, "-c", f"ROOT={ROOT!r}\n" + CHILD, str(n), str(dm)], env=env,
                                 capture_output=True, text=True)
            line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
            print(f"group_m={g:3d} {line}", flush=True)


if __name__ == "__main__":
    main()
