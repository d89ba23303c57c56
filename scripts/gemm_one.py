"""One recompute GEMM at OPT-30B (or argv[2]) width over n ACT tokens, for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_01792_b200 import api
n = int(sys.argv[1]) if len(sys.argv) > 1 else 43264
cfg = api.ModelConfig.preset(sys.argv[2] if len(sys.argv) > 2 else "opt-30b"); cfg.num_layers = 1
eng = api.Engine(cfg, seed=1, max_seq=64, max_batch=1, weights_on_device=False,
                 caps=api.PoolCaps(kv_host=16, act_host=(n + 15) // 16 + 8), mode="hybrid")
eng.admit_synthetic(["x"], [16], seed=3)
print(eng.time_kv_gen(n, reps=2) * 1e3, "ms")
