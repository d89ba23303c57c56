import sys, os
sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import numpy as np
import hybridsim_oracle as O
from paper_2501_01792_b200 import api
seed = 8
rng = O.SplitMix64(O.mix_seed(seed, 0x657175))
L = rng.uniform_int(1, 4); H = [1, 2, 4][rng.uniform_int(0, 2)]; d = 128 * H if rng.uniform_int(0, 1) else 64 * H
tpb = [8, 16][rng.uniform_int(0, 1)]; P = rng.uniform_int(3, 60)
cfg = api.ModelConfig(num_layers=L, hidden_dim=d, num_heads=H, ffn_dim=2 * d, vocab_size=64, tokens_per_block=tpb)
wseed = O.mix_seed(seed, 0x77)
ids = [rng.uniform_int(0, 63) for _ in range(P)]
tok = rng.uniform_int(0, 63)
order = sys.argv[1].split(",") if len(sys.argv) > 1 else ["kv_only", "act_only", "hybrid"]
eng = api.Engine(cfg, seed=wseed, max_seq=P + 2, max_batch=1)
for mode in order:
    eng.configure_cache(api.PoolCaps(kv_host=8, act_host=8, act_gpu=2), mode=mode, allocation=api.HostAllocation(1, 1))
    eng.prefill(["q"], [ids])
    eng.set_profile(True)
    x = O.f16_bits_to_f64(eng.decode_step(["q"], [tok])["x"])
    print(mode, np.abs(x).max(), {k: round(v, 3) for k, v in eng.last_stats().items()})
