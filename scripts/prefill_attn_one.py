"""One prefill attention call (tcgen05 two-tile kernel) at n_req x P tokens, H heads of head_dim hd, for ncu."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_01792_b200 import kernels  # noqa: E402

n_req, P, H, hd = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (8, 1024, 56, 128)))
rng = np.random.default_rng(0)
qkv = kernels.f32_to_f16_bits(rng.uniform(-1, 1, (n_req * P, 3 * H * hd)).astype(np.float32))
for _ in range(2):
    kernels.prefill_attention(qkv, n_req, P, H)
print("ok")
