import sys, numpy as np
sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import hybridsim_oracle as O
from paper_2501_01792_b200 import api
g = np.load("tests/golden/golden.npz")
cfg = api.ModelConfig(num_layers=12, hidden_dim=768, num_heads=12, ffn_dim=3072, vocab_size=50272)
eng = api.Engine(cfg, seed=42, max_seq=160, rescale=True, max_batch=1)
tr = eng.forward_trace(g["opt125m_shape/ids"].tolist())
f = O.f16_bits_to_f64
for l in range(12):
    a = f(tr["layer_inputs"][l]); b = g["opt125m_shape/layer_inputs"][l]
    k = f(tr["k"][l]); kb = g["opt125m_shape/k"][l]
    print(l, "X maxrel %.4f rms %.4f | K maxrel %.4f rms %.4f" % (np.abs(a-b).max()/np.abs(b).max(), np.linalg.norm(a-b)/np.linalg.norm(b), np.abs(k-kb).max()/np.abs(kb).max(), np.linalg.norm(k-kb)/np.linalg.norm(kb)))
o = f(tr["output"]); ob = g["opt125m_shape/output"]
print("out", np.abs(o-ob).max()/np.abs(ob).max(), np.linalg.norm(o-ob)/np.linalg.norm(ob))
