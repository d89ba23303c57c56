"""Numpy emulation of the OPT layer variant with bf16 rounding where the engine rounds
(LN outputs, QKV, attention, residual adds, FFN hidden) vs the fp64 oracle, with and
without rounding the residual stream (CPU; DESIGN.md §8 item 5)."""
import sys, numpy as np
sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import hybridsim_oracle as O
def bf(x):  # round to bf16 (nearest even) in fp64
    a = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((a + 0x7FFF + ((a >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)
def fwd(ids, w, round_res=True, round_other=True):
    R = bf if round_other else (lambda v: v)
    RR = bf if round_res else (lambda v: v)
    x = RR(O.embed(ids, w)); n = x.shape[0]
    for l in range(w.config.num_layers):
        lw, e = w.layers[l], w.extras[l]
        xa = R(O.layer_norm(x, e["ln1_g"], e["ln1_b"]))
        q, k, v = R(xa @ lw["w_q"] + e["b_q"]), R(xa @ lw["w_k"] + e["b_k"]), R(xa @ lw["w_v"] + e["b_v"])
        att = R(O.attention_rows(q, k, v, [t + 1 for t in range(n)], w.config.num_heads, True))
        x1 = RR(x + att @ lw["w_proj"] + e["b_o"])
        h = R(np.maximum(R(O.layer_norm(x1, e["ln2_g"], e["ln2_b"])) @ lw["w_ffn1"] + e["b_1"], 0.0))
        x = RR(x1 + h @ lw["w_ffn2"] + e["b_2"])
    return R(O.layer_norm(x, w.final_ln["gamma"], w.final_ln["beta"]))
cfg = O.ModelConfig(num_layers=2, hidden_dim=256, num_heads=2, ffn_dim=512, vocab_size=512, tokens_per_block=8).validate()
w = O.with_opt_extras(O.prepare_weights(O.generate_weights(cfg, 42, 96)), 42)
rng = np.random.default_rng(0)
e_all, e_nores = [], []
for s in range(60):
    ids = rng.integers(0, 512, int(rng.integers(1, 60))).tolist()
    ref = O.forward_prompt_opt(ids, w).output[-1]
    rel = lambda a: float(np.abs(a - ref).max() / np.abs(ref).max())
    e_all.append(rel(fwd(ids, w)[-1])); e_nores.append(rel(fwd(ids, w, round_res=False)[-1]))
print("bf16 everywhere: max %.3e median %.3e" % (max(e_all), np.median(e_all)))
print("fp32/64 residual: max %.3e median %.3e" % (max(e_nores), np.median(e_nores)))
x = O.embed([1,2,3], w); print("embed mean/std", x.mean(), x.std())
