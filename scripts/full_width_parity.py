"""One-off parity check at full model width (default OPT-30B: d 7168, 56
heads, f 28672; one layer, small vocab) — the sizes the unit tests do not
reach: hybrid host pools, streamed weights, prefill of 2 ragged prompts + 3
decode steps vs the fp64 oracle on the same bf16 weights. Writes
gpurun_out/full_width_parity[_<model>_<arch>].json.

    python scripts/full_width_parity.py [--model opt-66b] [--arch opt]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import hybridsim_oracle as O  # noqa: E402  (checker)
from paper_2501_01792_b200 import api  # noqa: E402


def rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="opt-30b")
    ap.add_argument("--arch", default="reference", choices=["reference", "opt"])
    a = ap.parse_args(argv)
    t0 = time.time()
    pre = api.ModelConfig.preset(a.model)
    d, H, f = pre.hidden_dim, pre.num_heads, pre.ffn_dim
    cfg = O.ModelConfig(num_layers=1, hidden_dim=d, num_heads=H, ffn_dim=f, vocab_size=1024,
                        tokens_per_block=16).validate()
    w = O.prepare_weights(O.generate_weights(cfg, 42, 128))
    if a.arch == "opt":
        w = O.with_opt_extras(w, 42)
    fwd = O.forward_prompt_opt if a.arch == "opt" else O.forward_prompt
    mc = api.ModelConfig(num_layers=1, hidden_dim=d, num_heads=H, ffn_dim=f, vocab_size=1024)
    wd = {"embedding": w.embedding, "positional": w.positional, "layers": w.layers}
    if a.arch == "opt":
        wd.update(extras=w.extras, final_ln=w.final_ln)
    eng = api.Engine(mc, weights=wd, max_batch=2, weights_on_device=False,
                     caps=api.PoolCaps(kv_host=8, act_host=8, act_gpu=1), allocation=api.HostAllocation(1, 1),
                     mode="hybrid", arch=a.arch)
    rng = np.random.default_rng(5)
    prompts = [rng.integers(0, 1024, 37).tolist(), rng.integers(0, 1024, 50).tolist()]
    eng.prefill(["a", "b"], prompts)
    seqs = [list(p) for p in prompts]
    errs = []
    for step in range(3):
        toks = rng.integers(0, 1024, 2).tolist()
        res = eng.decode_step(["a", "b"], toks, want_x=True, want_logits=True)
        for b in range(2):
            seqs[b].append(toks[b])
            out = fwd(seqs[b], w).output[-1:]
            errs.append({"step": step, "request": b, "x_rel": rel(O.f16_bits_to_f64(res["x"][b]), out[0]),
                         "logits_rel": rel(res["logits"][b], O.logits_tied(out, w)[0])})
    # recomputed K/V of the ACT blocks and stored KV blocks vs the oracle trace
    tr = fwd(seqs[1], w)
    row, blk_errs = 0, []
    for e in eng.cache.table("b").entries:
        n = e.filled_tokens
        blk = O.f16_bits_to_f64(eng.read_block(e.kind, e.location, e.pbn, 0))
        if int(e.kind) == 1:  # ACT blocks hold the layer input (OPT: LN1 of it)
            want = tr.act[0] if a.arch == "opt" else tr.layer_inputs[0]
            blk_errs.append(rel(blk[:n], want[row:row + n]))
        else:
            blk_errs.append(rel(blk[0].transpose(1, 0, 2).reshape(16, d)[:n], tr.k[0][row:row + n]))
        row += n
    res = {"config": f"{a.model} width (d {d}, {H} heads x {d // H}, f {f}), arch {a.arch}, 1 layer, vocab 1024; "
                     "hybrid 1:1 host pools + 1 ACT/gpu block, weights streamed",
           "decode": errs, "max_rel": max(max(e["x_rel"], e["logits_rel"]) for e in errs),
           "cache_block_max_rel": max(blk_errs), "tolerance": 1e-2, "seconds": time.time() - t0}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    tag = "" if (a.model, a.arch) == ("opt-30b", "reference") else f"_{a.model}_{a.arch}"
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", f"full_width_parity{tag}.json"), "w"), indent=1)
    print(json.dumps({k: res[k] for k in ("max_rel", "cache_block_max_rel", "seconds")}))
    assert res["max_rel"] <= 1e-2 and res["cache_block_max_rel"] <= 1e-2


if __name__ == "__main__":
    main()
