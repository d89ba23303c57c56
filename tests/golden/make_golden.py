"""Generate tests/golden/* by running the UNMODIFIED reference (hybridsim,
built from /root/reference/proj/src by oracle/Makefile into
oracle/_ref/libhybridsim_ref.so) through the ctypes shim.

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin the oracle restatement (tests/test_oracle.py) and the
product's host logic (tests/test_host_cpu.py) without needing the reference
at test time. Outputs: golden.npz (numerics), golden.json (integer/planner).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))

import hybridsim_oracle as O  # noqa: E402
import ref_lib as R  # noqa: E402


def weights_case(out, tag, L, d, H, f, V, tpb, seed, max_seq, rescale):
    rw = R.RefWeights(L, d, H, f, V, tpb, seed, max_seq)
    raw = {"emb": rw.get(0), "pos": rw.get(1)}
    for l in range(L):
        for i, n in enumerate(O.WEIGHT_NAMES):
            raw[f"{n}{l}"] = rw.get(2 + i, l)
    if rescale:  # push the oracle-prepared (rescaled, bf16) weights into the reference
        cfg = O.ModelConfig(num_layers=L, hidden_dim=d, num_heads=H, ffn_dim=f, vocab_size=V,
                            tokens_per_block=tpb).validate()
        ow = O.prepare_weights(O.generate_weights(cfg, seed, max_seq))
        rw.set(0, 0, ow.embedding)
        rw.set(1, 0, ow.positional)
        for l in range(L):
            for i, n in enumerate(O.WEIGHT_NAMES):
                rw.set(2 + i, l, ow.layers[l][n])
    else:
        # keep small raw tensors for the bit-exact generator pin
        for k, v in raw.items():
            out[f"{tag}/raw/{k}"] = v
    rng = np.random.default_rng(seed)
    ids = rng.integers(0, V, 12).astype(np.int32)
    ins, k, v, o = rw.forward_prompt(ids)
    out[f"{tag}/ids"] = ids
    out[f"{tag}/layer_inputs"] = ins
    out[f"{tag}/k"] = k
    out[f"{tag}/v"] = v
    out[f"{tag}/output"] = o
    tok = int(rng.integers(0, V))
    go, gk, gv = rw.generation_step(tok, len(ids), k, v)
    out[f"{tag}/gen_token"] = np.array([tok])
    out[f"{tag}/gen_output"] = go
    out[f"{tag}/gen_k"] = gk
    out[f"{tag}/gen_v"] = gv
    rk, rv = rw.recompute_kv(L - 1, ins[L - 1])
    out[f"{tag}/recompute_k"] = rk
    out[f"{tag}/recompute_v"] = rv


def config1_case(out, B=4, P=128, G=32, seed=42):
    """BASELINE configs[0] on the reference: OPT-125M shape (rescaled, fp16
    weights pushed in), B prompts of P tokens, G greedy tokens through the
    tied head (x E^T; an extension — the reference has no LM head). Request
    b: forward_prompt(prompt[:-1]) (decoder.cpp:144-157), then G
    generation_steps (decoder.cpp:159-174) fed prompt[-1], t0, t1, ...; the
    context of every step is assembled as in verify.cpp:62-73 at KV:ACT 0.5
    (ACT, KV, ACT, ... blocks of 16): ACT-kind prompt blocks are rebuilt by
    recompute_kv_from_activation from their layer inputs, KV-kind blocks and
    decode-grown rows are the stored K,V. Saves per step the fed token, the
    output x, the greedy token and its top-2 logit margin."""
    L, d, H, f, V, tpb = 12, 768, 12, 3072, 50272, 16
    cfg = O.ModelConfig(num_layers=L, hidden_dim=d, num_heads=H, ffn_dim=f, vocab_size=V,
                        tokens_per_block=tpb).validate()
    rw = R.RefWeights(L, d, H, f, V, tpb, seed, P + G + 1)
    ow = O.prepare_weights(O.generate_weights(cfg, seed, P + G + 1))
    rw.set(0, 0, ow.embedding)
    rw.set(1, 0, ow.positional)
    for l in range(L):
        for i, n in enumerate(O.WEIGHT_NAMES):
            rw.set(2 + i, l, ow.layers[l][n])
    E = ow.embedding
    rng = np.random.default_rng(3)
    prompts = rng.integers(0, V, (B, P)).astype(np.int32)
    fed = np.zeros((G, B), np.int32)
    toks = np.zeros((G, B), np.int32)
    xs = np.zeros((G, B, d), np.float32)
    margin = np.zeros((G, B))
    for b in range(B):
        ins, k, v, _ = rw.forward_prompt(prompts[b, :-1])
        n0 = P - 1
        for blk in range(0, (n0 + tpb - 1) // tpb, 2):  # ACT-kind blocks (tie -> ACT first)
            sl = slice(blk * tpb, min((blk + 1) * tpb, n0))
            for l in range(L):
                k[l, sl], v[l, sl] = rw.recompute_kv(l, ins[l, sl])
        tok = int(prompts[b, -1])
        for g in range(G):
            o, nk, nv = rw.generation_step(tok, n0 + g, k, v)
            k = np.concatenate([k, nk[:, None, :]], axis=1)
            v = np.concatenate([v, nv[:, None, :]], axis=1)
            lg = o[0] @ E.T
            top = np.argsort(lg)[-2:]
            fed[g, b] = tok
            toks[g, b] = int(top[1])
            xs[g, b] = o[0]
            margin[g, b] = (lg[top[1]] - lg[top[0]]) / np.abs(lg).max()
            tok = int(top[1])
    out["config1/prompts"] = prompts
    out["config1/fed"] = fed
    out["config1/tokens"] = toks
    out["config1/x"] = xs
    out["config1/margin"] = margin


def tables_case(tpb, lens, gens, mode, act_host, kv_host, act_gpu, frees=()):
    """Replay simulate()'s add_token order (sim.cpp:150-223, 308-310) on the
    reference HybridCache + next_block_kind."""
    a, k, g = act_host, kv_host, act_gpu
    if mode in ("kv_only", "token_recompute"):
        k += a // 2
        a = 0
        g = 0
    elif mode == "act_only":
        a += 2 * k
        k = 0
    c = R.RefCache(tpb, k, 0, a, g)
    ids = [f"r{i}" for i in range(len(lens))]
    for rid, n in zip(ids, lens):
        c.create_request(rid, n)

    def add(rid):
        if c.context_len(rid) % tpb == 0:
            if mode == "hybrid":
                na, nk = c.blocks_by_kind(rid)
                kind = R.next_block_kind(na, nk, a, k)
            else:
                kind = "ACT" if mode == "act_only" else "KV"
            c.append_block(rid, kind)
        c.fill_token(rid)

    for rid, n in zip(ids, lens):
        for _ in range(n):
            add(rid)
    for it in range(max(gens)):
        for rid, g_ in zip(ids, gens):
            if it < g_:
                add(rid)
    for rid in frees:
        c.free_request(rid)
    return json.loads(c.dump_json())


def main():
    if not R.available():
        sys.exit("build the reference first: make -C oracle")
    out = {}
    weights_case(out, "toy", 2, 32, 4, 64, 50, 4, 42, 40, rescale=False)
    weights_case(out, "toy_rescaled", 3, 256, 2, 512, 512, 16, 7, 40, rescale=True)
    weights_case(out, "opt125m_shape", 12, 768, 12, 3072, 50272, 16, 42, 160, rescale=True)
    config1_case(out)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)

    j = {"block_tables": [], "next_block_kind": [], "plan": [], "fit_linear": [], "equivalence": [],
         "flops": [], "bytes_of": []}
    scenarios = [
        dict(tpb=16, lens=[128] * 4, gens=[32] * 4, mode="hybrid", act_host=40, kv_host=40, act_gpu=0),
        dict(tpb=16, lens=[128] * 4, gens=[32] * 4, mode="hybrid", act_host=40, kv_host=40, act_gpu=6),
        dict(tpb=16, lens=[100, 37, 64], gens=[20, 9, 33], mode="hybrid", act_host=30, kv_host=60, act_gpu=2),
        dict(tpb=8, lens=[50, 51], gens=[7, 30], mode="kv_only", act_host=10, kv_host=40, act_gpu=3),
        dict(tpb=8, lens=[50, 51], gens=[7, 30], mode="act_only", act_host=10, kv_host=40, act_gpu=3),
        dict(tpb=5, lens=[23, 17, 9], gens=[11, 4, 19], mode="hybrid", act_host=14, kv_host=6, act_gpu=1),
        dict(tpb=16, lens=[64, 64, 64], gens=[16, 16, 16], mode="hybrid", act_host=100, kv_host=50, act_gpu=0,
             frees=["r1"]),
    ]
    for s in scenarios:
        j["block_tables"].append({"args": s, "dump": tables_case(**s)})
    rng = np.random.default_rng(11)
    for _ in range(40):
        ah, kh = int(rng.integers(0, 50)), int(rng.integers(1, 50))
        a, k = int(rng.integers(0, 30)), int(rng.integers(0, 30))
        j["next_block_kind"].append([a, k, ah, kh, R.next_block_kind(a, k, ah, kh)])
    for _ in range(60):
        b = [float(rng.uniform(1e-7, 1e-4)), float(rng.uniform(0, 1e-3)), float(rng.uniform(1e-7, 1e-4)),
             float(rng.uniform(0, 1e-3)), float(rng.uniform(1e-4, 5e-2))]
        sa = float(rng.choice([1024.0, 4096.0, 28672.0 * 48]))
        mem = [float(rng.uniform(1e5, 1e9)), float(rng.uniform(0, 1e4)), 2 * sa, sa]
        tpb = int(rng.choice([4, 8, 16]))
        ag = int(rng.integers(0, 5))
        try:
            res = R.plan_host_allocation(b, mem, tpb, ag)
            err = None
        except R.RefError as e:
            res, err = None, e.code
        j["plan"].append({"bundle": b, "mem": mem, "tpb": tpb, "act_gpu": ag, "alloc": res, "err": err,
                          "init": list(R.initial_cache_allocation(b, tpb, ag))})
    for _ in range(20):
        n = int(rng.integers(2, 12))
        xs = rng.uniform(1, 1e5, n).round().tolist()
        ys = (np.array(xs) * rng.uniform(1e-9, 1e-6) + rng.uniform(-1e-4, 1e-3)
              + rng.normal(0, 1e-5, n)).tolist()
        j["fit_linear"].append({"x": xs, "y": ys, "fit": R.fit_linear(xs, ys).tolist()})
    for seed in range(25):
        dev, ex = R.equivalence(seed)
        j["equivalence"].append([seed, dev, ex])
    lib = R.lib()
    for kind in range(6):
        for (d, f, n, k, L) in [(4096, 16384, 1, 0, 48), (7168, 28672, 64, 3, 48), (768, 3072, 1000, 11, 12)]:
            j["flops"].append([kind, d, f, n, k, L, lib.ref_flop_count(kind, d, f, n, k, L)])
    for d, tpb in [(7168, 1), (7168, 16), (768, 16), (4096, 8)]:
        j["bytes_of"].append([d, tpb, int(lib.ref_bytes_of(0, d, tpb, 2)), int(lib.ref_bytes_of(1, d, tpb, 2))])
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(j, fh, indent=0)
    print("wrote", os.path.join(HERE, "golden.npz"), os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
