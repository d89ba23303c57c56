"""Debug one failing fuzz seed (not a test)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)
import numpy as np
import hybridsim_oracle as O
import test_engine_gpu as T
from paper_2501_01792_b200.api import HostAllocation, PoolCaps
from paper_2501_01792_b200 import CapacityError


worst_lg = [0.0]


def run(seed, graphs=True, wod=None, arch="opt", verbose=False):
    worst = 0.0
    cfg = T.small_cfg(L=2, d=256, H=2, f=512, tpb=8)
    w = T.opt_weights(cfg, max_seq=96) if arch == "opt" else T.oracle_weights(cfg, max_seq=96)
    fwd = O.forward_prompt_opt if arch == "opt" else O.forward_prompt
    rng = np.random.default_rng(1000 + seed)
    caps = PoolCaps(kv_host=14, act_host=10, act_gpu=3)
    alloc = HostAllocation(int(rng.integers(1, 4)), int(rng.integers(1, 4)))
    eng = (T.make_opt_engine if arch == "opt" else T.make_engine)(
        cfg, w, max_batch=4, max_seq=96, caps=caps, mode="hybrid", allocation=alloc,
        weights_on_device=bool(seed % 2) if wod is None else wod)
    eng.set_graphs(graphs)
    seqs, next_id = {}, 0
    for op in range(70):
        live = list(seqs)
        r = rng.random()
        if (r < 0.25 and len(live) < 4) or not live:
            n_new = int(rng.integers(1, min(2, 4 - len(live)) + 1))
            ids = [f"q{next_id + i}" for i in range(n_new)]
            prompts = [rng.integers(0, cfg.vocab_size, int(rng.integers(0, 30))).tolist() for _ in ids]
            try:
                eng.prefill(ids, prompts)
            except CapacityError:
                continue
            next_id += n_new
            seqs.update({i: list(p) for i, p in zip(ids, prompts)})
            if verbose:
                print("prefill", ids, [len(p) for p in prompts])
        elif r < 0.35:
            victim = live[int(rng.integers(0, len(live)))]
            eng.free_request(victim)
            del seqs[victim]
            if verbose:
                print("free", victim)
        else:
            batch = [x for x in live if rng.random() < 0.7] or live[:1]
            batch = [x for x in batch if len(seqs[x]) < 90]
            if not batch:
                continue
            toks = rng.integers(0, cfg.vocab_size, len(batch)).tolist()
            try:
                res = eng.decode_step(batch, toks, want_x=True, want_logits=True)
            except CapacityError:
                continue
            for i, rid in enumerate(batch):
                seqs[rid].append(toks[i])
                out = fwd(seqs[rid], w).output[-1:]
                ref = out[0]
                e = T.rel(T.f64(res["x"][i]), ref)
                worst_lg[0] = max(worst_lg[0], T.rel(res["logits"][i], O.logits_tied(out, w)[0]))
                tab = [(int(x.kind), int(x.location), x.pbn, x.filled_tokens) for x in eng.cache.table(rid).entries]
                worst = max(worst, e)
                if e > 1e-2 and verbose:
                    print(f"op {op} decode {batch} {rid} len {len(seqs[rid])} rel {e:.3e} table {tab}")
    return worst


if __name__ == "__main__":
    for arch in ("opt", "reference"):
        worst_lg[0] = 0.0
        ws = [run(seed, arch=arch) for seed in range(100, 140)]
        print(arch, "worst logits rel over all seeds %.3e" % worst_lg[0])
        print(arch, "worst rel per seed: max %.3e median %.3e; > 1e-2 in %d of %d" %
              (max(ws), float(np.median(ws)), sum(w > 1e-2 for w in ws), len(ws)), flush=True)
        print(" ".join(f"{w:.2e}" for w in ws), flush=True)
