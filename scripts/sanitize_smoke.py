"""Small run of every kernel of the path for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): engine prefill + decode in
hybrid mode with host pools and streamed weights, token-recompute mode,
split-K and split-attention paths, the chunked prefill pipeline, OPT layers
and the head-sharded tensor-parallel group.

    compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2501_01792_b200 import api, kernels  # noqa: E402


def main():
    cfg = api.ModelConfig(num_layers=2, hidden_dim=256, num_heads=2, ffn_dim=512, vocab_size=512, tokens_per_block=16)
    rng = np.random.default_rng(0)
    prompts = [rng.integers(0, 512, 37).tolist(), rng.integers(0, 512, 20).tolist()]
    eng = api.Engine(cfg, seed=3, max_seq=64, max_batch=2, weights_on_device=False,
                     caps=api.PoolCaps(kv_host=8, act_host=8, act_gpu=1), allocation=api.HostAllocation(1, 1))
    eng.prefill(["a", "b"], prompts)
    for _ in range(2):
        eng.decode_step(["a", "b"], [1, 2], want_logits=True, want_argmax=True)
    eng.configure_cache(api.PoolCaps(kv_host=8), mode="token_recompute", recompute_ratio=0.5)
    eng.prefill(["a"], [prompts[0]])
    eng.decode_step(["a"], [5])
    eng.close()
    a = kernels.f32_to_f16_bits(rng.uniform(-1, 1, (64, 1024)))
    w = kernels.f32_to_f16_bits(rng.uniform(-0.05, 0.05, (256, 1024)))
    kernels.gemm_f16_splitk(a, w, 4, 1, 128)
    # weight-streaming decode GEMM: units cut over 7 CTAs (partials + reduce), whole units, bias + residual
    bias = kernels.f32_to_f16_bits(rng.uniform(-1, 1, (256,)))
    kernels.gemm_f16_wstream(a, w, 0, bias, kernels.f32_to_f16_bits(rng.uniform(-1, 1, (64, 256))), ctas=7)
    kernels.gemm_f16_wstream(a[:5], w, 1, ctas=0)
    kernels.gemm_f16_wstream(a, w, 3, ctas=3)
    q = kernels.f32_to_f16_bits(rng.uniform(-1, 1, (2, 256)))
    pool = kernels.f32_to_f16_bits(rng.uniform(-1, 1, (8, 2, 2, 16, 128)))
    refs = np.array([[0, 1, 2, 3], [4, 5, 6, 7]], np.int32)
    kernels.decode_attention(q, pool, pool, refs, np.array([4, 3], np.int32), np.array([60, 40], np.int32), 2,
                             True, 2)
    # persistent two-tile prefill attention: several items per CTA, odd tile count
    qkv = kernels.f32_to_f16_bits(rng.uniform(-1, 1, (2 * 640, 3 * 256)))
    kernels.prefill_attention(qkv, 2, 640, 2)
    # session-2 paths: chunked offloaded prefill (store stream), OPT layers
    # (LayerNorm, bias / residual epilogues), head-sharded TP over the
    # in-process group (all-gather + fp32 all-reduce), flash prefill attention
    ocfg = api.ModelConfig(num_layers=2, hidden_dim=256, num_heads=4, ffn_dim=512, vocab_size=512)
    e2 = api.Engine(ocfg, seed=5, max_seq=64, max_batch=2, weights_on_device=False, arch="opt",
                    caps=api.PoolCaps(kv_host=8, act_host=8, act_gpu=1), allocation=api.HostAllocation(1, 1),
                    max_prefill_tokens=24)
    e2.prefill(["a", "b"], prompts)
    e2.decode_step(["a", "b"], [3, 4], want_logits=True)
    e2.close()
    import threading
    group = api.TensorParallel.local_group(2)
    engs = [api.Engine(ocfg, seed=5, max_seq=64, max_batch=2, weights_on_device=bool(r), arch="opt", tp=group[r],
                       caps=api.PoolCaps(kv_host=8, act_host=8, act_gpu=1), allocation=api.HostAllocation(1, 1))
            for r in range(2)]

    def run(e):
        e.prefill(["a", "b"], prompts)
        e.decode_step(["a", "b"], [3, 4])
    ts = [threading.Thread(target=run, args=(e,)) for e in engs]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in engs:
        e.close()
    # batch-partitioned ranks sharing one weight stream (in-process group, 2 decode steps
    # so the cross-step prefetch of layers 0/1 is sharded too); block sizes 4 and 64
    wgroup = api.TensorParallel.local_group(2)
    wengs = [api.Engine(cfg, seed=3, max_seq=64, max_batch=2, weights_on_device=False, weight_share=wgroup[r],
                        caps=api.PoolCaps(kv_host=8, act_host=8, act_gpu=1), allocation=api.HostAllocation(1, 1))
             for r in range(2)]

    def run_ws(r):
        ids = [f"w{r}a", f"w{r}b"]
        wengs[r].prefill(ids, prompts)
        for _ in range(2):
            wengs[r].decode_step(ids, [5, 6])
    ts = [threading.Thread(target=run_ws, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in wengs:
        e.close()
    for tpb in (4, 64):
        c3 = api.ModelConfig(num_layers=1, hidden_dim=256, num_heads=2, ffn_dim=512, vocab_size=512,
                             tokens_per_block=tpb)
        e3 = api.Engine(c3, seed=7, max_seq=96, max_batch=2, weights_on_device=True,
                        caps=api.PoolCaps(kv_host=40, act_host=40, act_gpu=2), allocation=api.HostAllocation(1, 1))
        e3.prefill(["a", "b"], prompts)
        e3.decode_step(["a", "b"], [1, 2])
        e3.close()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
