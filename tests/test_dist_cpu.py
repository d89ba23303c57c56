"""N>1 host path on CPU: world_size-2 gloo process group exercising bench.py's
rank plumbing (barrier, max-over-ranks timing, summed tokens) and the
batch partition (each rank its own requests / cache, no data collective)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys, json
sys.path.insert(0, ROOT)
import bench
from paper_2501_01792_b200 import api
world, rank, local, dist = bench.dist_setup(None)
assert world == 2 and dist.get_backend() == "gloo"
# per-rank partition of the batch: rank-local allocator, identical policy
cache = api.HybridCache(16, api.PoolCaps(64, 0, 64, 0))
alloc = api.HostAllocation(1, 2)
ids = [f"g{rank}r{i}" for i in range(4)]
for rid in ids:
    cache.create_request(rid, 40)
    for _ in range(40):
        if cache.context_len(rid) % 16 == 0:
            cache.append_block(rid, api.next_block_kind(*cache.blocks_by_kind(rid), alloc))
        cache.fill_token(rid)
t_local = 1.5 + rank          # pretend device seconds
bench.barrier(dist)
t = bench.max_over_ranks(dist, t_local)
tok = bench.sum_over_ranks(dist, 4.0 * 10)
print(json.dumps({"rank": rank, "max_t": t, "tokens": tok,
                  "tables": json.loads(cache.dump_json())["requests"][0]["entries"]}))
dist.destroy_process_group()
"""


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_bench_plumbing(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(f"ROOT = {ROOT!r}\n" + WORKER)
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE="2", LOCAL_WORLD_SIZE="2",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        o, e = p.communicate(timeout=240)
        assert p.returncode == 0, e
        outs.append(o.strip().splitlines()[-1])
    import json
    res = [json.loads(o) for o in outs]
    assert all(r["max_t"] == 2.5 for r in res)            # max over ranks
    assert all(r["tokens"] == 80.0 for r in res)          # whole-job tokens
    assert res[0]["tables"] == res[1]["tables"]           # same policy, independent pools


def test_reference_arm_nonzero_ranks_exit_silently(tmp_path):
    """--impl reference under N>1: rank 0 alone prints; others exit 0."""
    code = f"""
import sys, json
sys.path.insert(0, {ROOT!r})
import bench
class A: pass
a = A(); a.gpus = 2; a.steps = 1; a.warmup = 0; a.prompt = 8; a.ratio = 0.5; a.batch = 2; a.gen = 4
bench.reference_arm(a, 2, 1, None)
print("done")
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == "done"


def test_reference_arm_never_loads_the_product():
    """bench.py --impl reference runs the reference library only: the product
    package is never imported and libhybridcache_b200.so never mapped; its
    config equals the one our arm builds (same r from the same bundle)."""
    import importlib.util
    if importlib.util.find_spec("ref_lib") is None:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref_lib as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    code = f"""
import sys, json
sys.path.insert(0, {ROOT!r})
sys.argv = ["bench.py", "--impl", "reference", "--model", "opt-6.7b", "--layers", "1", "--steps", "1",
            "--warmup", "0", "--batch", "4", "--prompt", "64", "--gen", "16"]
import bench
bench.main()
assert not any(m.startswith("paper_2501_01792_b200") for m in sys.modules), "product imported"
maps = open("/proc/self/maps").read()
assert "libhybridcache_b200" not in maps, "product library mapped"
assert "libhybridsim_ref" in maps
"""
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["cpu_baseline"]["single_thread"]["cores"] == 1
    assert line["config"]["timed_context"] == 64 + 8


def test_both_arms_plan_the_same_ratio():
    """The reference arm's planner (the reference's plan_host_allocation) and
    ours (bit-exact restatement) pick the same r from the committed bundle."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import bench
    import ref_lib as R
    from paper_2501_01792_b200 import api
    if not R.available():
        pytest.skip("oracle/_ref not built")
    path = os.path.join(ROOT, "profiles", "planner_bundle_opt-30b.json")
    cfg = api.ModelConfig.preset("opt-30b")
    ref = bench.planned_ratio(R.parse_bundle(path), cfg, 128 * (1024 + 256), R.plan_host_allocation)
    ours = bench.planned_ratio(bench.read_bundle(path), cfg, 128 * (1024 + 256),
                               lambda b5, m4, tpb, ag: list(api.plan_host_allocation(
                                   api.TimingBundle(api.LinearTimeModel(b5[0], b5[1]),
                                                    api.LinearTimeModel(b5[2], b5[3]), b5[4]),
                                   api.MemoryBudget(*m4), tpb, ag).__dict__.values()))
    assert ref == ours and 0.0 < ref[0] < 1.0


def test_config4_strong_split_covers_global_batch():
    """Config 4 (OPT-66B, global batch 128 over 2/4/8 ranks): the per-rank
    slices partition the global batch exactly (strong scaling)."""
    sys.path.insert(0, ROOT)
    import bench
    sys.argv = ["bench.py", "--config", "4"]
    a = bench.parse()
    assert a.model == "opt-66b" and a.global_batch == 128 and a.ratio == -1.0 and a.scaling == "strong"
    for world in (1, 2, 3, 4, 8):
        sizes = [bench.per_rank_batch(a, world, r) for r in range(world)]
        assert sum(sizes) == 128 and max(sizes) - min(sizes) <= 1
    sys.argv = ["bench.py"]
    b = bench.parse()
    assert b.model == "opt-30b" and b.scaling == "weak" and b.ratio == -1.0  # planner-chosen by default
    assert bench.per_rank_batch(b, 8, 7) == 128
    sys.argv = ["bench.py", "--config", "5"]  # the OPT-13B ratio sweep
    c = bench.parse()
    assert (c.model, c.prompt, c.batch, c.scaling) == ("opt-13b", 2048, 64, "weak")
    assert c.sweep.split(",")[:5] == ["0", "0.25", "0.5", "0.75", "1"] and "tr0.5" in c.sweep
    sys.argv = ["bench.py"]


def test_weight_share_group_selection(monkeypatch):
    """The shared weight stream is an opt-in variant (--share-weights; the
    default partition has no collective) and needs one GPU per rank on one
    node; world 1 never shares."""
    sys.path.insert(0, ROOT)
    import bench
    sys.argv = ["bench.py"]
    a = bench.parse()
    assert not a.share_weights
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "2")
    assert bench.weight_share_group(a, 2, 0, 0, None) == (None, 1)  # default: whole-layer streams
    sys.argv = ["bench.py", "--share-weights"]
    b = bench.parse()
    assert bench.weight_share_group(b, 1, 0, 0, None) == (None, 1)
    assert bench.weight_share_group(b, 2, 0, 0, None) == (None, 1)  # no CUDA devices here: ranks share none
    sys.argv = ["bench.py"]


def test_calibrate_planner_widens_budget_for_small_batches():
    """Config 4 split 8 ways (16 requests next to 130 GB of weights): the
    reference's workload-sized budget (0.9 x the workload) cannot hold Alg. 1's
    initial blocks; the bench widens the factor until the planner has room
    and reports it. Larger batches keep the reference's 0.9."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2501_01792_b200 import api

    class FakeEngine:  # measured rates of a B200: recompute 1.9e-7 s/token, link 6.7e-7 s/token (OPT-66B)
        def time_kv_gen(self, n, reps=3):
            return 1.9e-7 * n + 3e-5

        def time_load_kv(self, n, reps=2):
            return 6.7e-7 * n + 8e-6

    cfg = api.ModelConfig.preset("opt-66b")
    for batch, want_factor in ((16, "6.0"), (64, "1.5"), (128, "0.9")):
        p = bench.calibrate_planner(FakeEngine(), cfg, 55.6, 10 * 1024 * 16, batch * (1024 + 256))
        assert 0.0 < p["planned_r"] <= 1.0
        assert len(p["kv_gen_samples"]) >= 2
        if want_factor:
            assert f"+ {want_factor} x" in p["m_host_source"]


@pytest.mark.parametrize("r", [0.0, 0.25, 1 / 3, 0.5, 0.75, 0.9432, 1.0])
def test_pool_plan_covers_the_workload(r):
    """bench.pool_plan sizes the host pools for B requests growing to P+steps
    tokens at ACT share r: replaying next_block_kind (plan.cpp:154-164) block
    by block never needs more blocks of a kind than the plan provides, and
    host_layers_for folds layers only as far as the pinned budget demands."""
    sys.path.insert(0, ROOT)
    import math
    import bench
    from paper_2501_01792_b200 import api
    cfg = api.ModelConfig.preset("opt-30b")
    B, P, steps = 8, 1024, 12
    mode, alloc, caps = bench.pool_plan(cfg, B, P, steps, r)
    nb = math.ceil((P + steps) / cfg.tokens_per_block)
    act = kv = 0
    for _ in range(B):
        a = k = 0
        for _ in range(nb):
            if mode == "hybrid":
                kind = api.next_block_kind(a, k, alloc)
            else:
                kind = api.BlockKind.ACT if mode == "act_only" else api.BlockKind.KV
            if kind == api.BlockKind.ACT:
                a += 1
            else:
                k += 1
        act, kv = act + a, kv + k
    assert act <= caps.act_host and kv <= caps.kv_host
    if 0 < r < 1:
        assert abs(act / (act + kv) - r) <= 1.0 / nb + 1e-9  # the realised share tracks the setting
    per_layer = caps.kv_host * api.HybridCache.bytes_of("KV", cfg) + caps.act_host * api.HybridCache.bytes_of("ACT", cfg)
    for budget in (per_layer * 48 + 1e9, per_layer * 10 + 1e9, 1.0):
        lp = bench.host_layers_for(cfg, caps, budget, 1e9)
        assert 2 <= lp <= cfg.num_layers
        assert lp == cfg.num_layers or lp * per_layer <= budget - 1e9 or lp == 2
