#!/usr/bin/env python
"""Benchmark: offloaded OPT-30B-shape decode over the KV-activation hybrid
cache (BASELINE.json configs[2]: weights + hybrid cache in pinned host
memory, batch 128, prompt 1024, gen 256), generated tokens/s.

A "step" is one decode iteration: all 48 layers for the whole per-GPU batch
(128 requests), streaming each layer's weights and host KV/ACT blocks over the
host link, recomputing K/V of the ACT blocks on the tensor cores, attention
over the hybrid block table, and the new token's cache writes. Multi-GPU:
batch-partitioned (each rank its own 128 requests, pools and host link; no
collective on the data path) -> scaling "weak".

    python bench.py [--gpus N --steps K --warmup W] [--ratio R] [--impl reference]

Prints ONE JSON line on rank 0. See DESIGN.md §Measurement for every field.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "generated tokens/sec, OPT-30B offloaded, per KV:ACT ratio, at 1/2/4/8 B200"
# NVLink 5 model for the emulated multi-rank variants: NCCL all-reduce /
# all-gather bus bandwidth measured on B200 NVSwitch nodes (725 GB/s;
# /opt/skills/guides/B200_PROFILING.md; peer copies reach 770 GB/s per direction)
NVLINK_BUSBW = 725e9
# recompute GEMM DRAM bytes per ACT row from ncu captures at OPT-30B width, default raster
# (1-SM kernel, group_m 16, A kept in L2), scaled by rows in the bench's roofline.traffic:
# profiles/r02_recompute_dram_sweep.txt and r02_ncu_recompute_fused.txt
RECOMPUTE_NCU_BYTES_PER_ROW = (15.37e9 + 3.51e9) / 122880
RECOMPUTE_NCU_BYTES_PER_ROW_FUSED = (14.22e9 + 0.23e9) / 122880
RECOMPUTE_NCU_NOTE = ("fused (kAttnPart) 14.45 GB, kKvPaged 18.88 GB at 122880 rows; [Wk|Wv] (205 MB > L2) "
                      "re-read once per 16-tile M group, profiles/r02_recompute_dram_sweep.txt")
# best host->device rate of the standalone link probe on this pool's B200 boxes
# (scripts/link_probe.py -> profiles/r01_link_probe.json: one copy stream,
# >= 64 MB chunks; more streams or SM zero-copy reads add nothing)
LINK_PROBE_GBS = 55.59


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=3, choices=[3, 4, 5],
                   help="BASELINE configs[] entry (1-based): 3 = OPT-30B, 128 requests per GPU (weak scaling); "
                        "4 = OPT-66B fully offloaded, global batch 128 split across the ranks (strong scaling), "
                        "planner-chosen ratio; 5 = OPT-13B, prompt 2048, ratio sweep 0 -> 1 beside pure KV and the "
                        "token-recompute baseline")
    p.add_argument("--model", default="")
    p.add_argument("--batch", type=int, default=0, help="requests per GPU (config 3 default 128)")
    p.add_argument("--global-batch", type=int, default=0, help="total requests split across ranks (config 4: 128)")
    p.add_argument("--tp", type=int, default=1,
                   help="head-sharded tensor parallelism over the torchrun ranks (NCCL): every rank serves the whole "
                        "global batch for H/N heads and streams 1/N of the weights, KV and ACT bytes")
    p.add_argument("--tp-emulate", type=int, default=0,
                   help="time ONE rank of an N-way head-sharded group on this single GPU (collectives skipped, "
                        "NVLink time modelled) and print a projection line instead of the bench line")
    p.add_argument("--share-weights", action="store_true",
                   help="N>1 variant: the batch-partitioned ranks share ONE weight stream (1/N of every layer per "
                        "host link + an NVLink all-gather). Default off: the north star's partition has no "
                        "collective — every rank streams whole layers over its own host link")
    p.add_argument("--share-emulate", type=int, default=0,
                   help="time ONE rank of N batch-partitioned ranks sharing the weight stream on this single GPU "
                        "(all-gather skipped, NVLink time modelled) and print a projection line")
    p.add_argument("--prompt", type=int, default=1024)
    p.add_argument("--gen", type=int, default=256, help="generation length of the workload (config)")
    p.add_argument("--ratio", type=float, default=None,
                   help="ACT share r of context blocks; default -1 = the planner's choice from measured rates "
                        "(north-star (5)); 0.3333 = the paper's KV:ACT 2:1 for OPT-30B on an RTX 4090 (PAPER.md:714)")
    p.add_argument("--host-gb", type=float, default=0.0, help="pinned host budget per rank (0: auto)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--arch", default="reference", choices=["reference", "opt"],
                   help="decoder layer: the reference's (default) or OPT's (biases, pre-LN, residuals)")
    p.add_argument("--prefill", default="real", choices=["real", "synthetic"],
                   help="build the decode cache by the real prefill of synthetic prompts (default) or by "
                        "pattern-filled bookkeeping-only admission")
    p.add_argument("--layers", type=int, default=0, help="override num_layers (smoke/profiling only)")
    p.add_argument("--no-sweep", action="store_true", help="skip the per-ratio / planner / HBM-tier variants")
    p.add_argument("--sweep", default="0,0.3333333333333333,0.5,1,tr0.5",
                   help="ACT shares r to time besides the headline; trX = token-recompute baseline at ratio X")
    p.add_argument("--no-config2", action="store_true", help="skip the OPT-6.7B resident (config 2) variant")
    p.add_argument("--artifacts", default="", help="write the reference CLI's artifacts (kv_gen.csv, load_kv.csv, "
                                                    "bundle.json, plan.json, metrics.json, trace.json) here")
    p.add_argument("--bundle", default="committed",
                   help="timing bundle the planner ratio comes from: 'committed' = profiles/planner_bundle_<model>.json "
                        "(B200-measured, read by BOTH arms so they run the same r), 'live' = this run's calibration, "
                        "or a path")
    p.add_argument("--full-generation", action="store_true",
                   help="time the whole generation instead: real prefill of P tokens + G decode steps, every step "
                        "timed (prints the measured generation line; minutes)")
    a = p.parse_args()
    if a.config == 5:  # BASELINE configs[4]: the OPT-13B ratio sweep (batch 64 as SURVEY.md §8(d) sizes it)
        a.model = a.model or "opt-13b"
        a.prompt = 2048 if a.prompt == 1024 else a.prompt
        a.batch = a.batch or 64
        if a.sweep == "0,0.3333333333333333,0.5,1,tr0.5":
            a.sweep = "0,0.25,0.5,0.75,1,tr0.5"
    if a.config == 4:
        a.model = a.model or "opt-66b"
        a.global_batch = a.global_batch or 128
    a.model = a.model or "opt-30b"
    a.ratio = -1.0 if a.ratio is None else a.ratio
    a.scaling = "strong" if a.global_batch else "weak"
    return a


def per_rank_batch(args, world, rank):
    """Requests this rank owns: --batch per GPU (weak scaling), or an even
    split of --global-batch (strong scaling)."""
    if args.global_batch:
        world = max(world, getattr(args, "share_emulate", 0))  # an emulated rank owns its 1/N slice
        base, extra = divmod(args.global_batch, world)
        return base + (1 if rank < extra else 0)
    return args.batch or 128


# ---------------------------------------------------------------- helpers ---
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as td
        # HC_DIST_BACKEND=gloo + fewer GPUs than ranks: a plumbing smoke test of
        # the multi-rank path with several ranks sharing one device
        backend = os.environ.get("HC_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        if backend == "nccl" and local_world > torch.cuda.device_count():
            # NCCL refuses two ranks on one device: fall back to gloo for the
            # barrier / max-over-ranks plumbing (timing stays on CUDA events)
            print(f"bench: {local_world} ranks share {torch.cuda.device_count()} GPU(s); using gloo",
                  file=sys.stderr)
            backend = "gloo"
        if torch.cuda.is_available():
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
        td.init_process_group(backend=backend)
        dist = td
    return world, rank, local, dist


def parse_cpulist(text):
    cpus = set()
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        else:
            cpus.add(int(part))
    return cpus


_ALL_CPUS = None  # affinity before bind_numa (restored for the CPU baseline)


def bind_numa(local):
    """Pin this rank to the CPUs of its GPU's NUMA node before any pinned host
    allocation: cudaHostAlloc pages are placed by first touch, so each GPU's
    host pools (and its DMA reads) stay on the socket its PCIe link hangs off —
    with 8 ranks streaming ~55 GB/s each, cross-socket traffic would cap the
    aggregate. Returns the node (or None when the topology is unknown)."""
    from paper_2501_01792_b200 import kernels
    try:
        bus = kernels.device_pci_bus_id(local).lower()
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as fh:
            node = int(fh.read().strip())
        if node < 0:
            return None
        with open(f"/sys/devices/system/node/node{node}/cpulist") as fh:
            cpus = parse_cpulist(fh.read()) & os.sched_getaffinity(0)
        if cpus:
            global _ALL_CPUS
            _ALL_CPUS = os.sched_getaffinity(0)
            os.sched_setaffinity(0, cpus)
        return node
    except Exception:  # no sysfs / no GPU: leave placement to the OS
        return None


def barrier(dist):
    if dist is not None:
        dist.barrier()


def max_over_ranks(dist, x: float) -> float:
    if dist is None:
        return x
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, x: float) -> float:
    if dist is None:
        return x
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def mem_available_bytes() -> float:
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return float(line.split()[1]) * 1024
    except OSError:
        pass
    return 64e9


def mem_total_bytes() -> float:
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemTotal:"):
                    return float(line.split()[1]) * 1024
    except OSError:
        pass
    return 64e9


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            j = json.load(fh)
        return j.get("hbm_gbs", 6650.0), j.get("bf16_tflops_sustained", 1400.0), j.get("bf16_tflops", 1590.0), "measured"
    except (OSError, ValueError):
        return 6650.0, 1400.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.f.flush()
        self.f.seek(0)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU baseline ---
def cpu_reference_sample(dims, ctx: int, n_act: int, threads: int, chunk: int = 64):
    """The reference's own CPU path for this workload, bounded: ONE request at
    ONE layer of one decode step at full model width — generation_step of
    that layer over a context of `ctx` tokens (decoder.cpp:159-174) plus
    recompute_kv_from_activation (decoder.cpp:123-129) of a `chunk`-row slice
    of the request's ACT rows, scaled to its n_act ACT tokens (the reference
    GEMM is row-parallel, matrix.cpp:28, so its cost is linear in rows).
    run() returns seconds per request-layer; a step of B requests x L layers
    costs B x L of them, so tokens/s = 1 / (L x run()). Vocabulary 16 (the
    reference has no LM head; the embedding table does not enter the
    per-layer cost)."""
    os.environ["OMP_NUM_THREADS"] = str(threads)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref_lib as R  # noqa: E402  (checker / baseline only)
    d, H, f, tpb = dims.hidden_dim, dims.num_heads, dims.ffn_dim, dims.tokens_per_block
    rng = np.random.default_rng(0)
    ck = rng.uniform(-0.1, 0.1, (1, ctx, d))
    cv = rng.uniform(-0.1, 0.1, (1, ctx, d))
    a = rng.uniform(-0.1, 0.1, (chunk, d))
    if R.available():
        kind = "reference"
        threads = R.set_threads(threads)  # torchrun exports OMP_NUM_THREADS=1 before libgomp loads
        rw = R.RefWeights(1, d, H, f, 16, tpb, 42, ctx + 2)

        def run():
            t0 = time.perf_counter()
            rw.generation_step(1, ctx, ck, cv)
            t1 = time.perf_counter()
            if n_act:
                rw.recompute_kv(0, a)
            t2 = time.perf_counter()
            return (t1 - t0) + (t2 - t1) * n_act / chunk
    else:
        import hybridsim_oracle as O  # noqa: E402
        kind = "port"
        wl = {n: rng.uniform(-0.1, 0.1, sh) for n, sh in zip(O.WEIGHT_NAMES, [(d, d)] * 4 + [(d, f), (f, d)])}
        w = O.DecoderWeights(O.ModelConfig(num_layers=1, hidden_dim=d, num_heads=H, ffn_dim=f,
                                           vocab_size=16).validate(), ctx + 2,
                             rng.uniform(-0.1, 0.1, (16, d)), rng.uniform(-0.1, 0.1, (ctx + 2, d)), [wl])

        def run():
            t0 = time.perf_counter()
            O.generation_step(1, ctx, [ck[0]], [cv[0]], w)
            t1 = time.perf_counter()
            if n_act:
                O.recompute_kv_from_activation(a, 0, w)
            t2 = time.perf_counter()
            return (t1 - t0) + (t2 - t1) * n_act / chunk

    sample = (f"1 request x 1 layer of one decode step at {dims.name} width (d={d}): generation_step over context "
              f"{ctx} + recompute_kv_from_activation of {chunk} of its {n_act} ACT rows (scaled linearly); x "
              f"{dims.num_layers} layers per token")
    return kind, run, sample, threads, R if kind == "reference" else None


def single_thread_leg(dims, ctx, n_act, reps=2):
    """The same sample with OMP_NUM_THREADS=1."""
    kind, run, sample, _, R = cpu_reference_sample(dims, ctx, n_act, 1)
    run()
    t = statistics.mean([run() for _ in range(reps)])
    return {"value": 1.0 / (dims.num_layers * t), "unit": "tokens/s", "cores": 1, "kind": kind, "steps": reps}


def reference_arm(args, world, rank, dist):
    """The reference's CPU path on this host: never imports the product."""
    if rank != 0:
        return
    dims = reference_dims(args.model)
    if args.layers:
        dims.num_layers = args.layers
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref_lib as R  # noqa: E402
    B = per_rank_batch(args, world, 0)
    bp = bundle_path(args)
    if args.ratio >= 0:
        r, src = args.ratio, "--ratio"
    elif bp and R.available():
        r, factor, _ = planned_ratio(R.parse_bundle(bp), dims, B * (args.prompt + args.gen), R.plan_host_allocation)
        src = (f"planner: the reference's plan_host_allocation (plan.cpp:106-152) on the B200-measured bundle "
               f"{os.path.relpath(bp, ROOT)}, workload-sized m_host (x{factor})")
    else:
        r, src = 1.0 / 3.0, "the paper's KV:ACT 2:1 (PAPER.md:714): no committed bundle"
    ctx = args.prompt + args.gen // 2
    n_act = int(round(r * ctx))
    threads = os.cpu_count() or 1
    kind, run, sample, threads, _ = cpu_reference_sample(dims, ctx, n_act, threads)
    for _ in range(args.warmup):
        run()
    ts = [run() for _ in range(args.steps)]
    t = statistics.mean(ts)
    v = 1.0 / (dims.num_layers * t)
    st = single_thread_leg(dims, ctx, n_act)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": B * dims.num_layers * t * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, dims, world, r, src, ctx),
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": threads, "kind": kind, "sample": sample,
                         "single_thread": st},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


class Dims:
    """Model dimensions without importing the product (the reference arm must
    not load libhybridcache_b200.so)."""

    def __init__(self, name, layers, d, heads, ffn, vocab, tpb):
        self.name, self.num_layers, self.hidden_dim, self.num_heads = name, layers, d, heads
        self.ffn_dim, self.vocab_size, self.tokens_per_block = ffn, vocab, tpb


def reference_dims(model):
    """ModelConfig::preset (model.cpp:37-43) through the reference library,
    else the oracle's restatement."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref_lib as R  # noqa: E402  (reference arm / baseline only)
    if R.available():
        return Dims(model, *R.model_preset(model))
    import hybridsim_oracle as O  # noqa: E402
    c = O.preset(model)
    return Dims(model, c.num_layers, c.hidden_dim, c.num_heads, c.ffn_dim, c.vocab_size, c.tokens_per_block)


def bundle_path(args):
    if args.bundle == "live":
        return None
    if args.bundle == "committed":
        p = os.path.join(ROOT, "profiles", f"planner_bundle_{args.model}.json")
        return p if os.path.exists(p) else None
    return args.bundle


def read_bundle(path):
    """bundle.json (timing.cpp:147-153) -> (kv slope, kv icept, load slope, load icept, t_load_w, s_w_layer, s_w_total)."""
    with open(path) as fh:
        j = json.load(fh)
    return (j["kv_gen"]["slope"], j["kv_gen"]["intercept"], j["load_kv"]["slope"], j["load_kv"]["intercept"],
            j["t_load_w"], float(j["s_weight_layer"]), float(j["s_weight_total"]))


def planned_ratio(b7, dims, workload_tokens, plan_fn):
    """plan_host_allocation (plan.cpp:106-152) over a WORKLOAD-sized host
    budget, as the reference's interior-balance test sizes it
    (test_sim.cpp:281-282: m_host = s_weight + 0.9 x workload blocks x
    s_kv_block; widened only when Alg. 1 raises CapacityError). plan_fn(b5,
    mem4, tpb, act_gpu) -> (act_host, kv_host, ...) is the reference's planner
    in the reference arm and the product's (bit-exact) in ours, so both arms
    derive the same r from the same bundle."""
    L, d, tpb = dims.num_layers, dims.hidden_dim, dims.tokens_per_block
    s_kv, s_act = float(tpb * 2 * d * 2) * L, float(tpb * d * 2) * L  # bytes_of x L (plan.cpp:46-49)
    blocks = workload_tokens / tpb
    err = None
    for factor in (0.9, 1.5, 3.0, 6.0, 12.0):
        mem = [b7[6] + blocks * s_kv * factor, b7[6], s_kv, s_act]
        try:
            a = plan_fn(list(b7[:5]), mem, tpb, 0)
            return a[0] / max(a[0] + a[1], 1), factor, list(a)
        except Exception as e:  # CapacityError (plan.cpp:79) in either library
            err = e
    raise err


def bench_config(args, dims, world, r, ratio_source, timed_ctx):
    """The `config` object, built identically by both arms (same workload,
    same r, same timed context)."""
    B = per_rank_batch(args, world, 0)
    gb = args.global_batch or B * world
    return {"workload": f"BASELINE configs[{args.config - 1}]: {dims.name}-shape offloaded decode (weights + hybrid "
                        f"KV/ACT cache in pinned host memory), " +
                        (f"global batch {gb} split over {world} GPU(s)" if args.global_batch else f"batch {B}/GPU") +
                        f", prompt {args.prompt}, gen {args.gen}",
            "model": dims.name, "global_batch": gb, "batch_per_gpu": B, "seq_len": args.prompt, "gen_len": args.gen,
            "act_share_r": round(r, 6),
            "kv_act_ratio": (f"{(1 - r) / r:.3f}:1" if 0 < r < 1 else ("kv_only" if r <= 0 else "act_only")),
            "ratio_source": ratio_source, "timed_context": timed_ctx,
            "timed_context_note": "decode steps timed at the generation's mean context P + G/2",
            "parallelism": f"batch-partitioned x{world} (no collective)", "arch": args.arch,
            "l2": "inputs larger than L2 (~100+ GB streamed host->HBM per step)"}


# ------------------------------------------------------------------ ours ---
def pool_plan(cfg, B, P, steps, r):
    """Block pools and ratio setting for B requests of up to P+steps tokens
    at ACT share r (r=0 kv_only, r=1 act_only, else hybrid via next_block_kind)."""
    from paper_2501_01792_b200 import api
    tpb = cfg.tokens_per_block
    nb = math.ceil((P + steps) / tpb)
    mode = "kv_only" if r <= 0 else ("act_only" if r >= 1 else "hybrid")
    act_per = 0 if mode == "kv_only" else (nb if mode == "act_only" else math.ceil(r * nb) + 1)
    kv_per = 0 if mode == "act_only" else (nb if mode == "kv_only" else math.ceil((1 - r) * nb) + 1)
    a = int(round(r * 1000))
    return mode, api.HostAllocation(a, 1000 - a), api.PoolCaps(kv_host=B * kv_per, act_host=B * act_per)


def host_layers_for(cfg, caps, budget, w_bytes_pinned, tpn=1):
    from paper_2501_01792_b200 import api
    per_layer = (caps.kv_host * api.HybridCache.bytes_of("KV", cfg) +
                 caps.act_host * api.HybridCache.bytes_of("ACT", cfg)) / tpn  # a TP rank holds 1/N of both
    if per_layer == 0:
        return cfg.num_layers
    return int(min(cfg.num_layers, max(2, (budget - w_bytes_pinned) // per_layer)))


def run_steps(eng, ids, tokens, t0, n, prof=False):
    """n decode steps starting at token row t0; returns summed stats."""
    out = {"argmax": np.zeros(len(ids), np.int32)}
    acc = {"dev_ms": 0.0, "launches": 0, "h2d": 0.0, "d2h": 0.0, "wall": 0.0}
    eng.set_profile(prof)
    last = None
    for s in range(n):
        w0 = time.perf_counter()
        eng.decode_step(ids, tokens[t0 + s], want_x=False, want_argmax=True, out=out)
        acc["wall"] += time.perf_counter() - w0
        st = eng.last_stats()
        acc["dev_ms"] += st["step_ms"]
        acc["launches"] += int(st["launches"])
        acc["h2d"] += st["h2d_bytes"]
        acc["d2h"] += st["d2h_bytes"]
        last = st
    eng.set_profile(False)
    acc["last"] = last
    return acc


def act_context_tokens(eng, ids):
    return sum(e.filled_tokens for rid in ids for e in eng.cache.table(rid).entries if int(e.kind) == 1)


def variant(eng, cfg, ids, tokens, P, r, caps_mode_alloc, host_layers, steps, warmup, link_gbs, seed, act_gpu=0,
            token_recompute=None):
    """Re-configure the pools for one KV:ACT ratio and time `steps` decode steps."""
    from paper_2501_01792_b200 import api
    mode, alloc, caps = caps_mode_alloc
    if act_gpu:
        caps = api.PoolCaps(kv_host=caps.kv_host, act_host=caps.act_host, act_gpu=act_gpu)
    rc_ratio = 0.0
    if token_recompute is not None:  # SimMode::TokenRecompute baseline on the KV-only pools
        mode, rc_ratio = "token_recompute", token_recompute
    eng.configure_cache(caps, mode=mode, allocation=alloc, host_layers=host_layers, recompute_ratio=rc_ratio)
    eng.admit_synthetic(ids, [P] * len(ids), seed=seed)
    run_steps(eng, ids, tokens, 0, warmup)
    acc = run_steps(eng, ids, tokens, warmup, steps)
    ms = acc["dev_ms"] / steps
    B = len(ids)
    return {"act_share_r": round(r, 4), "mode": mode, "recompute_ratio": rc_ratio, "act_gpu_blocks": act_gpu,
            "tokens_per_s": B * 1e3 / ms,
            "ms_per_step": ms, "h2d_gb_per_step": acc["h2d"] / steps / 1e9,
            "link_frac": (acc["h2d"] / steps / (link_gbs * 1e9)) / (ms / 1e3) if link_gbs else None,
            "e2e_tokens_per_s": B * steps / acc["wall"], "steps": steps,
            "act_context_tokens": act_context_tokens(eng, ids)}


def _np_default(o):
    return o.item() if hasattr(o, "item") else str(o)


def write_artifacts(out_dir, eng, cfg, ids, planner, prof, mode, r, prefill=None):
    """The reference CLI's artifacts from MEASURED B200 data, in its schemas
    (main.cpp:75-115, 146-166, 255-275; timing.cpp:147-153; plan.cpp:22-28):
    the unmodified `hybridsim plan --bundle` / `simulate --plan` can consume them."""
    from paper_2501_01792_b200 import api
    os.makedirs(out_dir, exist_ok=True)
    meta = {"version": "b200-measured", "seed": 42, "inputs": {}}
    cfgj = {"name": cfg.name, "num_layers": cfg.num_layers, "hidden_dim": cfg.hidden_dim,
            "num_heads": cfg.num_heads, "ffn_dim": cfg.ffn_dim, "vocab_size": cfg.vocab_size,
            "tokens_per_block": cfg.tokens_per_block, "bytes_per_scalar": cfg.bytes_per_scalar, "seed": 0}
    if planner and "kv_gen_samples" in planner:
        for name, key in (("kv_gen.csv", "kv_gen_samples"), ("load_kv.csv", "load_kv_samples")):
            with open(os.path.join(out_dir, name), "w") as fh:
                fh.write("n_tokens,seconds\n" + "".join(f"{n:.0f},{s:.9e}\n" for n, s in planner[key]))
        per, total = api.weight_bytes(cfg)
        bundle = {"kv_gen": {"slope": planner["t_kv_gen"]["slope_s_per_token"],
                             "intercept": planner["t_kv_gen"]["intercept_s"], "r2": planner["t_kv_gen"]["r2"],
                             "intercept_clamped": planner["t_kv_gen"]["intercept_s"] == 0.0},
                  "load_kv": {"slope": planner["t_load_kv"]["slope_s_per_token"],
                              "intercept": planner["t_load_kv"]["intercept_s"], "r2": planner["t_load_kv"]["r2"],
                              "intercept_clamped": planner["t_load_kv"]["intercept_s"] == 0.0},
                  "t_load_w": planner["t_load_w_s"], "s_weight_layer": per, "s_weight_total": total,
                  "model": cfgj, "meta": meta}
        with open(os.path.join(out_dir, "bundle.json"), "w") as fh:
            json.dump(bundle, fh, indent=2, default=_np_default)
        plan = dict(planner["allocation"])
        plan["predicted"] = {"t_pcie": planner["planned_t_pcie_s"], "t_computation": planner["planned_t_comp_s"]}
        plan["meta"] = meta
        with open(os.path.join(out_dir, "plan.json"), "w") as fh:
            json.dump(plan, fh, indent=2, default=_np_default)
    L = cfg.num_layers
    kvb, actb = api.HybridCache.bytes_of("KV", cfg), api.HybridCache.bytes_of("ACT", cfg)
    kv_blocks = act_host_blocks = 0
    for rid in ids:
        for e in eng.cache.table(rid).entries:
            if int(e.kind) == 0 and int(e.location) == 0:
                kv_blocks += 1
            elif int(e.kind) == 1 and int(e.location) == 0:
                act_host_blocks += 1
    w_layer, _ = api.weight_bytes(cfg)
    step_s = prof["step_ms"] / 1e3
    busy = (prof["recompute_ms"] + prof["attn_ms"] + prof["gemm_ms"]) / prof["step_ms"]
    metrics = {"tokens_generated": len(ids), "makespan_s": step_s, "throughput_tok_s": len(ids) / step_s,
               "pcie_busy": prof["copy_ms"] / prof["step_ms"], "gpu_busy": min(busy, 1.0),
               "prefill_s": prefill["prefill_s"] if prefill else 0.0, "gen_s": step_s,
               "traffic": {"weights": w_layer * L, "kv_load": kv_blocks * kvb * L, "act_load": act_host_blocks * actb * L,
                           # the new token's cache rows, stored by mapped writes from the append kernels
                           "kv_store": prof["d2h_kv"], "act_store": prof["d2h_act"]},
               "mode": mode, "act_share_r": r, "batch": len(ids),
               "measured_on": "B200: one profiled decode step at the mean context (prefill_s: the measured prefill "
                              "of the same run, not part of makespan_s; the whole generation is "
                              "metrics_full_generation.json)",
               "meta": meta}
    with open(os.path.join(out_dir, "metrics.json"), "w") as fh:
        json.dump(metrics, fh, indent=2, default=_np_default)
    tr = eng.trace()
    tr["meta"] = meta
    with open(os.path.join(out_dir, "trace.json"), "w") as fh:
        json.dump(tr, fh, default=_np_default)


def run_prefill(eng, cfg, ids, P, rank, tflops_sust, link_gbs):
    """Offloaded prefill of len(ids) random prompts of P tokens (one profiled
    call): time, tensor FLOPs (flops.cpp:16-22: QKV + causal attention +
    proj/FFN per layer), bytes streamed in (weights) and stored out (blocks)."""
    import torch
    d, f, L, H = cfg.hidden_dim, cfg.ffn_dim, cfg.num_layers, cfg.num_heads
    rng = np.random.default_rng(100 + rank)
    prompts = [rng.integers(0, cfg.vocab_size, P).tolist() for _ in ids]
    torch.cuda.synchronize()
    eng.set_profile(True)
    w0 = time.perf_counter()
    eng.prefill(ids, prompts)
    wall = time.perf_counter() - w0
    eng.set_profile(False)
    st = eng.last_stats()
    n = len(ids)
    gemm_flops = L * 2.0 * n * P * (4 * d * d + 2 * d * f)
    attn_flops = L * n * 2.0 * d * P * (P + 1)  # attention_causal FLOPs (flops.cpp:19)
    s = st["step_ms"] / 1e3
    return {"requests": n, "prompt": P, "prefill_s": s, "wall_s": wall, "prompt_tokens_per_s": n * P / s,
            "gemm_tflops": gemm_flops / (st["gemm_ms"] / 1e3) / 1e12 if st["gemm_ms"] else None,
            "attention_tflops": attn_flops / (st["attn_ms"] / 1e3) / 1e12 if st["attn_ms"] else None,
            "split_ms": {"qkv_proj_ffn_gemms": st["gemm_ms"], "causal_attention": st["attn_ms"],
                         "weight_h2d_stream": st["copy_ms"], "block_d2h_stream": st["store_ms"]},
            "h2d_gb": st["h2d_bytes"] / 1e9, "d2h_gb": st["d2h_bytes"] / 1e9,
            "d2h_gbs": st["d2h_bytes"] / (st["store_ms"] / 1e3) / 1e9 if st["store_ms"] else None,
            "tensor_roofline_s": (gemm_flops + attn_flops) / (tflops_sust * 1e12),
            "link_roofline_s": max(st["h2d_bytes"], st["d2h_bytes"]) / (link_gbs * 1e9) if link_gbs else None,
            "launches": int(st["launches"])}


def calibrate_planner(eng, cfg, link_gbs, caps_act_rows, workload_tokens, act_gpu=0, tpn=1, wsn=1, caps_kv_blocks=0):
    """North-star (5): measured recompute-GEMM and host-link samples ->
    bundle_from_samples (timing.cpp:172-183) -> plan_host_allocation
    (plan.cpp:106-152) over a WORKLOAD-sized host budget, as the reference's
    own interior-balance test sizes it (test_sim.cpp:281-282: m_host =
    s_weight + 0.9 x workload blocks x s_kv_block) — the whole-DRAM budget
    (plan.cpp:41-51) cannot even hold OPT-66B's weights plus the initial ACT
    blocks on a 196 GB host (CapacityError, plan.cpp:79)."""
    from paper_2501_01792_b200 import api
    ns = [n for n in (4096, 16384, 32768, 65536) if n <= caps_act_rows]
    if len(ns) < 2:  # small per-rank batches (config 4 split 8 ways): smaller samples, still >= 2
        ns = [n for n in (512, 1024, 2048, 4096, 8192) if n <= caps_act_rows][-3:]
    kv = [(float(n), eng.time_kv_gen(n, reps=3)) for n in ns]
    # link samples: KV-token byte counts the pinned pools and a staging slot hold
    kv_tok = 2 * cfg.hidden_dim * 2 // tpn
    room = max(caps_kv_blocks * api.HybridCache.bytes_of("KV", cfg), caps_act_rows * cfg.hidden_dim * 2)
    ln = [n for n in (4096, 16384, 32768, 65536) if n * kv_tok <= room] or [n for n in (256, 1024, 2048)]
    ld = [(float(n), eng.time_load_kv(n, reps=2)) for n in ln]
    bundle = api.bundle_from_samples(kv, ld, link_gbs * 1e9, cfg)
    if tpn > 1:  # a head-sharded rank streams and stores 1/N of every weight and block
        bundle.t_load_w /= tpn
        bundle.s_weight_layer //= tpn
        bundle.s_weight_total //= tpn
    if wsn > 1:  # ranks sharing the weight stream: each link carries 1/N of every layer
        bundle.t_load_w /= wsn
    mem = api.budget_for(0.0, cfg, bundle)
    if tpn > 1:
        mem.s_kv_block /= tpn
        mem.s_act_block /= tpn
    workload_blocks = workload_tokens / cfg.tokens_per_block
    # small per-rank batches next to large weights (config 4 split 4-8 ways): the
    # initial balanced blocks may not fit 0.9 x the workload (CapacityError,
    # plan.cpp:79) — widen the budget until Alg. 1 has room, and say so
    for factor in (0.9, 1.5, 3.0, 6.0, 12.0):
        mem.m_host = mem.s_weight + workload_blocks * mem.s_kv_block * factor
        try:
            alloc = api.plan_host_allocation(bundle, mem, cfg.tokens_per_block, act_gpu)
            break
        except api.CapacityError:
            if factor == 12.0:
                raise
    r = alloc.act_host / max(alloc.act_host + alloc.kv_host, 1)
    return {"kv_gen_samples": kv, "load_kv_samples": ld,
            "t_kv_gen": {"slope_s_per_token": bundle.t_kv_gen.slope, "intercept_s": bundle.t_kv_gen.intercept,
                         "r2": bundle.t_kv_gen.r_squared},
            "t_load_kv": {"slope_s_per_token": bundle.t_load_kv.slope, "intercept_s": bundle.t_load_kv.intercept,
                          "r2": bundle.t_load_kv.r_squared},
            "t_load_w_s": bundle.t_load_w, "m_host": mem.m_host,
            "m_host_source": f"workload-sized: s_weight + {factor} x B(P+G)/tpb x s_kv_block (test_sim.cpp:281-282 "
                             "uses 0.9; widened only when Alg. 1 raises CapacityError)",
            "allocation": alloc.__dict__, "planned_r": r,
            "planned_t_pcie_s": api.planned_t_pcie(bundle, cfg.tokens_per_block, alloc),
            "planned_t_comp_s": api.planned_t_computation(bundle, cfg.tokens_per_block, alloc, act_gpu)}


def tp_group(args, world, rank, local, dist):
    """--tp N: NCCL group over the torchrun ranks (ids from rank 0, broadcast
    over torch.distributed); --tp-emulate N: one rank's timing stand-in."""
    from paper_2501_01792_b200 import api
    if args.tp > 1:
        if world != args.tp:
            raise SystemExit("--tp N needs exactly N torchrun ranks")
        obj = [api.TensorParallel.nccl_unique_ids() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return api.TensorParallel.nccl(obj[0], rank, world, local), args.tp
    if args.tp_emulate > 1:
        return api.TensorParallel.emulated(0, args.tp_emulate), args.tp_emulate
    return None, 1


def weight_share_group(args, world, rank, local, dist):
    """Batch-partitioned ranks sharing one weight stream (Engine(weight_share=)):
    an NCCL group over the torchrun ranks when every rank has its own GPU
    (NVLink all-gather); --share-emulate N: one rank's timing stand-in."""
    from paper_2501_01792_b200 import api
    if args.share_emulate > 1:
        return api.TensorParallel.emulated(0, args.share_emulate), args.share_emulate
    if world > 1 and args.share_weights and args.tp <= 1:
        import torch
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        if torch.cuda.device_count() < local_world or local_world != world:
            return None, 1  # ranks share a GPU (plumbing smoke test) or span nodes: whole-layer streams
        obj = [api.TensorParallel.nccl_unique_ids() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return api.TensorParallel.nccl(obj[0], rank, world, local), world
    return None, 1


def our_arm(args, cfg, world, rank, local, dist):
    from paper_2501_01792_b200 import api, kernels
    if kernels.device_count() == 0:
        raise SystemExit("bench needs a CUDA device")
    hbm_peak, tflops_sust, tflops_burst, peak_src = measured_peaks()
    numa_node = bind_numa(local)
    tp, tpn = tp_group(args, world, rank, local, dist)
    ws, wsn = weight_share_group(args, world, rank, local, dist) if tp is None else (None, 1)
    if args.share_emulate > 1:
        args.no_sweep = True
    if tp is not None:  # heads are sharded, requests are not: every rank serves the global batch
        args.no_sweep = True
        B = args.global_batch or args.batch or 128
    else:
        B = per_rank_batch(args, world, rank)
    P, L, d = args.prompt, cfg.num_layers, cfg.hidden_dim
    total_steps = args.warmup + args.steps + 2
    # the timed steps sit at the generation's mean context P + G/2: after the
    # real prefill of P tokens, each request is grown by n_adv tokens through
    # the allocator in decode order (the block tables G/2 real steps would
    # leave; slots pattern-filled), then warm-up, one profiled step, K timed
    ctx_mid = P + args.gen // 2
    c0 = ctx_mid - (args.steps - 1) // 2  # context before the first timed step
    n_adv = max(0, c0 - (args.warmup + 1) - P)
    span = P + n_adv + total_steps  # tokens per request the pools must hold
    max_seq = max(span, P + args.gen + 4) + 1
    # planner ratio (north-star (5)): paper Alg. 1 on a B200-measured timing
    # bundle — by default the committed one both arms read (same r), the
    # live calibration below is reported beside it
    bp = bundle_path(args)
    if args.ratio >= 0:
        r, r_src = args.ratio, "--ratio"
    elif bp:
        r, factor, _ = planned_ratio(read_bundle(bp), cfg, B * (P + args.gen),
                                     lambda b5, m4, tpb, ag: list(api.plan_host_allocation(
                                         api.TimingBundle(api.LinearTimeModel(b5[0], b5[1]),
                                                          api.LinearTimeModel(b5[2], b5[3]), b5[4]),
                                         api.MemoryBudget(*m4), tpb, ag).__dict__.values()))
        r_src = (f"planner: the reference's plan_host_allocation (plan.cpp:106-152) on the B200-measured bundle "
                 f"{os.path.relpath(bp, ROOT)}, workload-sized m_host (x{factor})")
    else:
        r, r_src = 1.0 / 3.0, "live"  # replaced by the live planner below
    mode, alloc, caps = pool_plan(cfg, B, span, 0, r)
    w_layer, _ = api.weight_bytes(cfg)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    # pinned host budget: what the node has available minus a 40 GB reserve
    # for the OS and this process, split over the node's ranks (pinned pages
    # cannot be reclaimed; folding keeps the streamed bytes)
    budget = args.host_gb * 1e9 if args.host_gb > 0 else max(16e9, mem_available_bytes() - 40e9) / local_world
    w_rank = w_layer / tpn  # pinned weight bytes per layer on this rank
    Lw = L if L * w_rank <= 0.55 * budget else max(2, int(0.55 * budget // w_rank))
    Lp = host_layers_for(cfg, caps, budget, Lw * w_rank, tpn)
    t_setup = time.time()
    eng = api.Engine(cfg, seed=42, max_seq=max_seq, rescale=True, max_batch=B, weights_on_device=False,
                     caps=caps, host_layers=Lp, weight_layers=Lw, mode=mode, allocation=alloc, device=local,
                     arch=args.arch, tp=tp, weight_share=ws)
    ids = [f"g{0 if tp else rank}r{i}" for i in range(B)]
    # host-link peak: a large pinned H2D copy on the engine's copy stream, all
    # ranks copying at once (ranks share PCIe switches)
    tpb = cfg.tokens_per_block
    n_tok = min(max(caps.kv_host * tpb, caps.act_host * tpb // 2), 65536)
    barrier(dist)
    # (best of 3 trials of 4 back-to-back copies: the copy engine's sustained peak)
    link_gbs = (n_tok * 2 * (d // tpn) * 2) / min(eng.time_load_kv(n_tok, reps=4) for _ in range(3)) / 1e9 \
        if n_tok else None
    barrier(dist)
    # live calibration (north-star (5)): measured recompute-GEMM and link samples
    planner = None
    if link_gbs and caps.act_host:
        try:
            planner = calibrate_planner(eng, cfg, link_gbs, caps.act_host * tpb, B * (P + args.gen), tpn=tpn,
                                        wsn=wsn, caps_kv_blocks=caps.kv_host)
        except Exception as e:  # planner failure must not kill the bench line
            planner = {"error": str(e)}
    if r_src == "live" and planner and "planned_r" in planner:
        r = planner["planned_r"]
        r_src = "planner: plan_host_allocation (plan.cpp:106-152) on this run's live calibration"
        mode, alloc, caps = pool_plan(cfg, B, span, 0, r)
        Lp = host_layers_for(cfg, caps, budget, Lw * w_rank, tpn)
        eng.configure_cache(caps, mode=mode, allocation=alloc, host_layers=Lp)
    setup_s = time.time() - t_setup
    # the cache the decode steps read is built by the real offloaded prefill
    # of B synthetic prompts (weights streamed once per layer, host blocks
    # stored by D2H runs) — measured, and reported as its own stage
    if args.prefill == "real":
        eng.fill_pools(seed=1 + rank)  # slots handed out by advance_synthetic hold finite values
        prefill = run_prefill(eng, cfg, ids, P, rank, tflops_sust, link_gbs)
    else:
        prefill = None
        eng.admit_synthetic(ids, [P] * B, seed=1 + rank)
    eng.advance_synthetic(ids, n_adv)

    rng = np.random.default_rng(rank)
    tokens = rng.integers(0, cfg.vocab_size, (total_steps, B)).astype(np.int32)
    run_steps(eng, ids, tokens, 0, args.warmup)
    # one profiled (untimed) step: per-kernel split + copy-stream GB/s
    prof = run_steps(eng, ids, tokens, args.warmup, 1, prof=True)["last"]
    act_tokens = act_context_tokens(eng, ids)
    if args.artifacts and rank == 0:
        write_artifacts(args.artifacts, eng, cfg, ids, planner, prof, mode, r, prefill)

    clocks = ClockSampler(local)
    barrier(dist)
    import torch
    torch.cuda.synchronize()
    clocks.start()
    acc = run_steps(eng, ids, tokens, args.warmup + 1, args.steps)
    torch.cuda.synchronize()
    barrier(dist)
    clk = clocks.stop()

    dev_s = max_over_ranks(dist, acc["dev_ms"] / 1e3)
    wall_s = max_over_ranks(dist, acc["wall"])
    # TP ranks produce the same tokens (heads are sharded); batch-partitioned ranks add up
    tokens_total = float(B * args.steps) if tp is not None else sum_over_ranks(dist, float(B * args.steps))
    value = tokens_total / dev_s
    e2e = tokens_total / wall_s
    ms_per_step = dev_s * 1e3 / args.steps
    h2d_step = acc["h2d"] / args.steps

    # dominant kernel: the recompute GEMM (tcgen05). algorithmic FLOPs/launch
    # = 4 d^2 x ACT context tokens of the layer (flops.cpp:14)
    rec_launch_ms = prof["recompute_ms"] / max(prof["recompute_launches"], 1)
    rec_flops = 4.0 * d * d * act_tokens / max(prof["recompute_launches"] / L, 1)
    rec_rows = act_tokens / max(prof["recompute_launches"] / L, 1)  # ACT rows per launch
    achieved = rec_flops / (rec_launch_ms / 1e3) / 1e12 if rec_launch_ms > 0 else 0.0
    fused = eng.fused_recompute()
    if fused:  # recompute fused with the attention: partial records instead of K|V
        rec_kernel = "gemm_tn_kernel<256,kAttnPart> (ACT->K|V recompute fused with decode attention)"
        rec_alg = rec_rows * d * 2 + 2 * d * d * 2 + rec_rows / tpb * cfg.num_heads * (cfg.head_dim + 4) * 4
        rec_alg_note = "A + [Wk|Wv] read once, one partial record per block and head written"
    else:
        rec_kernel = "gemm_tn_kernel<256,kKvPaged> (ACT->K|V recompute)"
        rec_alg = rec_rows * (3 * d * 2) + 2 * d * d * 2
        rec_alg_note = "A + [Wk|Wv] read once, K|V written once"
    roof = {"kernel": rec_kernel, "bound": "tensor",
            "achieved": achieved, "peak": tflops_sust, "unit": "TFLOP/s",
            "frac": achieved / tflops_sust if tflops_sust else None,
            "traffic": rec_rows * (RECOMPUTE_NCU_BYTES_PER_ROW_FUSED if fused else RECOMPUTE_NCU_BYTES_PER_ROW),
            "traffic_note": (f"ncu dram__bytes_read+write per launch scaled by ACT rows ({RECOMPUTE_NCU_NOTE}); "
                             f"algorithmic {rec_alg:.3e} B ({rec_alg_note}). DESIGN.md §3"),
            "peak_source": f"{peak_src} bf16_tflops_sustained (MEASURED_PEAKS.json); burst {tflops_burst}",
            "frac_vs_burst": achieved / tflops_burst if tflops_burst else None,
            "frac_note": ("the kernel is timed inside a long step, so the peak is the sustained figure (cuBLAS "
                          "back to back for 4 s); a launch between copy-stream waits can run cooler than that "
                          "and exceed it (frac > 1) — frac_vs_burst is the single-launch bound"),
            "flops_per_launch": rec_flops, "launch_ms": rec_launch_ms}
    # per-step roofline (north_star): slower of link bytes / link BW, tensor
    # FLOPs / tensor peak, HBM bytes / HBM BW
    ctx = c0 + (args.steps - 1) / 2.0
    # (a head-sharded rank does 1/N of the FLOPs and HBM traffic)
    tensor_flops = L * (4.0 * d * d * act_tokens + 2.0 * B * (4 * d * d + 2 * d * cfg.ffn_dim)) / tpn
    # HBM: KV-cached context read by the attention, ACT rows read by the recompute (+ K|V written
    # and read back unless the recompute is fused with the attention), the layer weights
    kv_ctx_tokens = max(B * (ctx + 1) - act_tokens, 0.0)
    hbm_bytes = L * (kv_ctx_tokens * 2 * d * 2 + act_tokens * (d * 2 if fused else 5 * d * 2) + w_layer) / tpn \
        + h2d_step
    t_link = h2d_step / (link_gbs * 1e9) if link_gbs else 0.0
    t_tensor = tensor_flops / (tflops_sust * 1e12)
    t_hbm = hbm_bytes / (hbm_peak * 1e9)
    t_roof = max(t_link, t_tensor, t_hbm)
    step_roof = {"t_link_ms": t_link * 1e3, "t_tensor_ms": t_tensor * 1e3, "t_hbm_ms": t_hbm * 1e3,
                 "bound": ["link", "tensor", "hbm"][int(np.argmax([t_link, t_tensor, t_hbm]))],
                 "roofline_tokens_per_s_per_gpu": B / t_roof if t_roof else None,
                 "frac": (t_roof * 1e3) / ms_per_step if ms_per_step else None,
                 "link_peak_gbs": link_gbs, "link_peak_source": "measured: pinned H2D cudaMemcpyAsync on this box",
                 # the same step against independent link ceilings: the standalone probe's best
                 # (1-4 copy streams, 8-256 MB chunks, SM zero-copy; profiles/r01_link_probe.json)
                 # and PCIe Gen5 x16's nominal 64 GB/s per direction
                 "frac_vs_probe_ceiling": (h2d_step / (LINK_PROBE_GBS * 1e9)) / (ms_per_step / 1e3),
                 "frac_vs_pcie5_nominal": (h2d_step / 64e9) / (ms_per_step / 1e3),
                 "achieved_link_gbs": h2d_step / (ms_per_step / 1e3) / 1e9,
                 "copy_stream_gbs": prof["h2d_bytes"] / (prof["copy_ms"] / 1e3) / 1e9 if prof["copy_ms"] else None,
                 "profile_split_ms": {"recompute": prof["recompute_ms"], "attention": prof["attn_ms"],
                                      "qkv_proj_ffn": prof["gemm_ms"], "copy_stream": prof["copy_ms"]}}

    # whole-generation throughput (prefill + G decode steps, the paper's and
    # the sim's definition, sim.cpp:618-628): prefill measured above; decode
    # steps at context P+g projected from the measured step by streamed bytes
    # (the step is link-bound: step_roofline.bound == "link")
    gen = None
    if prefill is not None:
        dec_s = args.gen * ms_per_step / 1e3
        gen = {"prefill_s": prefill["prefill_s"], "step_ms_at_mean_context": ms_per_step, "decode_s": dec_s,
               "gen_len": args.gen, "tokens_per_s": B * args.gen / (prefill["prefill_s"] + dec_s),
               "tokens_per_s_all_ranks": B * args.gen * world / (prefill["prefill_s"] + dec_s),
               "prefill_share": prefill["prefill_s"] / (prefill["prefill_s"] + dec_s),
               "method": "prefill measured at P; G decode steps x the step measured at the mean context P + G/2 "
                         "(step time is linear in the context). The generation timed step by step: "
                         "bench.py --full-generation (profiles/r02_full_generation_opt30b.json)"}

    # ---- per-ratio sweep, planner, HBM-tiered variant (untimed by the contract)
    extra = {}
    if not args.no_sweep and world == 1:
        sweep_steps, sweep_warm = 2, 1
        sw_tokens = rng.integers(0, cfg.vocab_size, (sweep_steps + sweep_warm + 1, B)).astype(np.int32)
        # B200 extension: the host-only min-step planner (csrc/host/plan.hpp) on the same bundle,
        # Alg. 1's cost model plus the ACT blocks' own link time
        min_step, tbm, src_ms = None, None, None
        if bp:
            b7m = read_bundle(bp)
            tbm = api.TimingBundle(api.LinearTimeModel(b7m[0], b7m[1]), api.LinearTimeModel(b7m[2], b7m[3]), b7m[4])
            src_ms = os.path.relpath(bp, ROOT)
        elif planner and "t_kv_gen" in planner:  # no committed bundle for this model: this run's calibration
            tbm = api.TimingBundle(api.LinearTimeModel(planner["t_kv_gen"]["slope_s_per_token"],
                                                       planner["t_kv_gen"]["intercept_s"]),
                                   api.LinearTimeModel(planner["t_load_kv"]["slope_s_per_token"],
                                                       planner["t_load_kv"]["intercept_s"]), planner["t_load_w_s"])
            src_ms = "live calibration of this run"
        if tbm is not None:
            try:
                r_ms, caps_ms, (tc_ms, tl_ms) = api.plan_host_min_step(cfg, B, math.ceil(ctx_mid / cfg.tokens_per_block),
                                                                       tbm)
                min_step = {"r": r_ms, "predicted_t_comp_ms_per_layer": tc_ms * 1e3,
                            "predicted_t_link_ms_per_layer": tl_ms * 1e3, "bundle": src_ms,
                            "note": "plan_host_min_step: Alg. 1's cost model plus the ACT blocks' link time; "
                                    "min over r of max(t_link, t_comp) per layer"}
            except Exception as e:
                min_step = {"error": str(e)}
        rs = sorted(set(float(x) for x in args.sweep.split(",") if x and not x.startswith("tr")) | {r} |
                    ({planner["planned_r"]} if planner and "planned_r" in planner else set()) |
                    ({round(min_step["r"], 4)} if min_step and "r" in min_step else set()))
        per = []
        for tr in [float(x[2:]) for x in args.sweep.split(",") if x.startswith("tr")]:
            cm = pool_plan(cfg, B, ctx_mid, sweep_steps + sweep_warm + 1, 0.0)
            try:
                per.append(variant(eng, cfg, ids, sw_tokens, ctx_mid, 0.0, cm,
                                   host_layers_for(cfg, cm[2], budget, Lw * w_layer), sweep_steps, sweep_warm,
                                   link_gbs, 5, token_recompute=tr))
            except Exception as e:
                per.append({"token_recompute": tr, "error": str(e)})
        for rr in rs:
            if abs(rr - r) < 1e-6:
                per.append({"act_share_r": round(r, 4), "mode": mode, "act_gpu_blocks": 0, "tokens_per_s": value,
                            "ms_per_step": ms_per_step, "h2d_gb_per_step": h2d_step / 1e9,
                            "link_frac": step_roof["frac"], "e2e_tokens_per_s": e2e, "steps": args.steps,
                            "act_context_tokens": act_tokens, "headline": True})
                continue
            cm = pool_plan(cfg, B, ctx_mid, sweep_steps + sweep_warm + 1, rr)
            try:
                per.append(variant(eng, cfg, ids, sw_tokens, ctx_mid, rr, cm, host_layers_for(cfg, cm[2], budget, Lw * w_layer),
                                   sweep_steps, sweep_warm, link_gbs, 7 + len(per)))
            except Exception as e:
                per.append({"act_share_r": rr, "error": str(e)})
        extra["per_ratio"] = per
        if min_step and "r" in min_step:
            hit = [x for x in per if abs(x.get("act_share_r", -1) - round(min_step["r"], 4)) < 1e-4 and "tokens_per_s" in x]
            if hit:
                min_step["tokens_per_s"] = hit[0]["tokens_per_s"]
                min_step["vs_alg1"] = hit[0]["tokens_per_s"] / value
        extra["planner_min_step"] = min_step
        # B200 tiering: ACT blocks in HBM first (cache.cpp:85-91 placement),
        # sized to the free HBM; weights still streamed from pinned host memory
        try:
            cm = pool_plan(cfg, B, ctx_mid, sweep_steps + sweep_warm + 1, 1.0)
            free_b, _ = torch.cuda.mem_get_info(local)
            blk_all_layers = api.HybridCache.bytes_of("ACT", cfg) * L
            act_gpu = int(min(cm[2].act_host, 0.85 * (free_b - 8e9) // blk_all_layers))
            hv = variant(eng, cfg, ids, sw_tokens, ctx_mid, 1.0, cm, host_layers_for(cfg, cm[2], budget, Lw * w_layer),
                         sweep_steps, sweep_warm, link_gbs, 99, act_gpu=act_gpu)
            hv["note"] = ("ACT/gpu pool in HBM (ACT blocks placed on GPU first, cache.cpp:85-91); "
                          "weights + overflow blocks streamed from pinned host")
            extra["hbm_tiered"] = hv
        except Exception as e:
            extra["hbm_tiered"] = {"error": str(e)}

    ws_info = None
    if ws is not None:
        # per layer each rank receives the other ranks' (N-1)/N of the layer over
        # NVLink, on the gather stream (overlaps the copy stream's KV / ACT blocks)
        ag = (wsn - 1) / wsn * w_layer
        ws_info = {"size": wsn, "mode": "emulated" if args.share_emulate > 1 else "nccl",
                   "rank_h2d_gb_per_step": h2d_step / 1e9, "rank_weight_h2d_gb_per_step": L * w_layer / wsn / 1e9,
                   "nvlink_allgather_bytes_per_layer": ag}
        if args.share_emulate > 1:
            busbw = NVLINK_BUSBW
            t_ag = L * ag / busbw
            t_proj = max(ms_per_step / 1e3, t_ag + (ag / busbw))  # + one layer's gather exposed at the start
            ws_info.update({"note": "ONE of N batch-partitioned ranks timed on one GPU with 1/N of every weight "
                                    "layer streamed over its host link; the all-gather is skipped and NVLink time "
                                    "modelled at the measured NCCL bus bandwidth (own stream, overlapped)",
                            "rank_step_ms_measured": ms_per_step, "nvlink_allgather_ms_per_step": t_ag * 1e3,
                            "projected_step_ms": t_proj * 1e3, "projected_tokens_per_s_per_gpu": B / t_proj,
                            "projected_tokens_per_s_whole_job": wsn * B / t_proj})
    tp_info = None
    if tp is not None:
        # per layer: ACT all-gather (gather stream, overlaps the link and compute)
        # + two fp32 all-reduces of [B x d] (compute stream, serial)
        act_blk = api.HybridCache.bytes_of("ACT", cfg)
        cap_n = math.ceil(caps.act_host / tpn)
        ag_bytes = (tpn - 1) * cap_n * act_blk
        ar_bytes = 2 * (2.0 * (tpn - 1) / tpn) * B * d * 4
        tp_info = {"size": tpn, "mode": "nccl" if args.tp > 1 else "emulated",
                   "rank_h2d_gb_per_step": h2d_step / 1e9,
                   "allgather_bytes_per_layer": ag_bytes, "allreduce_bytes_per_layer": ar_bytes}
        if args.tp_emulate > 1:
            busbw = NVLINK_BUSBW
            t_ag, t_ar = L * ag_bytes / busbw, L * ar_bytes / busbw
            t_proj = max(ms_per_step / 1e3, t_ag) + t_ar
            tp_info.update({"note": "ONE rank of the N-way head-sharded group timed on one GPU: its weight / KV / "
                                    "ACT shards streamed, its heads computed, collectives skipped; NVLink time "
                                    "modelled at the measured NCCL bus bandwidth (gather overlapped on its "
                                    "own stream, all-reduces serial)",
                            "rank_step_ms_measured": ms_per_step, "nvlink_allgather_ms_per_step": t_ag * 1e3,
                            "nvlink_allreduce_ms_per_step": t_ar * 1e3, "projected_step_ms": t_proj * 1e3,
                            "projected_tokens_per_s": B / t_proj})
    res = None
    if rank == 0:
        res = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f16",
            "data": ("synthetic (reference-draw weights rescaled; random prompts, cache built by the real offloaded "
                     "prefill, then grown to the mean context in decode order)" if prefill else
                     "synthetic (reference-draw weights rescaled, pattern-filled cache)"),
            "config": bench_config(args, cfg, world, r, r_src, ctx_mid),
            "details": {"mode": mode, "host_layers_phys": Lp, "weight_layers_phys": Lw,
                        "host_pool_fold": ("none" if Lp == L and Lw == L else
                                           f"host storage folded to {Lp} cache / {Lw} weight layer copies "
                                           "(box DRAM); bytes streamed per layer unchanged"),
                        "pinned_budget_gb": budget / 1e9, "kv_host_blocks": caps.kv_host,
                        "act_host_blocks": caps.act_host, "numa_node": numa_node, "act_context_tokens": act_tokens,
                        "advanced_tokens_per_request": n_adv, "first_timed_context": c0,
                        "live_planned_r": planner.get("planned_r") if planner else None},
            "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": h2d_step + B * 4,
                    "d2h_bytes_per_step": acc["d2h"] / args.steps + B * 4,
                    "note": "decode_step C-ABI call with host token ids in / argmax out; includes the host-link "
                            "stream of weights + KV/ACT blocks and the new-token cache stores"},
            "gpu_launches": acc["launches"],
            "roofline": roof,
            "step_roofline": step_roof,
            "cpu_baseline": None,
            "clocks": clk,
            "setup_s": setup_s,
            "planner": planner,
            "prefill": prefill,
            "generation_e2e": gen,
            "tensor_parallel": tp_info,
            "weight_share": ws_info,
        }
        if ws is not None:
            res["config"]["parallelism"] = (f"batch-partitioned x{max(world, wsn)}, one weight stream shared over "
                                            f"NVLink (1/{wsn} of every layer per host link + all-gather)")
            if args.share_emulate > 1:
                res["config"]["parallelism"] += " (EMULATED: one rank on one GPU, all-gather skipped)"
                res["metric"] = METRIC + " [share-emulate: single-rank timing, NOT a whole-job measurement]"
        if tp is not None:
            res["scaling"] = "strong"
            res["config"]["parallelism"] = f"head-sharded tensor parallel x{tpn}" + (
                " (EMULATED: one rank on one GPU, collectives skipped)" if args.tp_emulate > 1 else " (NCCL)")
            res["config"]["global_batch"] = B
            if args.tp_emulate > 1:
                res["metric"] = METRIC + " [tp-emulate: single-rank timing, NOT a whole-job measurement]"
        res.update(extra)
    eng.close()
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            # after the engine released its pinned pools; every host core back
            if _ALL_CPUS:
                os.sched_setaffinity(0, _ALL_CPUS)
            n_act = int(round(r * ctx_mid))
            kind, run, sample, threads, _ = cpu_reference_sample(cfg, ctx_mid, n_act, os.cpu_count() or 1)
            run()  # warm
            t = statistics.mean([run() for _ in range(2)])
            res["cpu_baseline"] = {"value": 1.0 / (L * t), "unit": "tokens/s", "cores": threads, "kind": kind,
                                   "sample": sample, "single_thread": single_thread_leg(cfg, ctx_mid, n_act)}
        if not args.no_sweep and world == 1:
            try:
                res["hbm_resident"] = resident_variants(local, cfg, B, ctx_mid, args.arch)
            except Exception as e:
                res["hbm_resident"] = {"error": str(e)}
            # the offloaded workload itself (weights still streamed from pinned
            # host every layer) with an HBM cache tier planned by the reference's
            # own act_gpu / kv_on_gpu placement (cache.cpp:79-107): hybrid vs
            # pure KV vs pure ACT
            try:
                res["hbm_tiers_streamed_weights"] = resident_variants(local, cfg, B, ctx_mid, args.arch,
                                                                      weights_on_device=False)
            except Exception as e:
                res["hbm_tiers_streamed_weights"] = {"error": str(e)}
        if not args.no_sweep and world == 1 and args.config == 3:
            try:
                res["config1_e2e"] = config1_e2e(local, None if args.no_cpu_baseline else os.cpu_count() or 1)
            except Exception as e:
                res["config1_e2e"] = {"error": str(e)}
        if not args.no_sweep and not args.no_config2 and world == 1 and args.config == 3:
            try:
                res["config2_resident"] = config2_resident(local)
            except Exception as e:
                res["config2_resident"] = {"error": str(e)}
        print(json.dumps(res), flush=True)
    return res


def _host_mem_available():
    """MemAvailable from /proc/meminfo (bytes); 0 when unreadable (= unbounded)."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return float(line.split()[1]) * 1024
    except OSError:
        pass
    return 0.0


def resident_variants(local, cfg, B, P, arch, steps=2, warmup=1, reserve=3e9, only_planned=False,
                      weights_on_device=True):
    """The same workload with the weights AND the cache in HBM (B200 has 180 GB):
    KV and ACT blocks both placed on the GPU first (kv_on_gpu / ACT-first,
    cache.cpp:64-91). Pure KV does not fit, so its overflow blocks stream from
    pinned host memory; pure ACT fits but recomputes every context token each
    step. The capacity-constrained end of Alg. 1: with no
    link time left to hide recompute under, every KV block that fits saves
    4 d^2 tpb FLOPs per layer per step, so the capacity-only ACT share is the
    smallest one whose blocks fit the free HBM (r_fit); the balanced plan also
    streams KV blocks from pinned host while the tensor cores recompute (the
    link is idle with resident weights), minimising max(t_kv_gen, t_load_kv)
    per layer on rates measured here (r_planned). Sweeps r = 0 (KV, overflow to
    host), r_planned, r_fit, (1 + r_fit)/2 and r = 1."""
    import torch
    from paper_2501_01792_b200 import api
    L, tpb = cfg.num_layers, cfg.tokens_per_block
    total = steps + warmup + 3
    nb = math.ceil((P + total) / tpb)
    N = B * nb
    kv_all = api.HybridCache.bytes_of("KV", cfg) * L
    act_all = api.HybridCache.bytes_of("ACT", cfg) * L
    kv_one = api.HybridCache.bytes_of("KV", cfg)  # recompute output buffer per ACT block (one layer)
    eng = api.Engine(cfg, seed=42, max_seq=P + total + 1, rescale=True, max_batch=B,
                     weights_on_device=weights_on_device, caps=api.PoolCaps(), mode="act_only", device=local, arch=arch)
    # measured rates on this engine (north-star (5)): recompute GEMM vs ACT
    # tokens, host link vs KV tokens, through small calibration pools
    eng.configure_cache(api.PoolCaps(kv_host=1024, act_host=4096), mode="hybrid", host_layers=1)
    # (sustained rate: enough back-to-back launches for the power cap to settle, as in a step)
    kv_s = [(float(n), eng.time_kv_gen(n, reps=40)) for n in (4096, 16384, 32768, 65536)]
    ld_s = [(float(n), eng.time_load_kv(n, reps=2)) for n in (2048, 8192, 16384)]
    link_bps = 16384 * 2 * cfg.hidden_dim * 2 / ld_s[-1][1]
    bundle = api.bundle_from_samples(kv_s, ld_s, link_bps, cfg)
    eng.configure_cache(api.PoolCaps(), mode="act_only")
    free = torch.cuda.mem_get_info(local)[0] - reserve
    host_budget = 0.8 * _host_mem_available()  # pinned host tiers (page-locked: leave the OS headroom)
    # the library's HBM planners (csrc/host/plan.hpp): capacity-only (smallest
    # ACT share that fits) and balanced three tiers (ACT + KV in HBM, KV from
    # host, max(t_kv_gen, t_load_kv) minimised on the measured bundle)
    r_fit, caps_fit = api.plan_hbm_residency(cfg, B, nb, free)
    try:
        r_bal, caps_bal, t_bal = api.plan_hbm_tiers(cfg, B, nb, free, bundle, host_bytes=host_budget,
                                                    weights_streamed=not weights_on_device)
    except api.CapacityError as e:  # e.g. OPT-66B: 130 GB of weights leave too little HBM for this cache
        eng.close()
        return {"workload": f"{cfg.name}-shape, batch {B}, prompt {P}: weights + cache in HBM",
                "infeasible": str(e), "free_hbm_gb": free / 1e9, "host_budget_gb": host_budget / 1e9,
                "cache_gb": {"all_kv": N * kv_all / 1e9, "all_act": N * act_all / 1e9}}
    ids = [f"h{i}" for i in range(B)]
    tokens = np.random.default_rng(9).integers(0, cfg.vocab_size, (total, B)).astype(np.int32)
    out = {"workload": (f"{cfg.name}-shape, batch {B}, context {P}: " +
                        ("weights + cache in HBM" if weights_on_device else
                         "weights streamed from pinned host every layer, cache in HBM") +
                        " (KV and ACT placed on the GPU first); overflow blocks in pinned host memory"),
           "weights": "HBM" if weights_on_device else "pinned host, streamed per layer",
           "free_hbm_gb": free / 1e9, "host_budget_gb": host_budget / 1e9, "blocks": N, "r_fit": r_fit, "r_planned": r_bal,
           "planned_tiers": {"act_gpu": caps_bal.act_gpu, "kv_gpu": caps_bal.kv_gpu, "kv_host": caps_bal.kv_host,
                             "act_host": caps_bal.act_host, "predicted_t_comp_ms_per_layer": t_bal[0] * 1e3,
                             "predicted_t_link_ms_per_layer": t_bal[1] * 1e3},
           "bundle": {"kv_gen_slope": bundle.t_kv_gen.slope, "load_kv_slope": bundle.t_load_kv.slope},
           "per_ratio": []}
    def caps_at(r):  # the capacity rule at a forced share
        act_cap = 0 if r <= 0 else (N if r >= 1 else B * (math.ceil(r * nb) + 1))
        kv_need = 0 if r >= 1 else (N if r <= 0 else B * (math.ceil((1 - r) * nb) + 1))
        # KV/gpu blocks that fit next to the ACT blocks, their recompute slots and
        # the two per-layer staging slots of the overflow (kv_host) blocks
        room = free - act_cap * (act_all + kv_one) - 2 * kv_need * kv_one
        kv_gpu = int(max(0, min(kv_need, room // (kv_all - 2 * kv_one))))
        return api.PoolCaps(kv_host=kv_need - kv_gpu, kv_gpu=kv_gpu, act_gpu=act_cap)

    def tiered_alloc(c):  # HostAllocation target of a three-tier plan: ACT/gpu share of all blocks
        return api.HostAllocation(c.act_gpu, N - c.act_gpu)

    jobs = []  # (r, caps, allocation, tag)
    for r in ([r_bal] if only_planned else sorted({0.0, r_fit, r_bal, (1.0 + r_fit) / 2, 1.0})):
        a = int(round(r * 1000))
        if r == r_bal:
            jobs.append((r, caps_bal, tiered_alloc(caps_bal), "planned"))
        else:
            jobs.append((r, caps_fit if r == r_fit else caps_at(r), api.HostAllocation(a, 1000 - a),
                         "capacity_only" if r == r_fit else ""))
    while jobs:
        r, caps, alloc, tag = jobs.pop(0)
        retried = tag.startswith("retry:")
        tag = tag[len("retry:"):] if retried else tag
        act_cap, kv_gpu = caps.act_gpu, caps.kv_gpu
        mode = "kv_only" if r <= 0 else ("act_only" if r >= 1 else "hybrid")
        host_need = caps.kv_host * kv_all + caps.act_host * act_all
        if host_budget > 0 and host_need > host_budget:
            out["per_ratio"].append({"act_share_r": round(r, 4), "skipped":
                                     f"host tiers need {host_need / 1e9:.0f} GB pinned > budget {host_budget / 1e9:.0f} GB"})
            continue
        if r >= 1 and act_cap * (act_all + kv_one) > free:
            out["per_ratio"].append({"act_share_r": round(r, 4), "skipped":
                                     f"ACT blocks need {act_cap * (act_all + kv_one) / 1e9:.0f} GB HBM > free "
                                     f"{free / 1e9:.0f} GB"})
            continue
        try:
            eng.configure_cache(caps, mode=mode, allocation=alloc, kv_on_gpu=True)
            eng.admit_synthetic(ids, [P] * B, seed=11)
            run_steps(eng, ids, tokens, 0, warmup)
            acc = run_steps(eng, ids, tokens, warmup, steps)
            prof = run_steps(eng, ids, tokens, warmup + steps, 1, prof=True)["last"]
            ms = acc["dev_ms"] / steps
            out["per_ratio"].append({"act_share_r": round(r, 4), "mode": mode, "tokens_per_s": B * 1e3 / ms,
                                     "profile_split_ms": {"recompute": prof["recompute_ms"],
                                                          "attention": prof["attn_ms"],
                                                          "qkv_proj_ffn": prof["gemm_ms"],
                                                          "copy_stream": prof["copy_ms"],
                                                          "step_profiled": prof["step_ms"]},
                                     "recompute_rows": prof["recompute_rows"],
                                     "ms_per_step": ms, "kv_gpu_blocks": kv_gpu, "kv_host_blocks": caps.kv_host,
                                     "act_gpu_blocks": act_cap, "h2d_gb_per_step": acc["h2d"] / steps / 1e9,
                                     "planned": tag == "planned", "capacity_only": tag == "capacity_only",
                                     "replanned": tag == "replanned", "retried_host_alloc": retried})
            if tag == "planned" and prof["recompute_rows"] > 0 and prof["recompute_ms"] > 0:
                # closed loop (north-star (5)): the recompute rate measured IN the step
                # (power cap, concurrent DMA) replaces the isolated calibration slope,
                # and the balance is re-solved on it
                slope = prof["recompute_ms"] / 1e3 / prof["recompute_rows"]
                b2 = api.TimingBundle(api.LinearTimeModel(slope, 0.0, 1.0, False), bundle.t_load_kv,
                                      bundle.t_load_w, bundle.s_weight_layer, bundle.s_weight_total)
                r2, caps2, t2 = api.plan_hbm_tiers(cfg, B, nb, free, b2, host_bytes=host_budget,
                                                   weights_streamed=not weights_on_device)
                out["replanned"] = {"insitu_kv_gen_slope": slope, "r": r2,
                                    "tiers": {"act_gpu": caps2.act_gpu, "kv_gpu": caps2.kv_gpu,
                                              "kv_host": caps2.kv_host, "act_host": caps2.act_host},
                                    "predicted_t_comp_ms_per_layer": t2[0] * 1e3,
                                    "predicted_t_link_ms_per_layer": t2[1] * 1e3}
                if caps2.act_gpu != caps_bal.act_gpu:
                    jobs.insert(0, (r2, caps2, tiered_alloc(caps2), "replanned"))
        except Exception as e:
            if "cudaHostAlloc" in str(e) and not retried:
                # page-locking the host tier can fail transiently while the OS
                # reclaims the previous tier's pages: release every pool and retry once
                try:
                    eng.configure_cache(api.PoolCaps(), mode="act_only")
                except Exception:
                    pass
                import gc
                gc.collect()
                time.sleep(5)
                jobs.insert(0, (r, caps, alloc, "retry:" + tag))
                continue
            out["per_ratio"].append({"act_share_r": round(r, 4), "error": str(e)})
    eng.close()
    return out


def config1_e2e(local, cpu_threads, B=4, P=128, G=32):
    """BASELINE configs[0] end to end: OPT-125M shape, batch 4, prompt 128, gen
    32, KV:ACT 0.5 (HostAllocation{K, K}: ACT, KV, ACT, ... blocks in pinned
    host pools). GPU: prefill + 32 greedy decode steps through the C ABI
    (token ids in, argmax out, fed back), wall clock. CPU reference (the
    reference library on this host): one request's prefill + 32 steps, each
    assembling its context from stored KV blocks and ACT blocks recomputed by
    recompute_kv_from_activation (verify.cpp:62-73), then generation_step +
    tied-head greedy token; tokens/s scaled to the request."""
    from paper_2501_01792_b200 import api
    cfg = api.ModelConfig(num_layers=12, hidden_dim=768, num_heads=12, ffn_dim=3072, vocab_size=50272,
                          name="opt-125m")
    tpb = cfg.tokens_per_block
    nb = math.ceil((P + G) / tpb)
    K = B * nb
    rng = np.random.default_rng(3)
    prompts = [rng.integers(0, cfg.vocab_size, P).tolist() for _ in range(B)]
    eng = api.Engine(cfg, seed=42, max_seq=P + G + 1, rescale=True, max_batch=B, weights_on_device=True,
                     caps=api.PoolCaps(kv_host=K, act_host=K), allocation=api.HostAllocation(K, K), mode="hybrid",
                     device=local)

    def generate(tag):
        rids = [f"{tag}{i}" for i in range(B)]
        t0 = time.perf_counter()
        eng.prefill(rids, prompts)
        toks = [p[-1] for p in prompts]
        out = {"argmax": np.zeros(B, np.int32)}
        seqs = []
        for _ in range(G):
            eng.decode_step(rids, toks, want_x=False, want_argmax=True, out=out)
            toks = out["argmax"].tolist()
            seqs.append(toks)
        wall = time.perf_counter() - t0
        for r in rids:
            eng.free_request(r)
        return wall, seqs

    generate("w")  # warm-up
    walls = [generate(f"t{i}_")[0] for i in range(3)]
    wall = statistics.median(walls)
    eng.close()
    res = {"workload": "opt-125m-shape, batch 4, prompt 128, gen 32 greedy, KV:ACT 0.5, cache in pinned host pools",
           "gpu": {"tokens_per_s": B * G / wall, "wall_s": wall, "includes": "prefill + 32 decode steps, C-ABI "
                   "calls with host token ids / argmax"}}
    if cpu_threads:
        os.environ["OMP_NUM_THREADS"] = str(cpu_threads)
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import ref_lib as R  # noqa: E402  (CPU baseline only)
        if R.available():
            cpu_threads = R.set_threads(cpu_threads)
            rw = R.RefWeights(12, 768, 12, 3072, 50272, tpb, 42, P + G + 1)
            emb = rw.get(0)
            t0 = time.perf_counter()
            ins, k, v, out = rw.forward_prompt(prompts[0])
            ctx_k = np.array(k)
            ctx_v = np.array(v)
            tok = int(np.argmax(out[-1] @ emb.T))
            for g in range(G):
                # ACT-kind blocks (every other block) are rebuilt from their activations
                kk, vv = ctx_k.copy(), ctx_v.copy()
                n = ctx_k.shape[1]
                for blk in range(0, (min(n, P) + tpb - 1) // tpb, 2):
                    sl = slice(blk * tpb, min((blk + 1) * tpb, P))
                    for l in range(12):
                        kk[l, sl], vv[l, sl] = rw.recompute_kv(l, ins[l, sl])
                o, nk, nv = rw.generation_step(tok, n, kk, vv)
                ctx_k = np.concatenate([ctx_k, nk[:, None, :]], axis=1)
                ctx_v = np.concatenate([ctx_v, nv[:, None, :]], axis=1)
                tok = int(np.argmax(o[0] @ emb.T))
            cpu_s = time.perf_counter() - t0
            res["cpu_reference"] = {"tokens_per_s": G / cpu_s, "wall_s": cpu_s, "cores": cpu_threads,
                                    "kind": "reference", "sample": "1 request: forward_prompt(128) + 32 greedy "
                                    "steps (ACT blocks recomputed each step + generation_step)"}
            res["gpu_over_cpu"] = res["gpu"]["tokens_per_s"] / res["cpu_reference"]["tokens_per_s"]
    return res


def config2_resident(local, B=64, P=512, steps=3, warmup=2):
    """BASELINE configs[1]: OPT-6.7B shape, batch 64, prompt 512, ACT-only
    cache resident in HBM, weights resident — the tensor-bound configuration
    (every step recomputes K|V of the whole context from X)."""
    from paper_2501_01792_b200 import api
    hbm_peak, tflops_sust, tflops_burst, _ = measured_peaks()
    cfg = api.ModelConfig.preset("opt-6.7b")
    L, d, f = cfg.num_layers, cfg.hidden_dim, cfg.ffn_dim
    total = steps + warmup + 2
    nb = math.ceil((P + total) / cfg.tokens_per_block)
    eng = api.Engine(cfg, seed=42, max_seq=P + total + 1, max_batch=B, weights_on_device=True,
                     caps=api.PoolCaps(act_gpu=B * nb), mode="act_only", device=local)
    ids = [f"c2r{i}" for i in range(B)]
    eng.admit_synthetic(ids, [P] * B, seed=5)
    tokens = np.random.default_rng(2).integers(0, cfg.vocab_size, (total, B)).astype(np.int32)
    run_steps(eng, ids, tokens, 0, warmup)
    prof = run_steps(eng, ids, tokens, warmup, 1, prof=True)["last"]
    act = act_context_tokens(eng, ids)
    fused = eng.fused_recompute()
    acc = run_steps(eng, ids, tokens, warmup + 1, steps)
    eng.close()
    ms = acc["dev_ms"] / steps
    rec_ms = prof["recompute_ms"] / max(prof["recompute_launches"], 1)
    rec_tflops = 4.0 * d * d * act / (rec_ms / 1e3) / 1e12 if rec_ms else None
    flops = L * (4.0 * d * d * act + 2.0 * B * (4 * d * d + 2 * d * f))
    ctx = P + warmup + 2
    # ACT rows read by the recompute (+ its K|V written and read back by the attention
    # unless the recompute is fused with it) and the layer weights
    hbm = L * (act * (d * 2 if fused else 5 * d * 2) + (4 * d * d + 2 * d * f) * 2)
    t_roof = max(flops / (tflops_sust * 1e12), hbm / (hbm_peak * 1e9))
    return {"workload": "opt-6.7b-shape, batch 64, prompt 512, ACT-only cache + weights resident in HBM",
            "tokens_per_s": B * 1e3 / ms, "ms_per_step": ms, "e2e_tokens_per_s": B * steps / acc["wall"],
            "recompute_tflops": rec_tflops, "recompute_frac_of_sustained": rec_tflops / tflops_sust if rec_tflops else None,
            "step_roofline": {"bound": "tensor" if flops / (tflops_sust * 1e12) >= hbm / (hbm_peak * 1e9) else "hbm",
                              "t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms,
                              "roofline_tokens_per_s": B / t_roof},
            "profile_split_ms": {"recompute": prof["recompute_ms"], "attention": prof["attn_ms"],
                                 "qkv_proj_ffn": prof["gemm_ms"]},
            "act_context_tokens": act, "recompute_rows": prof["recompute_rows"],
            "recompute_fused_with_attention": fused, "launches_per_step": acc["launches"] / steps}


def full_generation(args, cfg, local):
    """The whole generation, timed: real prefill of B prompts of P tokens, then
    G decode steps, every step timed with CUDA events (the paper's and the
    sim's end-to-end definition, sim.cpp:618-628)."""
    from paper_2501_01792_b200 import api, kernels
    if kernels.device_count() == 0:
        raise SystemExit("bench needs a CUDA device")
    hbm_peak, tflops_sust, _, _ = measured_peaks()
    bind_numa(local)
    B, P, G, L = args.batch or 128, args.prompt, args.gen, cfg.num_layers
    bp = bundle_path(args)
    alloc6 = None
    if args.ratio >= 0:
        r, src = args.ratio, "--ratio"
    else:
        r, factor, alloc6 = planned_ratio(read_bundle(bp), cfg, B * (P + G),
                                     lambda b5, m4, tpb, ag: list(api.plan_host_allocation(
                                         api.TimingBundle(api.LinearTimeModel(b5[0], b5[1]),
                                                          api.LinearTimeModel(b5[2], b5[3]), b5[4]),
                                         api.MemoryBudget(*m4), tpb, ag).__dict__.values()))
        src = f"planner on {os.path.relpath(bp, ROOT)}"
    mode, alloc, caps = pool_plan(cfg, B, P + G + 1, 0, r)
    w_layer, _ = api.weight_bytes(cfg)
    budget = args.host_gb * 1e9 if args.host_gb > 0 else max(16e9, mem_available_bytes() - 40e9)
    Lw = L if L * w_layer <= 0.55 * budget else max(2, int(0.55 * budget // w_layer))
    Lp = host_layers_for(cfg, caps, budget, Lw * w_layer)
    eng = api.Engine(cfg, seed=42, max_seq=P + G + 2, rescale=True, max_batch=B, weights_on_device=False, caps=caps,
                     host_layers=Lp, weight_layers=Lw, mode=mode, allocation=alloc, device=local, arch=args.arch)
    ids = [f"f{i}" for i in range(B)]
    rng = np.random.default_rng(100)
    prompts = [rng.integers(0, cfg.vocab_size, P).tolist() for _ in ids]
    import torch
    torch.cuda.synchronize()
    eng.set_profile(True)
    w0 = time.perf_counter()
    eng.prefill(ids, [p[:-1] for p in prompts])  # the last prompt token is the first decode step's input
    eng.set_profile(False)
    prefill_s = eng.last_stats()["step_ms"] / 1e3
    pre = eng.last_stats()
    out = {"argmax": np.zeros(B, np.int32)}
    toks = [p[-1] for p in prompts]
    step_ms, traffic = [], {k: pre[k] for k in ("h2d_weights", "h2d_kv", "h2d_act", "d2h_kv", "d2h_act")}
    busy = []  # (compute busy, copy busy) fractions of the profiled steps
    trace = None
    clocks = ClockSampler(local)
    clocks.start()
    for g in range(G):
        prof = g % 32 == 16  # every 32nd step profiled (CUDA events per kernel, eager)
        eng.set_profile(prof)
        eng.decode_step(ids, toks, want_x=False, want_argmax=True, out=out)
        st = eng.last_stats()
        step_ms.append(st["step_ms"])
        for k in traffic:
            traffic[k] += st[k]
        if prof:
            busy.append(((st["recompute_ms"] + st["attn_ms"] + st["gemm_ms"]) / st["step_ms"],
                         st["copy_ms"] / st["step_ms"]))
            if trace is None:
                trace = eng.trace()
        toks = out["argmax"].tolist()
    eng.set_profile(False)
    wall = time.perf_counter() - w0
    clk = clocks.stop()
    eng.close()
    dec_s = sum(step_ms) / 1e3
    makespan = prefill_s + dec_s
    gpu_dec = statistics.mean(b for b, _ in busy) if busy else None
    pcie_dec = statistics.mean(c for _, c in busy) if busy else None
    pre_busy = (pre["gemm_ms"] + pre["attn_ms"]) / pre["step_ms"] if pre["step_ms"] else 0.0
    pre_copy = pre["copy_ms"] / pre["step_ms"] if pre["step_ms"] else 0.0
    res = {
        "metric": METRIC + " [whole generation: prefill + G greedy decode steps, every step timed]",
        "value": B * G / makespan, "unit": "tokens/s", "n_gpus": 1, "dtype": "f16",
        "config": {"workload": f"{cfg.name}, batch {B}, prompt {P}, gen {G}, weights + cache in pinned host",
                   "act_share_r": r, "ratio_source": src, "mode": mode, "host_layers_phys": Lp,
                   "weight_layers_phys": Lw},
        "prefill_s": prefill_s, "decode_s": dec_s, "decode_tokens_per_s": B * G / dec_s,
        "wall_s": wall, "e2e_tokens_per_s": B * G / wall,
        "step_ms": {"first": step_ms[0], "mid": step_ms[len(step_ms) // 2], "last": step_ms[-1],
                    "mean": statistics.mean(step_ms), "all": [round(x, 3) for x in step_ms]},
        "clocks": clk}
    if args.artifacts:
        # the reference CLI's metrics.json (main.cpp:101-115, 255-261) for the MEASURED run:
        # busy fractions from the profiled steps (every 32nd) and the profiled prefill
        tb = {"weights": traffic["h2d_weights"], "kv_load": traffic["h2d_kv"], "act_load": traffic["h2d_act"],
              "kv_store": traffic["d2h_kv"], "act_store": traffic["d2h_act"]}
        tot = sum(tb.values())
        metrics = {"tokens_generated": B * G, "makespan_s": makespan, "throughput_tok_s": B * G / makespan,
                   "pcie_busy": (pre_copy * prefill_s + (pcie_dec or 0.0) * dec_s) / makespan,
                   "gpu_busy": (pre_busy * prefill_s + (gpu_dec or 0.0) * dec_s) / makespan,
                   "prefill_s": prefill_s, "gen_s": dec_s, "traffic": {k: int(v) for k, v in tb.items()},
                   "mode": mode, "batch": B, "prompt_len": P, "gen_len": G,
                   "traffic_report": dict({k: int(v) for k, v in tb.items()}, total=int(tot),
                                          context_load=int(tb["kv_load"] + tb["act_load"]),
                                          **{f"frac_{k}": v / tot for k, v in tb.items()}),
                   "measured_on": "B200, bench.py --full-generation (every step timed)",
                   "meta": {"version": "b200-measured", "seed": 42, "inputs": {}}}
        os.makedirs(args.artifacts, exist_ok=True)
        with open(os.path.join(args.artifacts, "metrics.json"), "w") as fh:
            json.dump(metrics, fh, indent=2)
        if trace is not None:
            trace["meta"] = metrics["meta"]
            with open(os.path.join(args.artifacts, "trace.json"), "w") as fh:
                json.dump(trace, fh)
        if bp and alloc6:  # the bundle the ratio came from and the plan Alg. 1 made of it
            import shutil
            shutil.copy(bp, os.path.join(args.artifacts, "bundle.json"))
            b7 = read_bundle(bp)
            tb5 = api.TimingBundle(api.LinearTimeModel(b7[0], b7[1]), api.LinearTimeModel(b7[2], b7[3]), b7[4])
            ha = api.HostAllocation(*alloc6)
            plan = dict(ha.__dict__, predicted={"t_pcie": api.planned_t_pcie(tb5, cfg.tokens_per_block, ha),
                                                "t_computation": api.planned_t_computation(tb5, cfg.tokens_per_block,
                                                                                           ha, 0)},
                        meta=metrics["meta"])
            with open(os.path.join(args.artifacts, "plan.json"), "w") as fh:
                json.dump(plan, fh, indent=2)
        res["artifacts"] = {"dir": args.artifacts, "metrics": {k: metrics[k] for k in
                                                               ("pcie_busy", "gpu_busy", "prefill_s", "gen_s")}}
    print(json.dumps(res), flush=True)


def main():
    args = parse()
    world, rank, local, dist = dist_setup(args)
    if args.impl == "reference":  # the reference's CPU path: the product is never imported
        reference_arm(args, world, rank, dist)
    else:
        from paper_2501_01792_b200 import api
        cfg = api.ModelConfig.preset(args.model)
        if args.layers:
            cfg.num_layers = args.layers
        if args.full_generation:
            if rank == 0:
                full_generation(args, cfg, local)
        else:
            our_arm(args, cfg, world, rank, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
