"""Recompute-GEMM SUSTAINED throughput sweep on the B200 (not a test).

The recompute GEMM runs inside long tensor-bound steps under the 1 kW power cap,
so what matters is its rate once clocks settle, not a burst of 10 launches.
Each setting runs gemm_tn_kernel<.., kKvPaged> (or the CTA-pair kernel)
back to back for ~`secs` seconds twice and reports the second window, with the
median SM clock and power nvidia-smi saw during it.

    python scripts/gemm_sustained.py [--n 122880] [--width 7168] [--secs 3]
        [--grid "pair=0,1;group=16,32;gn=0,16;l2=0,5;fused=0,1"]   (gn: weight-stationary raster)
"""
import argparse
import itertools
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json
sys.path.insert(0, ROOT)
from paper_2501_01792_b200 import api
n, dm, secs = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
cfg = api.ModelConfig.preset({7168: "opt-30b", 4096: "opt-6.7b", 5120: "opt-13b", 9216: "opt-66b"}[dm])
cfg.num_layers = 1
blocks = (n + 15) // 16 + 8
eng = api.Engine(cfg, seed=1, max_seq=64, max_batch=1, weights_on_device=True,
                 caps=api.PoolCaps(kv_host=16, act_host=blocks), mode="hybrid")
eng.admit_synthetic(["x"], [16], seed=3)
t1 = eng.time_kv_gen(n, reps=3)
reps = max(3, int(secs / t1))
eng.time_kv_gen(n, reps=reps)          # warm the clocks / power state
print("GO", flush=True)
t = eng.time_kv_gen(n, reps=reps)
print(json.dumps({"ms": t * 1e3, "tflops": 4.0 * dm * dm * n / t / 1e12, "burst_ms": t1 * 1e3, "reps": reps}))
"""


def smi_sampler(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True)
        try:
            c, pw = r.stdout.strip().split(",")
            out.append((float(c), float(pw)))
        except ValueError:
            pass
        time.sleep(0.2)


def run(n, dm, secs, env):
    p = subprocess.Popen([sys.executable, "-c", f"ROOT={ROOT!r}\n" + CHILD, str(n), str(dm), str(secs)],
                         env=dict(os.environ, **env), stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    samples, stop, th = [], threading.Event(), None
    lines = []
    for line in p.stdout:
        lines.append(line)
        if line.startswith("GO"):
            th = threading.Thread(target=smi_sampler, args=(stop, samples), daemon=True)
            th.start()
    stop.set()
    if th:
        th.join()
    err = p.stderr.read()
    p.wait()
    res = None
    for line in lines:
        if line.startswith("{"):
            res = json.loads(line)
    if res is None:
        return {"error": err[-400:]}
    if samples:
        cs = sorted(s[0] for s in samples)
        ps = sorted(s[1] for s in samples)
        res["sm_mhz"] = cs[len(cs) // 2]
        res["power_w"] = ps[len(ps) // 2]
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=122880)
    ap.add_argument("--width", type=int, default=7168)
    ap.add_argument("--secs", type=float, default=3.0)
    ap.add_argument("--grid", default="pair=0,1;group=16,32;l2=0,5")
    a = ap.parse_args()
    axes = {}
    for part in a.grid.split(";"):
        k, v = part.split("=")
        axes[k] = v.split(",")
    keys = list(axes)
    for combo in itertools.product(*[axes[k] for k in keys]):
        st = dict(zip(keys, combo))
        env = {"HC_GEMM_PAIR": st.get("pair", "0"), "HC_GEMM_PAIR_MAX_K": "100000",
               "HC_GEMM_GROUP_M": st.get("group", "16"), "HC_GEMM_L2HINT": st.get("l2", "0"),
               "HC_FUSED_RECOMPUTE": st.get("fused", "1"), "HC_GEMM_GROUP_N": st.get("gn", "0")}
        res = run(a.n, a.width, a.secs, env)
        print(json.dumps({"n": a.n, "width": a.width, **st, **res}), flush=True)


if __name__ == "__main__":
    main()
