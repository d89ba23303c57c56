"""A/B of kernel settings on BASELINE config 2 (OPT-6.7B, B 64, P 512, ACT-only
cache + weights in HBM: the tensor-bound configuration), interleaved over
rounds so clock / power drift hits every setting alike. Each setting is an
environment (e.g. "HC_GEMM_PAIR=0"); each run is a fresh process (the knobs
are read once per process). Not a test.

    python scripts/config2_ab.py ROUNDS "SETTING_A" "SETTING_B" ...
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys
sys.path.insert(0, %r)
import bench
r = bench.config2_resident(0)
print("RESULT " + json.dumps({"tok_s": r["tokens_per_s"], "ms": r["ms_per_step"],
                              "rec_tflops": r["recompute_tflops"], "split": r["profile_split_ms"]}))
""" % ROOT


def main():
    rounds = int(sys.argv[1])
    settings = sys.argv[2:] or [""]
    res = {s: [] for s in settings}
    for _ in range(rounds):
        for s in settings:
            env = dict(os.environ)
            for kv in s.split():
                k, v = kv.split("=", 1)
                env[k] = v
            out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, cwd=ROOT)
            line = [x for x in out.stdout.splitlines() if x.startswith("RESULT ")]
            r = json.loads(line[-1][7:]) if line else {"error": out.stderr[-400:]}
            res[s].append(r)
            print(json.dumps({"setting": s, **r}), flush=True)
    for s, rs in res.items():
        ok = [r for r in rs if "tok_s" in r]
        if ok:
            print(json.dumps({"setting": s, "mean_tok_s": sum(r["tok_s"] for r in ok) / len(ok),
                              "mean_rec_tflops": sum(r["rec_tflops"] for r in ok) / len(ok), "n": len(ok)}))


if __name__ == "__main__":
    main()
