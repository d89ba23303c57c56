"""Decode (M = batch) GEMMs on the B200: device microseconds per launch and
weight GB/s for the tile kernel + split-K (mode 0) and the weight-streaming
stream-K kernel (mode 1, wstream.cuh), back-to-back launches with W streamed
from HBM (hc_gemm_bench). Not a test.

    python scripts/decode_gemm_bench.py [reps]
"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2501_01792_b200._native import lib, check  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    shapes = []
    for name, d, f, V, B in (("opt-6.7b", 4096, 16384, 50272, 64), ("opt-30b", 7168, 28672, 50272, 128),
                             ("opt-30b", 7168, 28672, 50272, 32)):
        shapes += [(name, B, "qkv", 3 * d, d, 0), (name, B, "proj", d, d, 0), (name, B, "ffn1", f, d, 1),
                   (name, B, "ffn2", d, f, 0), (name, B, "lm_head", V, d, 3)]
    out = []
    for name, M, op, N, K, epi in shapes:
        row = {"model": name, "M": M, "op": op, "N": N, "K": K}
        for mode in (0, 1, 2):
            us = C.c_double()
            check(lib().hc_gemm_bench(M, N, K, epi, mode, reps, C.byref(us)))
            row[f"us_{mode}"] = us.value
            row[f"wgbs_{mode}"] = N * K * 2 / (us.value * 1e-6) / 1e9
        out.append(row)
        print(json.dumps(row), flush=True)
    tot = {}
    for r in out:
        k = (r["model"], r["M"])
        t = tot.setdefault(k, [0.0, 0.0, 0.0, 0.0])
        for i in range(3):
            t[i] += r[f"us_{i}"]
        t[3] += r["N"] * r["K"] * 2
    for (name, M), t in tot.items():
        print(json.dumps({"model": name, "M": M, **{f"all_us_{i}": t[i] for i in range(3)},
                          **{f"wgbs_{i}": t[3] / t[i] / 1e3 for i in range(3)}}))


if __name__ == "__main__":
    main()
