"""Soak run of the serving fuzz (tests/test_engine_gpu.py::test_engine_fuzz_against_oracle)
over many seeds and all cache modes (not a test; GPU box):

    python scripts/soak_fuzz.py [first_seed] [n_seeds]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)

import test_engine_gpu as T  # noqa: E402


def main():
    first = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    fails = runs = 0
    for seed in range(first, first + n):
        for mode, arch in (("hybrid", "reference"), ("kv_only", "reference"), ("act_only", "reference"),
                           ("hybrid", "opt")):
            runs += 1
            try:
                T.test_engine_fuzz_against_oracle(None, seed, mode, arch)
            except Exception as e:  # noqa: BLE001 — reported, the soak goes on
                fails += 1
                print("FAIL", seed, mode, arch, repr(e)[:400], flush=True)
    print(f"soak done: {runs} sessions, {fails} failures", flush=True)


if __name__ == "__main__":
    main()
