"""BASELINE configs[1] alone (OPT-6.7B shape, batch 64, prompt 512,
ACT-only cache + weights resident in HBM): prints bench.config2_resident()."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

if __name__ == "__main__":
    print(json.dumps(bench.config2_resident(0)))
