"""The N>1 bench path as the driver launches it — torchrun, one process per
rank, each rank its own engine, requests, pools and copy streams (SURVEY.md
§8(e): batch partition, no data-path collective) — run with two ranks on the
ONE GPU this box has (HC_DIST_BACKEND=gloo carries the barrier / max-over-ranks
plumbing; NCCL refuses two ranks per device). Checks the JSON line the driver
parses: whole-job tokens summed over ranks, device time max over ranks."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("share", [False])
def test_two_process_bench_on_one_gpu(native, share):
    env = dict(os.environ, HC_DIST_BACKEND="gloo", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--model", "opt-6.7b", "--layers", "2", "--batch", "8", "--prompt", "64", "--gen", "16",
           "--no-sweep", "--no-cpu-baseline", "--host-gb", "8", "--bundle", "live"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 alone prints
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["scaling"] == "weak"
    assert j["config"]["global_batch"] == 16 and j["config"]["batch_per_gpu"] == 8
    assert j["value"] > 0 and j["e2e"]["value"] > 0
    # whole-job value = both ranks' tokens over the slowest rank's device time
    assert abs(j["value"] - 2 * 8 * j["steps"] / (j["ms_per_step"] * j["steps"] / 1e3)) <= 1e-6 * j["value"]
    assert j["gpu_launches"] > 0
