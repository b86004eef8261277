"""bench.py on the GPU through the multi-GPU code path as one rank (--nccl-single): an NCCL
process group, the bucketed all-reduce of the flat gradient buffer on its side stream,
barriers and the max over ranks — the path `python bench.py --gpus N` takes on N GPUs
(SURVEY §8(e)); this round's boxes have one GPU."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_nccl_code_path_one_rank():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C1", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--nccl-single"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(line) == 1, r.stdout[-2000:]
    d = json.loads(line[0])
    assert d["n_gpus"] == 1 and d["value"] > 0
    assert d["config"]["allreduce"].startswith("NCCL sum"), d["config"]["allreduce"]
    assert d["gpu_launches"] > 0
