"""bench.py contract checks that run without a GPU: the reference (oracle) arm prints one
JSON line with the keys the driver reads (BASELINE metric, impl, cpu_baseline, e2e)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--config", "C0", "--ref-pixels", "8", "--ref-grads", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("fwd+bwd frames/sec") and d["unit"] == "frames/s"
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C0")


def _dry_run(*extra):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run-gloo", "--steps", "2",
                        "--warmup", "3", *extra], capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_bench_gpus2_relaunches_two_gloo_ranks():
    """`python bench.py --gpus 2` without a torchrun environment re-launches itself as two
    ranks (torch.distributed.run, 127.0.0.1); the dry run exercises the distributed step
    (partition, flat-buffer all-reduce in buckets checked against the sum over ranks,
    bitwise-equal replicas, barrier + max-over-ranks timing) and reports n_gpus = 2."""
    d = _dry_run("--gpus", "2", "--config", "C3", "--views-per-step", "4", "--bucket-mb", "0")
    assert d["n_gpus"] == 2 and d["config"]["views_per_step_per_rank"] == 4
    assert d["config"]["parallelism"].startswith("view-parallel dp2")
    assert d["value"] > 0 and d["scaling"] == "weak"


def test_bench_epoch_mode_and_more_ranks_than_views():
    d = _dry_run("--gpus", "2", "--config", "C3", "--views-per-step", "epoch")
    assert d["config"]["views_per_step_per_rank"] == 100  # ceil(200 views / 2 ranks)
    d = _dry_run("--gpus", "3", "--config", "C0")  # 1 view, 3 ranks
    assert d["n_gpus"] == 3


def test_bench_rejects_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run-gloo", "--gpus", "2"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr
