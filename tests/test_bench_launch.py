"""`python bench.py --gpus 2` on one host: the script re-launches itself under torchrun (one rank
per GPU; gloo here on CPU), every rank reports, rank 0 prints ONE line with n_gpus == 2
(VERDICT r1 item 6).  The reference arm runs on rank 0 alone, the other ranks exit 0."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "PMG_BENCH_LAUNCHED")}
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    return lines[0]


def test_self_launch_two_ranks_gloo():
    line = _run("--gpus", "2", "--impl", "selftest", "--steps", "1", "--warmup", "0")
    assert line["n_gpus"] == 2
    # rank 0: 1000 units in 1 s, rank 1: 2000 units in 2 s -> 3000 / 2
    assert line["units"] == 3000.0 and line["seconds"] == 2.0 and line["value"] == 1500.0


def test_self_launch_reference_arm_rank0_only():
    line = _run("--gpus", "2", "--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0")
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
