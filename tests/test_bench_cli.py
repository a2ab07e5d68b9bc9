"""bench.py's contract pieces that run without a GPU: the reference arm's
JSON line (the oracle port timed on host cores), and ``--gpus N`` relaunching
itself as N ranks under torch.distributed.run (rank 0 alone prints)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return [json.loads(l) for l in lines]


def test_reference_arm_line():
    (line,) = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--n-p", "64", "--n-theta", "32"])
    assert line["impl"] == "reference" and line["n_gpus"] == 1 and line["steps"] == 1
    assert line["value"] > 0 and line["unit"] == "slices/s" and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "slices/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_gpus_flag_relaunches_ranks():
    lines = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--n-p", "64",
                  "--n-theta", "32"])
    assert len(lines) == 1                      # rank 0 prints, rank 1 exits without work
    assert lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
