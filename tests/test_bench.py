"""bench.py's contract on CPU: the reference arm (the C oracle port on the
host cores) prints one JSON line with the keys the driver reads; under
torchrun every rank but 0 exits 0 without work.  The GPU arm needs a B200
and is exercised by the round-end bench run."""

from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, *args):
    env = dict(os.environ, **(extra_env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                           "--config", "cfg2", "--steps", "2", "--warmup", "1", *args],
                          capture_output=True, text=True, env=env, cwd=ROOT, timeout=300)


def test_reference_arm_line():
    p = _run()
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["steps"] == 2 and line["warmup"] == 1 and line["higher_is_better"] is True
    assert line["value"] > 0 and line["cpu_baseline"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_exit_quietly():
    p = _run({"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"})
    assert p.returncode == 0, p.stderr
    assert p.stdout.strip() == ""


def test_reference_arm_runs_reference_package():
    """The reference arm's side entry times the reference package itself
    (baseline/_ref) on the same code, single worker and all cores."""
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "mindist")):
        import pytest

        pytest.skip("baseline/_ref not installed")
    p = _run(None, "--ref-python-max-g", "3")
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    ref = line["reference_python"]
    assert ref["workers_1"]["combinations"] == 2 * (48 + 1128 + 17296)
    assert ref["workers_1"]["bounds_trace"][:3] == [[1, 4, 16], [2, 6, 15], [3, 8, 12]]


def test_spawned_ranks_json_contract():
    """`bench.py --gpus 2` outside torchrun spawns two ranks itself (here in
    the hidden gloo self-test mode: no device work) and rank 0 alone prints
    one JSON line with n_gpus = 2 and the max-over-ranks step time."""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--cpu-selftest", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert p.returncode == 0, p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["steps"] == 3 and line["warmup"] == 3
    # rank 1 sleeps 4 ms per step, rank 0 2 ms: the reported time is rank 1's
    assert line["ms_per_step"] >= 3.5


def test_reference_arm_under_spawn():
    """The reference arm launched with --gpus 2: rank 0 prints the line
    (the GPU count only labels it), rank 1 exits without work."""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "cfg1", "--gpus", "2", "--steps", "1", "--warmup", "1",
                        "--no-extra"],
                       capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert p.returncode == 0, p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
