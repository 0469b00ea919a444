"""bench.py contract: one JSON line with the driver's keys (default and reference arms)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
        "cpu_baseline"}


def _run(args, timeout=900):
    env = dict(os.environ, HC_BENCH_NO_CLOCKS="1")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_runs_on_the_host():
    d = _run(["--impl", "reference", "--workload", "cfg1", "--steps", "2", "--warmup", "3",
              "--cpu-seconds", "0.5"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert KEYS <= set(d) and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_b200_arm_full_line_with_cpu_baseline():
    d = _run(["--workload", "cfg1", "--steps", "6", "--warmup", "3", "--cpu-seconds", "0.5"])
    assert KEYS <= set(d) and {"roofline", "gpu_launches", "clocks"} <= set(d)
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["cpu_baseline"]["value"] > 0 and d["roofline"]["bound"] == "hbm"
