"""bench.py contract: one JSON line with the driver's keys (default and reference arms)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest


def _free_port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]

ROOT = Path(__file__).resolve().parent.parent
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
        "cpu_baseline"}


def _run(args, timeout=900, ranks=1, **env_kw):
    env = dict(os.environ, HC_BENCH_NO_CLOCKS="1", **env_kw)
    launch = [sys.executable, str(ROOT / "bench.py")] if ranks == 1 else [
        sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
        "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "bench.py")]
    out = subprocess.run([*launch, *args], capture_output=True,
                         text=True, timeout=timeout, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_timing_protocol_per_workload():
    """L2 flush only where a step's K/V fits in L2 (cfg1); settle steps only for the
    frequently drifting workload (cfg4); both enter the config both arms print."""
    sys.path.insert(0, str(ROOT))
    import bench

    args = bench.parse(["--workload", "cfg1"])
    flush = {}
    for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        w = bench.workload_of(bench.parse(["--workload", name]))
        from paper_2601_13684_b200.workload import rho_for

        flush[name] = bench.l2_flush(args, w, rho_for(w.model, w.compression), 1)
        assert bench.settle_steps(w) == (96 if name == "cfg4" else 0)
        assert not bench.l2_flush(args, w, rho_for(w.model, w.compression), 2)
    assert flush == {"cfg1": True, "cfg2": False, "cfg3": False, "cfg4": False, "cfg5": False}


def test_reference_arm_runs_on_the_host():
    d = _run(["--impl", "reference", "--workload", "cfg1", "--steps", "2", "--warmup", "3"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert KEYS <= set(d) and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_b200_arm_full_line_with_cpu_baseline_and_parity():
    args = ["--workload", "cfg1", "--steps", "12", "--warmup", "3"]
    d = _run(args + ["--secondary", "none"])
    assert KEYS <= set(d) and {"roofline", "gpu_launches", "clocks", "parity"} <= set(d)
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["cpu_baseline"]["value"] > 0 and d["roofline"]["bound"] == "hbm"
    p = d["parity"]
    assert p["within_tolerance"] and p["events_identical"] and p["step"] == 15
    assert d["config"]["l2"].startswith("flushed")  # cfg1's K/V fits in L2
    assert d["roofline"]["read_only_peak_gbs"] > 1000 and d["phase_block"]["steps"] == 12
    ref = _run(["--impl", "reference"] + args)
    assert ref["config"] == d["config"]  # both arms run the same workload


@pytest.mark.gpu
@pytest.mark.parametrize("shard,launch", [("sequences", "torchrun"), ("slabs", "torchrun"),
                                          ("slabs", "self"), ("units", "torchrun"),
                                          ("batch", "torchrun")])
def test_two_rank_paths_run_end_to_end(shard, launch):
    """Functional check of the N>1 bench paths on one GPU: two ranks over gloo
    (HC_BENCH_BACKEND; the driver's runs use NCCL, one GPU per rank).  Slab and
    unit modes exercise the fire exchange and the all-gather of O; "self" is
    `bench.py --gpus 2` re-launching itself under torchrun.  The numbers of such
    a run are not measurements."""
    wl = ["--workload", "cfg3", "--layers", "2"] if shard == "batch" else \
        ["--workload", "cfg2", "--layers", "4"]
    d = _run(["--gpus", "2", "--shard", shard, *wl, "--steps", "16", "--warmup", "3",
              "--calib-samples", "2"],
             ranks=2 if launch == "torchrun" else 1, HC_BENCH_BACKEND="gloo")
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["scaling"] == ("weak" if shard == "sequences" else "strong")
    assert d["config"]["parallelism"].startswith(shard)
