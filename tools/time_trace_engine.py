"""Time this package's trace-mode CacheEngine (GPU) on the 128K export of a GPU run
(tests/golden/scale_128k) -- the drop-in for heterocache.engine.CacheEngine -- and check
that it reproduces the GPU tensor-mode StepRows and events recorded in the fixture.

    python tools/time_trace_engine.py [out.json]
"""

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

from golden_io import key  # noqa: E402
from paper_2601_13684_b200.budget import BudgetPlan  # noqa: E402
from paper_2601_13684_b200.engine import CacheEngine, EngineConfig  # noqa: E402
from paper_2601_13684_b200.profiling import taxonomy_from_roles  # noqa: E402
from paper_2601_13684_b200.trace import TraceManifest, make_trace  # noqa: E402


def main(out=None):
    D = ROOT / "tests/golden/scale_128k"
    run = json.loads((D / "scale_run.json").read_text())
    with np.load(D / "scale_trace.npz") as z:
        tr = make_trace(TraceManifest(**run["manifest"]), z["indices"], z["scores"])
    m = run["manifest"]
    tax = taxonomy_from_roles({key(h): r for h, r in run["roles"].items()},
                              [(tuple(p), [tuple(s) for s in sats]) for p, sats in run["clusters"]],
                              num_layers=m["num_layers"], heads_per_layer=m["heads_per_layer"],
                              s_stable={key(h): v for h, v in run["s_stable"].items()})
    p = run["plan"]
    plan = BudgetPlan(rho=p["rho"], prefill_len=p["prefill_len"], num_heads=p["num_heads"],
                      num_full=p["num_full"], num_comp=p["num_comp"], l_base=p["l_base"],
                      l_base_int=p["l_base_int"],
                      lengths={key(h): n for h, n in p["lengths"].items()})
    eng = CacheEngine(tr, tax, plan, EngineConfig(**run["config"]))
    st = eng.prefill_init()
    eng.decode_step(st, 1)  # warm-up (device upload, first launches)
    eng = CacheEngine(tr, tax, plan, EngineConfig(**run["config"]))
    st = eng.prefill_init()
    rows = [eng._measure(st, 0)]
    T = m["decode_steps"]
    t0 = time.perf_counter()
    got = [eng.decode_step(st, t) for t in range(1, T + 1)]
    dt = (time.perf_counter() - t0) / T
    same = [r.to_json_dict() for r in got] == run["gpu_rows"][1:]
    res = {"trace_engine_decode_step_ms": dt * 1e3, "steps": T, "layers": m["num_layers"],
           "kv_heads": m["heads_per_layer"], "prefill_len": m["prefill_len"],
           "trace_topk": m["trace_topk"], "rows_identical_to_tensor_mode": same}
    print(json.dumps(res))
    if out:
        Path(out).write_text(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
