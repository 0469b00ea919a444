"""Time the REFERENCE engine (heterocache.engine.CacheEngine, pure Python, 1 core) on the
128K export of a GPU run (tests/golden/scale_128k): SURVEY 8d CPU baseline (i), the
reference's own decision + measure path per decode step.  Build container only (imports
/root/reference).

    python tools/time_reference_engine.py [out.json]
"""
import json, sys, time
import numpy as np
ROOT = __import__("pathlib").Path(__file__).resolve().parent.parent
sys.path[:0] = ["/root/reference/pkg/src", str(ROOT / "tests"), str(ROOT)]
from golden_io import key
from heterocache.budget import BudgetPlan
from heterocache.engine import CacheEngine, EngineConfig
from heterocache.profiling import Cluster, HeadProfile, TaxonomyResult
from heterocache.trace import TraceManifest, make_trace
D = str(ROOT / "tests/golden/scale_128k") + "/"
run = json.load(open(D + "scale_run.json"))
z = np.load(D + "scale_trace.npz")
tr = make_trace(TraceManifest(**run["manifest"]), z["indices"], z["scores"])
cid = {}
clusters = []
for i, (p, sats) in enumerate(run["clusters"]):
    clusters.append(Cluster(i, tuple(p), tuple(tuple(s) for s in sats)))
    for m in [tuple(p)] + [tuple(s) for s in sats]:
        cid[m] = i
heads = {key(h): HeadProfile(layer=key(h)[0], head=key(h)[1], s_stable=run["s_stable"][h], s_sim=0.0,
                             role=r, cluster_id=cid.get(key(h))) for h, r in run["roles"].items()}
m = run["manifest"]
tax = TaxonomyResult(num_layers=m["num_layers"], heads_per_layer=m["heads_per_layer"], tau_stable=0.5,
                     tau_sim=0.5, profiling_topk=None, heads=heads, clusters=tuple(clusters))
p = run["plan"]
plan = BudgetPlan(rho=p["rho"], prefill_len=p["prefill_len"], num_heads=p["num_heads"], num_full=p["num_full"],
                  num_comp=p["num_comp"], l_base=p["l_base"], l_base_int=p["l_base_int"],
                  lengths={key(h): n for h, n in p["lengths"].items()})
eng = CacheEngine(tr, tax, plan, EngineConfig(**run["config"]))
st = eng.prefill_init()
t0 = time.perf_counter()
T = m["decode_steps"]
for t in range(1, T + 1):
    eng.decode_step(st, t)
dt = (time.perf_counter() - t0) / T
res = {"reference_decode_step_ms": dt * 1e3, "layers": m["num_layers"], "kv_heads": m["heads_per_layer"],
                  "prefill_len": m["prefill_len"], "trace_topk": m["trace_topk"], "steps": T,
       "cfg3_scale": 28 * 4 / (m["num_layers"] * 1),
       "cfg3_steps_per_s": 1.0 / (dt * 28 * 4 / (m["num_layers"] * 1)), "cores": 1}
print(json.dumps(res))
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(json.dumps(res, indent=1) + "\n")
