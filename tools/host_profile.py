"""Host-side cost of the decode loop (where does the wall time go?)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

from paper_2601_13684_b200.decoder import HeteroCacheDecoder
from paper_2601_13684_b200.engine import EngineConfig
from paper_2601_13684_b200.workload import CONFIGS, SyntheticKV, plan_for

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
m = w.model
tax, plan = plan_for(w)
cfg = EngineConfig(window=8)
K = 200
dec = HeteroCacheDecoder(tax, plan, cfg, batch=w.batch, group=m.group, max_decode=K + 16,
                         track_sets=False)
gen = SyntheticKV(m, batch=w.batch, prefill_len=w.prefill_len, num_layers=w.num_layers,
                  hot=plan.l_base_int, seed=5)
for l in range(w.num_layers):
    k, v, q = gen.layer_kv(l)
    dec.prefill_layer(l, k, v, q)
torch.cuda.synchronize()
dec.finish_prefill()
pool = {ph: [gen.step_inputs(100 + 10 * ph + i, 0 if ph else None) for i in range(4)] for ph in (0, 1)}
out = torch.empty_like(pool[0][0][0])
host = {"boundary": [], "plain": []}
pr = cProfile.Profile()
torch.cuda.synchronize()
t0 = time.perf_counter()
pr.enable()
for t in range(1, K + 1):
    q, kn, vn = pool[(t // 100) % 2][t % 4]
    a = time.perf_counter()
    dec.decode_step(t, q, kn, vn, out, rows=False)
    host["boundary" if t % 8 == 0 else "plain"].append(time.perf_counter() - a)
pr.disable()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"wall per step {wall / K * 1e3:.3f} ms")
for k, v in host.items():
    print(f"{k}: n={len(v)} mean host {sum(v) / len(v) * 1e3:.3f} ms max {max(v) * 1e3:.3f} ms")
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
