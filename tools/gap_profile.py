"""Where does the inter-step idle time go?  (per-step gaps by step type)"""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2601_13684_b200.decoder import HeteroCacheDecoder
from paper_2601_13684_b200.engine import EngineConfig
from paper_2601_13684_b200.workload import CONFIGS, SyntheticKV, plan_for

w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
m = w.model
tax, plan = plan_for(w)
cfg = EngineConfig(window=8, transfer_bandwidth=64 << 20)
K = 300
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
dec.kernel_timing(True)
host = []
for t in range(1, K + 1):
    q, kn, vn = pool[(t // 100) % 2][t % 4]
    a = time.perf_counter()
    dec.decode_step(t, q, kn, vn, out, rows=False)
    host.append(time.perf_counter() - a)
torch.cuda.synchronize()
gaps = np.zeros(K, dtype=np.float32)
n = C.c_int32()
dec.lib.hc_engine_gaps(dec.handle, gaps.ctypes.data, K, C.byref(n))
gaps = gaps[:n.value]  # gaps[i] = idle before step i+2
steps = np.arange(2, n.value + 2)
after_boundary = (steps - 1) % 8 == 0
flip_region = np.array([(s % 100) < 4 for s in steps])
print("mean gap all %.3f ms" % gaps.mean())
print("after boundary: n=%d mean %.3f ms" % (after_boundary.sum(), gaps[after_boundary].mean()))
print("other: n=%d mean %.3f ms" % ((~after_boundary).sum(), gaps[~after_boundary].mean()))
print("largest gaps:", sorted(zip(gaps.round(3).tolist(), steps.tolist()))[-12:])
host = np.array(host) * 1e3
print("host ms per call: boundary %.3f other %.3f" % (host[7::8].mean(), np.delete(host, np.s_[7::8]).mean()))
