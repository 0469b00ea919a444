"""Host-side timeline of the steps that take a boundary decision (overlapped mode).

For each step after a window boundary, the time the host spends in each part of
decode_step: decode_begin (launch K4 over the non-satellites), the overlap
readback (waits for the boundary step's monitor on the GPU), the Python
decision, fire_batch (fire selection + gather issue), landing and decode_end
(waits for the gathers the step lands).  With the GPU step time beside it this
shows which part of the fire -> gather -> landing chain is exposed.

    python tools/boundary_profile.py [workload=cfg4] [steps=120]
"""

import sys
import time
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_13684_b200.decoder import HeteroCacheDecoder  # noqa: E402
from paper_2601_13684_b200.engine import EngineConfig  # noqa: E402
from paper_2601_13684_b200.workload import (CONFIGS, SyntheticKV, decode_queries,  # noqa: E402
                                            plan_for, staggered_shifts)


class Timed:
    """Wraps a ctypes library: accumulates wall time per entry point."""

    def __init__(self, lib, names, log):
        self._lib, self._names, self._log = lib, set(names), log

    def __getattr__(self, name):
        fn = getattr(self._lib, name)
        if name not in self._names:
            return fn

        def call(*a):
            t0 = time.perf_counter()
            if name == "hc_engine_fire_batch" and "overlaps_end" in self._log:
                self._log["python_decision"] += t0 - self._log["overlaps_end"]
            r = fn(*a)
            t1 = time.perf_counter()
            self._log[name] += t1 - t0
            if name == "hc_engine_overlaps":
                self._log["overlaps_end"] = t1
            return r
        return call


def main(name="cfg4", K=120, W=5):
    w = CONFIGS[name]
    m = w.model
    tax, plan = plan_for(w)
    T = W + K + 2
    cfg = EngineConfig(tau_drift=0.5, window=8, update_delay_steps=1,
                       transfer_bandwidth=int(w.link_mib_per_step * (1 << 20)))
    dec = HeteroCacheDecoder(tax, plan, cfg, batch=w.batch, group=m.group, max_decode=T,
                             track_sets=False, obs_window=max(1, min(32, 128 // m.group)))
    gen = SyntheticKV(m, batch=w.batch, prefill_len=w.prefill_len, num_layers=w.num_layers,
                      hot=plan.l_base_int, seed=20261018 + 3)
    for l in range(w.num_layers):
        k, v, q = gen.layer_kv(l, dec.W)
        dec.prefill_layer(l, k, v, q)
        del k, v, q
    torch.cuda.synchronize()
    dec.finish_prefill()
    qs = decode_queries(gen, T, staggered_shifts(w.batch, w.num_layers, W + 1, K + 2,
                                                  w.shift_every))
    kn, vn = gen.step_inputs(100, None)[1:]
    out = torch.empty_like(qs[0])
    for t in range(1, W + 1):
        dec.decode_step(t, qs[t], kn, vn, out, rows=False)
    torch.cuda.synchronize()
    names = ["hc_engine_decode_begin", "hc_engine_overlaps", "hc_engine_fire_batch",
             "hc_engine_land_batch", "hc_engine_decode_end", "hc_engine_decode_step"]
    shown = names + ["python_decision"]
    per_step = []
    dec.kernel_timing(True)
    dec.retrieval_stats()
    real = dec.lib
    import cProfile
    import pstats
    prof = cProfile.Profile()
    for t in range(W + 1, W + K + 1):
        log = defaultdict(float)
        dec.lib = Timed(real, names, log)
        boundary_next = (t - 1) % 8 == 0
        if boundary_next and "--cprofile" in sys.argv:
            prof.enable()
        a = time.perf_counter()
        dec.decode_step(t, qs[t], kn, vn, out, rows=False)
        log["total"] = time.perf_counter() - a
        log.pop("overlaps_end", None)
        prof.disable()
        dec.lib = real
        per_step.append((t, dict(log)))
    if "--cprofile" in sys.argv:
        pstats.Stats(prof).sort_stats("tottime").print_stats(14)
    dec.finish()
    torch.cuda.synchronize()
    ph = dec.kernel_timing(False)
    rs = dec.retrieval_stats()
    after = [d for t, d in per_step if (t - 1) % 8 == 0]
    other = [d for t, d in per_step if (t - 1) % 8 != 0]

    def mean(ds, k):
        return 1e3 * float(np.mean([d.get(k, 0.0) for d in ds])) if ds else 0.0
    print(f"{name}: GPU step {ph['step'] / ph['steps']:.3f} ms (K4 {ph['attention'] / ph['steps']:.3f}),"
          f" landing stall {rs['landing_stall_ms'] / max(1, K):.3f} ms/step avg,"
          f" gathers {rs['gather_ms']:.1f} ms in {rs['batches']} batches")
    for label, ds in (("after boundary", after), ("other", other)):
        parts = ", ".join(f"{k.replace('hc_engine_', '')} {mean(ds, k):.3f}"
                          for k in shown + ["total"] if mean(ds, k) > 0)
        print(f"  {label} (n={len(ds)}) host ms: {parts}")
    dec.close()


if __name__ == "__main__":
    a = [x for x in sys.argv[1:] if not x.startswith("--")]
    main(a[0] if a else "cfg4", int(a[1]) if len(a) > 1 else 120)
