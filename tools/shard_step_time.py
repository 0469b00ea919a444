"""Per-GPU step time of a unit shard, measured on ONE B200.

For N in 1, 2, 4, 8: bin-pack the workload's (sequence, layer, cluster-or-
loner) units over N ranks (parallel.assign_units), build the engine of the
most loaded rank only (hc_engine_create_sharded) and time its decode steps
with CUDA events, exactly as bench.py's device-resident loop does.  This is
the compute side of a strong-scaling run -- what one GPU of an N-GPU job
executes per step -- and NOT a multi-GPU measurement: the fire exchange (a
gloo all_gather of a few bytes per firing pivot at window boundaries, beside
the attention) and the NCCL all-gather of O are not in it, and fires are
accounted over this shard alone (LocalExchange), which changes completion
steps but not the work per step.

    python tools/shard_step_time.py [workload=cfg5] [steps=60] [out.json]
"""

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_13684_b200.decoder import HeteroCacheDecoder  # noqa: E402
from paper_2601_13684_b200.engine import EngineConfig  # noqa: E402
from paper_2601_13684_b200.parallel import assign_units, shard_units  # noqa: E402
from paper_2601_13684_b200.workload import (CONFIGS, SyntheticKV, algorithmic_bytes,  # noqa: E402
                                            decode_queries, plan_for, staggered_shifts)


def shard_time(w, tax, plan, world, K, W=5):
    m = w.model
    T = W + K + 2
    owned_all = assign_units(tax, plan, w.batch, world, T)
    units = shard_units(tax, plan, w.batch, T)
    load = np.zeros(world)
    for b, _, members, wt in units:
        load[int(np.flatnonzero(owned_all[:, b, members[0][0], members[0][1]])[0])] += wt
    r = int(load.argmax())
    cfg = EngineConfig(tau_drift=0.5, window=8, update_delay_steps=1,
                       transfer_bandwidth=int(w.link_mib_per_step * (1 << 20)))
    obs = max(1, min(32, 128 // m.group))
    dec = HeteroCacheDecoder(tax, plan, cfg, batch=w.batch, group=m.group, max_decode=T,
                             chunk=1024, track_sets=False, obs_window=obs,
                             owned=None if world == 1 else owned_all[r])
    gen = SyntheticKV(m, batch=w.batch, prefill_len=w.prefill_len, num_layers=w.num_layers,
                      hot=plan.l_base_int, seed=20261018 + 5)
    for l in range(w.num_layers):
        k, v, q = gen.layer_kv(l, obs)
        dec.prefill_layer(l, k, v, q)
        del k, v, q
    torch.cuda.synchronize()
    dec.finish_prefill()
    qs = decode_queries(gen, T, staggered_shifts(w.batch, w.num_layers, W + 1, K + 2))
    kn, vn = gen.step_inputs(100, None)[1:]
    out = torch.empty_like(qs[0])
    for t in range(1, W + 1):
        dec.decode_step(t, qs[t], kn, vn, out, rows=False)
    torch.cuda.synchronize()
    rows0 = dec.resident_rows(W + 1)
    dec.kernel_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(W + 1, W + K + 1):
        dec.decode_step(t, qs[t], kn, vn, out, rows=False)
    dec.join()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    ph = dec.kernel_timing(False)
    rows1 = dec.resident_rows(W + K)
    q_heads = int(dec.owned.sum()) * m.group
    bytes_ = algorithmic_bytes(int((rows0 + rows1) / 2), 1, 1, q_heads)
    k4 = ph["attention"] / max(1, ph["steps"])
    res = {"gpus": world, "rank_timed": r, "load_share": float(load[r] / load.sum()),
           "ms_per_step": ms, "k4_ms": k4, "shard_bytes_per_step": bytes_,
           "shard_hbm_gbs": bytes_ / (ms * 1e-3) / 1e9,
           "k4_gbs": bytes_ / (k4 * 1e-3) / 1e9 if k4 else None,
           "units": int(dec.owned.sum()), "device_bytes": dec.device_bytes}
    dec.close()
    del qs
    torch.cuda.empty_cache()
    return res


def main(name="cfg5", K=60, out=None):
    w = CONFIGS[name]
    tax, plan = plan_for(w)
    rows = []
    for world in (1, 2, 4, 8):
        t0 = time.time()
        r = shard_time(w, tax, plan, world, K)
        r["wall_s"] = time.time() - t0
        print(json.dumps(r), flush=True)
        rows.append(r)
    base = rows[0]["ms_per_step"]
    summary = {"workload": name, "steps": K, "note": __doc__.split("\n\n")[1].replace("\n", " "),
               "shards": rows,
               "projected_strong_speedup": {str(r["gpus"]): base / r["ms_per_step"] for r in rows}}
    if out:
        Path(out).write_text(json.dumps(summary, indent=1) + "\n")
    print(json.dumps(summary["projected_strong_speedup"]))


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "cfg5", int(a[1]) if len(a) > 1 else 60, a[2] if len(a) > 2 else None)
