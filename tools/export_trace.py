"""Export a tensor-mode GPU run as an HCTRACE1 trace.

Runs on the GPU box: a 128K-context Qwen2.5-7B-shaped decode (2 layers,
batch 1, observation window 1 = the reference's step-0 semantics) with a
planted topic shift, in measure mode, then writes

  <out>/scale_trace.npz   trace arrays: per-step records of every head -- the
                          engine's measure-mode records (step 0 and pivots:
                          top-max(l_base_int, l_h) -- pivots from their own
                          decision rows; other heads: top-1024 of their dense
                          GPU rows) in HCTRACE1 order, PAD tail
  <out>/scale_run.json    manifest, roles/clusters/plan/config and the GPU
                          engine's event log and StepRows (recall included)

tests/test_scale_replay.py replays the trace through the reference engine
(heterocache.engine.CacheEngine, when /root/reference is present) and the
pinned oracle, which must reproduce the GPU event log exactly: selection
parity closed at 128K context.
"""

import json
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2601_13684_b200.decoder import HeteroCacheDecoder  # noqa: E402
from paper_2601_13684_b200.engine import EngineConfig  # noqa: E402
from paper_2601_13684_b200.trace import PAD_INDEX  # noqa: E402
from paper_2601_13684_b200.workload import CONFIGS, SyntheticKV, plan_for  # noqa: E402


def main(out_dir: str, T: int = 16, shift: int = 7):
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    w = replace(CONFIGS["cfg3"], layers=2, batch=1)
    m = w.model
    tax, plan = plan_for(w)
    cfg = EngineConfig(tau_drift=0.5, window=4, update_delay_steps=1,
                       transfer_bandwidth=64 << 20)
    L, NL, H, G = w.prefill_len, w.num_layers, m.kv_heads, m.group
    dec = HeteroCacheDecoder(tax, plan, cfg, batch=1, group=G, max_decode=T, obs_window=1,
                             recall_topk=1024)
    gen = SyntheticKV(m, batch=1, prefill_len=L, num_layers=NL, hot=plan.l_base_int, seed=77)
    for l in range(NL):
        k, v, q = gen.layer_kv(l)
        dec.prefill_layer(l, k, v, q)
    torch.cuda.synchronize()
    dec.finish_prefill()
    K = dec.record_k
    idx = np.full((T + 1, NL, H, K), PAD_INDEX, dtype=np.uint32)
    sc = np.zeros((T + 1, NL, H, K), dtype=np.float32)

    def grab(t):
        for l in range(NL):
            for h in range(H):
                idx[t, l, h], sc[t, l, h] = dec.measure_records(0, (l, h))

    grab(0)
    for t in range(1, T + 1):
        q, kn, vn = gen.step_inputs(t, shift)
        o = torch.empty_like(q)
        dec.decode_step(t, q, kn, vn, o)
        grab(t)
    dec.sync()
    st = dec.states[0]
    np.savez_compressed(out / "scale_trace.npz", indices=idx, scores=sc)
    run = {
        "manifest": {"model_name": "qwen2.5-7b-128k-2layer-gpu", "num_layers": NL,
                     "heads_per_layer": H, "prefill_len": L, "decode_steps": T,
                     "trace_topk": K, "pool_kernel_used": 0, "bytes_per_kv_entry": 512},
        "roles": {f"{l},{h}": p.role for (l, h), p in tax.heads.items()},
        "s_stable": {f"{l},{h}": p.s_stable for (l, h), p in tax.heads.items()},
        "clusters": [[list(c.pivot), [list(s) for s in c.satellites]] for c in tax.clusters],
        "plan": {"rho": plan.rho, "prefill_len": plan.prefill_len, "num_heads": plan.num_heads,
                 "num_full": plan.num_full, "num_comp": plan.num_comp, "l_base": plan.l_base,
                 "l_base_int": plan.l_base_int,
                 "lengths": {f"{l},{h}": n for (l, h), n in plan.lengths.items()}},
        "config": {"tau_drift": cfg.tau_drift, "window": cfg.window,
                   "transfer_bandwidth": cfg.transfer_bandwidth,
                   "update_delay_steps": cfg.update_delay_steps, "sink_count": cfg.sink_count,
                   "recency_window": cfg.recency_window, "variant": cfg.variant,
                   "eval_every_step": cfg.eval_every_step},
        "gpu_events": [e.to_json_dict() for e in st.events],
        "gpu_rows": [r.to_json_dict() for r in st.rows],
        "gpu_dynamic": {f"{l},{h}": dec.dynamic_set(0, (l, h)).tolist() for (l, h) in dec.comp},
    }
    (out / "scale_run.json").write_text(json.dumps(run))
    print(f"exported T={T} K={K} events={len(st.events)}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/scale")
