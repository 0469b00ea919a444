"""Selection precision and output parity at 128K / 224K (round-2 evidence).

    python tools/selection_precision.py [--shapes cfg3,cfg5] [--materials fp32,fp16]
                                        [--out gpurun_out/selection_precision.json]

For each shape (tests/scale_parity.SHAPES) and pivot score material, decodes
T steps across a planted topic shift and reports: O / pivot-row error against
the fp32 oracle over the resident sets, the event log vs the oracle replay of
the GPU rows, and per-step top-k set differences between the GPU rows and the
oracle's fp32 / fp64 rows over the same K/V/Q (scale_parity.selection_precision).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import scale_parity as SP  # noqa: E402

LAYOUT = {"cfg3": dict(B=2, NL=2), "cfg5": dict(B=1, NL=1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="cfg3,cfg5")
    ap.add_argument("--materials", default="fp32,fp16")
    ap.add_argument("--T", type=int, default=24)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "selection_precision.json"))
    a = ap.parse_args()
    import torch

    torch.set_num_threads(max(1, (__import__("os").cpu_count() or 1)))
    res = []
    for shape in a.shapes.split(","):
        for mat in a.materials.split(","):
            t0 = time.time()
            ctx = SP.build(shape, T=a.T, score_material=mat, **LAYOUT[shape])
            SP.run(ctx)
            t_gpu = time.time() - t0
            events = SP.check_events(ctx)
            lands = sorted({e["completion_step"] for _, e in events if e["completion_step"] <= a.T})
            steps = sorted({1, 8, a.T} | set(lands))
            out = SP.check_outputs(ctx, steps)
            sel = SP.selection_precision(ctx)
            rec = dict(shape=shape, material=mat, L=ctx["L"], B=ctx["B"], NL=ctx["NL"], T=a.T,
                       l_base_int=ctx["plan"].l_base_int,
                       events=[dict(seq=b, trigger=e["trigger_step"], pivot=e["pivot"],
                                    completion=e["completion_step"]) for b, e in events],
                       checked_steps=steps, outputs=out, selection=SP.summarise(sel),
                       selection_nonzero=[x for x in sel if x["gpu_vs_fp32"] or x["fp32_vs_fp64"]
                                          or x["gpu_vs_fp64"]][:200],
                       seconds=dict(gpu=t_gpu, total=time.time() - t0))
            print(json.dumps({k: rec[k] for k in ("shape", "material", "outputs", "selection")}),
                  flush=True)
            res.append(rec)
            ctx["dec"].close()
            del ctx
            torch.cuda.empty_cache()
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
