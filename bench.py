#!/usr/bin/env python
"""HeteroCache-B200 decode hot-path benchmark (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload cfg5] [--secondary cfg3|none]

A "step" is one decode step of the workload's whole batch through the
reference-facing API (HeteroCacheDecoder.decode_step, the tensor-mode
CacheEngine.decode_step): append the token's K/V, fused ragged attention for
every head of every layer over its resident set, pivot score rows, K1
top-l_base + K2 overlap, and -- at window boundaries -- the drift test, fetch
selection and host-pool retrieval on the side stream.

Default workload: cfg5 (Llama-3.1-8B-shaped, 224K context, batch 8, 10%
budget, "sharded by (batch, KV-head) across 1/2/4/8 B200 with prefill
scoring/profiling included"), with head roles and budgets from synthetic
profiling (calibration.py: measure-mode decodes -> run_taxonomy ->
plan_budget) inside setup.  At N=1 a `secondary` block carries cfg3
(Qwen2.5-7B-shaped, 128K, batch 4) measured the same way in a child process.

N>1: `python bench.py --gpus N` re-launches itself under torchrun (one rank per
GPU) when WORLD_SIZE is unset.  Default sharding: slabs of ONE batch -- rank r
owns (sequence, layer) pairs [r*S, (r+1)*S) (parallel.slab_units; strong
scaling): boundary fires are exchanged with one fixed-size NCCL all-gather on
a side stream beside the attention (parallel.TensorFireExchange, completion
steps stay the reference's), and the e2e loop all-gathers O in place.
--shard sequences runs independent batches per rank (weak).

Measurement: warm-up W steps, then K device-timed steps with inputs resident
(`value`), then K end-to-end steps with every step's Q/K/V H2D from pinned
host memory and O D2H inside the timed region (`e2e`), both loops with the
same instrumentation.  `cpu_baseline` (N=1, rank 0) and `parity`: the CPU
decoder oracle (oracle/cpu_decoder.py) decodes a sample of sequences on the
same seeded inputs (oracle/synth.c reproduces the GPU generator bit for bit)
-- prefill selection, attention, drift monitor, fires, landings -- timed on
the host cores, and its outputs / events at a step after the first landing
are compared with the GPU's.

--impl reference: the same CPU decoder (and the CPU restatement of the
profiling) on the host cores, W + K steps on a sample of the workload's
sequences, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode attn steps/sec & HBM GB/s @128K/224K ctx, 1/2/4/8 B200 vs host-CPU ref"
# process-group backend of a multi-rank run: NCCL (one GPU per rank).  gloo is
# only for functional tests of the multi-rank paths on a single GPU
# (tests/test_bench_contract.py): its numbers are not measurements.
BACKEND = os.environ.get("HC_BENCH_BACKEND", "nccl")
COLL_DEV = "cuda" if BACKEND == "nccl" else "cpu"
FALLBACK_HBM_GBS = 6650.0
SEED_BASE = 20261018
O_ATOL, O_RTOL = 4e-3, 1e-2  # stated output tolerance (tests/scale_parity.py)
PARITY_STEP = 18             # first step after the first fires (boundary 16) land


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", default="cfg5")
    ap.add_argument("--secondary", default="cfg3",
                    help="N=1: a second workload measured in a child process ('none': skip)")
    ap.add_argument("--layers", type=int, default=0, help="override layer count (debug)")
    ap.add_argument("--batch", type=int, default=0,
                    help="override the batch (e.g. one rank's share of a batch-sharded run)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seqs", type=int, default=1,
                    help="sequences the CPU decoder samples (cpu_baseline, parity, reference)")
    ap.add_argument("--chunk", type=int, default=0,
                    help="split-K chunk (rows per K4 tile); 0: 1024, smaller for a step too "
                         "small to fill the GPU with 1024-row tiles")
    ap.add_argument("--l2", choices=("auto", "flush", "none"), default="auto",
                    help="flush L2 between timed steps (auto: when a step's resident K/V "
                         "would fit in 4x L2), timing each step on its own")
    ap.add_argument("--start-step", type=int, default=0,
                    help="decode this many steps untimed before warm-up (e.g. cfg4 at t = 8K)")
    ap.add_argument("--policy", choices=("heterocache", "full", "static_topk", "sink_window"),
                    default="heterocache",
                    help="baseline residency policies through the same engine (evaluation.py): "
                         "full = FullAttention (every head keeps its whole cache); static_topk / "
                         "sink_window at the heterocache plan's budget rho")
    ap.add_argument("--roles", choices=("profiled", "fixed"), default="profiled",
                    help="profiled: synthetic profiling in setup (run_taxonomy + plan_budget); "
                         "fixed: the survey's role mix with preset stabilities")
    ap.add_argument("--calib-samples", type=int, default=4)
    ap.add_argument("--calib-len", type=int, default=4096)
    ap.add_argument("--calib-steps", type=int, default=16)
    ap.add_argument("--obs-window", type=int, default=0,
                    help="prefill observation window (0: min(32, 128 // G))")
    ap.add_argument("--shard", choices=("auto", "batch", "slabs", "units", "sequences"),
                    default="auto",
                    help="N>1, one batch split over the ranks (strong): batch = whole sequences "
                         "per rank (auto when the batch divides), slabs = contiguous (sequence, "
                         "layer) ranges, units = bin-packed (sequence, layer, cluster) units; "
                         "sequences = every rank its own batch (weak)")
    ap.add_argument("--score-material", choices=("fp32", "fp16"), default="fp32",
                    help="pivot score material between K4 and the GQA-mean rows")
    ap.add_argument("--decisions", choices=("device", "host"), default="device",
                    help="boundary decisions on the device (devdec.cu; default where supported) "
                         "or on the host")
    ap.add_argument("--link-mib-per-step", type=float, default=0.0,
                    help="EngineConfig.transfer_bandwidth in MiB per decode step (host link "
                         "model); 0: the workload's measured-link value")
    return ap.parse_args(argv)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)", {}


def read_probe(gib: int = 4) -> dict:
    """Live read-only HBM bandwidth (hc_read_probe over a buffer larger than L2).

    The copy peak in MEASURED_PEAKS.json moves read+write traffic; K4 reads
    K/V and writes almost nothing, so it can exceed that figure.  This is the
    read-only ceiling measured on the same box, best over grid sizes and
    repetitions, timed with CUDA events on the launching stream."""
    import torch

    from paper_2601_13684_b200 import _lib

    lib = _lib.load()
    nbytes = gib << 30
    buf = torch.ones(nbytes // 4, dtype=torch.int32, device="cuda")
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    sink = torch.empty(sm * 32, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()
    best = {}
    for per_sm in (4, 8, 16, 32):
        ms = []
        for _ in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            rc = lib.hc_read_probe(buf.data_ptr(), nbytes, sink.data_ptr(), sm * per_sm,
                                   st.cuda_stream)
            b.record(st)
            if rc != 0:
                raise RuntimeError(lib.hc_last_error().decode())
            b.synchronize()
            ms.append(a.elapsed_time(b))
        best[per_sm] = nbytes / (min(ms[1:]) * 1e-3) / 1e9
    del buf, sink
    torch.cuda.empty_cache()
    per_sm = max(best, key=best.get)
    return {"gbs": best[per_sm], "bytes": nbytes, "ctas_per_sm": per_sm,
            "by_ctas_per_sm": {str(k): round(v, 1) for k, v in best.items()}}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.out, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.2)
        self.proc.terminate()
        self.proc.wait()
        self.out.flush()
        lines = [l.split(",") for l in Path(self.out.name).read_text().splitlines() if l.strip()]
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for f in lines:
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
                for n, v in zip(names, f[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# workload description shared by both arms
# ---------------------------------------------------------------------------


def workload_of(args):
    from dataclasses import replace

    from paper_2601_13684_b200.workload import CONFIGS

    w = CONFIGS[args.workload]
    if args.layers:
        w = replace(w, layers=args.layers)
    if args.batch:
        w = replace(w, batch=args.batch)
    return w


def seed_of(args) -> int:
    return SEED_BASE + int(args.workload[3:])


def hot_of(w) -> int:
    """Planted hot-set size: the base budget c * L (the data do not depend on
    the profiled plan, so both arms generate the same inputs)."""
    return max(1, int(round(w.compression * w.prefill_len)))


def obs_of(args, w) -> int:
    return args.obs_window or max(1, min(32, 128 // w.model.group))  # w_obs = 32


def schedule(args, w):
    """(shift steps per (sequence, layer), T capacity, first timed step - 1)."""
    from paper_2601_13684_b200.workload import staggered_shifts

    K, W, S0 = args.steps, args.warmup, args.start_step
    Z = settle_steps(w)
    shifts = staggered_shifts(w.batch, w.num_layers, S0 + W + 1, Z + 2 * K + 8, w.shift_every)
    if S0:  # the fast-forward drifts too
        pre = staggered_shifts(w.batch, w.num_layers, 1, S0 + W, w.shift_every)
        shifts = {key: pre[key] + shifts[key] for key in shifts}
    return shifts, S0 + W + Z + 2 * K + 8 + phase_steps(args)


def chunk_of(args, w) -> int:
    """The split-K chunk: 1024 rows, halved (down to 128) while the full-context
    tiles of one step would not give every SM four (cfg1: 32 tiles at 1024)."""
    if args.chunk:
        return args.chunk
    chunk = 1024
    units = w.batch * w.num_layers * w.model.kv_heads
    while chunk > 128 and units * -(-w.prefill_len // chunk) < 4 * 148:
        chunk //= 2
    return chunk


def settle_steps(w) -> int:
    """Untimed steps after the warm-up with the drift schedule already running, for
    workloads that drift every few steps (cfg4): eight drift periods, so the timed
    region starts in the steady state of fires, gathers and landings rather than
    at the schedule's first burst.  0 for the one-shift-per-run workloads."""
    return 8 * w.shift_every if 0 < w.shift_every <= 32 else 0


def phase_steps(args) -> int:
    """Steps of the instrumented block after the timed region (every phase event)."""
    return min(args.steps, 64)


def engine_config(args, w):
    from paper_2601_13684_b200.engine import EngineConfig

    return EngineConfig(tau_drift=0.5, window=8, update_delay_steps=1,
                        transfer_bandwidth=int((args.link_mib_per_step or w.link_mib_per_step)
                                               * (1 << 20)))


def shard_mode(args, w, world: int) -> str:
    """replicas (N=1), sequences (weak), slabs or units (strong) -- both arms."""
    if world == 1:
        return "replicas"
    mode = args.shard
    if mode == "auto":  # whole sequences of the batch per rank when they split evenly
        mode = "batch" if w.batch % world == 0 else "slabs"
    if mode == "batch" and w.batch % world:
        mode = "slabs"
    if mode == "slabs" and (w.batch * w.num_layers) % world:
        mode = "units"  # (sequence, layer) pairs do not split evenly: bin-pack clusters
    return mode


def scaling_of(args, mode: str) -> str:
    """strong: one batch whatever N (N=1 included, unless --shard sequences asks
    for a batch per rank); weak: every rank decodes its own batch."""
    if mode == "sequences" or (mode == "replicas" and args.shard == "sequences"):
        return "weak"
    return "strong"


def calib_spec(args):
    from paper_2601_13684_b200.calibration import CalibSpec

    return CalibSpec(samples=args.calib_samples, prefill_len=args.calib_len,
                     steps=args.calib_steps)


def layer_mixes(roles: dict, NL: int, H: int) -> dict:
    mixes = {}
    for l in range(NL):
        key = ",".join(roles[(l, h)] for h in range(H))
        mixes[key] = mixes.get(key, 0) + 1
    return mixes


L2_BYTES = 126 << 20  # B200 L2


def l2_flush(args, w, rho: float, world: int) -> bool:
    """Whether the timed steps run with an L2 flush between them: a step whose
    resident K/V (about rho of the full context at 512 B per token and KV head)
    fits in 4x L2 would otherwise be served from L2 on every step."""
    if args.l2 == "none" or world > 1 or args.policy != "heterocache":
        return False
    return args.l2 == "flush" or l2_resident_bytes(w, rho) < 4 * L2_BYTES


def l2_resident_bytes(w, rho: float) -> float:
    """About a step's resident K/V: rho of the full context, 512 B per token and KV head."""
    return w.batch * w.num_layers * w.model.kv_heads * w.prefill_len * 512 * rho


def make_config(args, w, cfg, rho, l_base_int, roles: dict, world: int, mode: str) -> dict:
    """The `config` object of both arms' lines (identical for the same run)."""
    from paper_2601_13684_b200.workload import DRIFT_PERIOD

    m = w.model
    par = {"replicas": "one GPU: the whole batch (the N=1 point of the batch-sharded series: "
                       "--gpus N splits this batch's sequences over N ranks)",
           "sequences": f"sequences x{world} (weak: each GPU decodes its own batch)",
           "batch": f"batch x{world} (strong: rank r decodes sequences [r*B/N, (r+1)*B/N) of "
                    f"one batch, decisions on its device, no exchange; O all-gathered in place)",
           "slabs": f"slabs x{world} (strong: rank r owns (sequence, layer) pairs "
                    f"[r*S, (r+1)*S) of one batch; NCCL fire exchange at boundaries, "
                    f"O all-gathered in place)",
           "units": f"units x{world} (strong: one batch's (sequence, layer, cluster) units "
                    f"bin-packed over the GPUs; NCCL fire exchange, O all-gather)"}[mode]
    return {
        "workload": f"{args.workload}: {w.name} ({m.name}-shaped, {w.num_layers} layers, "
                    f"{m.q_heads}q/{m.kv_heads}kv, d={m.head_dim})",
        "prefill_len": w.prefill_len, "global_batch": w.batch, "layers": w.num_layers,
        "compression": w.compression, "rho": rho, "l_base_int": l_base_int,
        "roles": ("profiled (run_taxonomy over synthetic calibration decodes)"
                  if args.roles == "profiled" else "fixed survey mix"),
        "layer_role_mixes": layer_mixes(roles, w.num_layers, m.kv_heads),
        "policy": args.policy, "decode_window": cfg.window, "tau_drift": cfg.tau_drift,
        "topic_shifts": (f"every cluster (sequence, layer) once per "
                         f"{w.shift_every or DRIFT_PERIOD} steps, staggered phases"),
        "split_k_chunk": chunk_of(args, w), "start_step": args.start_step,
        "settle_steps": settle_steps(w),
        "transfer_bandwidth_bytes_per_step": cfg.transfer_bandwidth,
        "score_material": args.score_material,
        "decisions": args.decisions,
        "l2": (f"flushed between timed steps ({2 * L2_BYTES >> 20} MB written; each step "
               f"timed on its own, start to end of its monitor, flush excluded)"
               if l2_flush(args, w, rho, world) else
               "inputs larger than L2 (resident K/V per step >> 126 MB)"
               if l2_resident_bytes(w, rho) >= 4 * L2_BYTES else
               "resident K/V per step fits in L2 and is not flushed (--l2 none, N > 1 or a "
               "baseline policy)"),
        "parallelism": par,
    }


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def gpu_plan(args, w):
    """(taxonomy, plan, profiling info) of the workload; profiled by default."""
    from paper_2601_13684_b200.workload import plan_for, rho_for

    if args.roles == "fixed":
        tax, plan = plan_for(w)
        return tax, plan, {"source": "fixed survey mix", "rho": rho_for(w.model, w.compression)}
    from paper_2601_13684_b200.calibration import calibrate

    t0 = time.time()
    tax, plan, info = calibrate(w.model, w.num_layers, w.compression, w.prefill_len,
                                calib_spec(args))
    info["profiling_s"] = time.time() - t0
    return tax, plan, info


def run_b200(args, rank, world):
    import torch

    from paper_2601_13684_b200 import _lib
    from paper_2601_13684_b200.decoder import HeteroCacheDecoder
    from paper_2601_13684_b200.workload import (SyntheticKV, algorithmic_bytes, decode_queries,
                                                plan_for)

    w = workload_of(args)
    m = w.model
    K, W, S0 = args.steps, args.warmup, args.start_step
    htax, hplan, prof = gpu_plan(args, w)
    if args.policy == "heterocache":
        tax, plan = htax, hplan
    elif args.policy == "full":
        tax, plan = plan_for(w, "full")
    else:
        tax, plan = None, None
    shifts, T = schedule(args, w)
    cfg = engine_config(args, w)
    lib = _lib.load()
    obs = obs_of(args, w)
    dkw = dict(batch=w.batch, group=m.group, max_decode=T, chunk=chunk_of(args, w), host_pool=True,
               track_sets=False, obs_window=obs, score_material=args.score_material,
               device_decisions=None if args.decisions == "device" else False)
    mode = shard_mode(args, w, world)
    owned_all = None
    Bl, seqs = w.batch, None  # sequences this rank decodes
    if mode == "batch":
        Bl = w.batch // world
        seqs = list(range(rank * Bl, (rank + 1) * Bl))
        dkw.update(batch=Bl)
    if mode in ("slabs", "units"):
        import torch.distributed as dist

        from paper_2601_13684_b200.parallel import TensorFireExchange, assign_units, slab_units

        if plan is None:
            raise SystemExit("--shard slabs/units support the heterocache and full policies")
        owned_all = slab_units(tax, w.batch, world) if mode == "slabs" else \
            assign_units(tax, plan, w.batch, world, T)
        n_piv = int(sum(owned_all[rank][b][p] for b in range(w.batch) for p in tax.pivots()))
        dkw.update(owned=owned_all[rank], exchange=TensorFireExchange(max(1, n_piv)))
    if plan is None:  # static baseline policy at the heterocache budget (evaluation.py:198-228)
        from paper_2601_13684_b200.evaluation import PolicySpec, policy_decoder

        dec = policy_decoder(PolicySpec(args.policy, rho=hplan.rho), num_layers=w.num_layers,
                             heads_per_layer=m.kv_heads, prefill_len=w.prefill_len,
                             engine_config=cfg, **dkw)
        tax, plan = dec.taxonomy, dec.plan
    else:
        dec = HeteroCacheDecoder(tax, plan, cfg, **dkw)
    seed = seed_of(args) + (rank if mode == "sequences" else 0)
    gen = SyntheticKV(m, batch=w.batch, prefill_len=w.prefill_len, num_layers=w.num_layers,
                      hot=hot_of(w), seed=seed, seqs=seqs)
    t0 = time.time()
    for l in range(w.num_layers):
        k, v, q = gen.layer_kv(l, obs)
        dec.prefill_layer(l, k, v, q)
        del k, v, q
    torch.cuda.synchronize()
    dec.finish_prefill()
    prefill_s = time.time() - t0
    pst = dec.prefill_stats()
    # K5 per layer: K read twice (two passes), 2*M*N*K flops per 128x128x128 tile and pass
    units_l = w.batch * m.kv_heads
    passes_k = 1 if obs * m.group <= 16 else 2  # small windows read K once (raw scores kept)
    score_bytes = passes_k * units_l * w.prefill_len * m.head_dim * 2
    score_flops = passes_k * 2 * units_l * ((w.prefill_len + 127) // 128 * 128) * 128 * m.head_dim
    score_ms = pst["score_ms"] / max(1, pst["layers"])
    qs = decode_queries(gen, T, shifts)
    kv_pool = [gen.step_inputs(100 + i, None)[1:] for i in range(4)]

    def inputs(t):
        return (qs[t],) + kv_pool[t % 4]

    out = torch.empty_like(qs[0])
    par_out = torch.empty_like(out)
    t_par = min(S0 + W + K, PARITY_STEP) if S0 == 0 else -1
    stream = torch.cuda.current_stream()
    t = 0
    for _ in range(S0 + W + settle_steps(w)):  # warm-up (+ the drift schedule's first periods)
        t += 1
        dec.decode_step(t, *inputs(t), par_out if t == t_par else out, rows=False)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # ---- timed region ----
    # loop A: inputs resident on the device (`value`); loop B: end to end through
    # the API, every step's Q / K_new / V_new H2D from pinned host memory and its
    # O D2H (`e2e`).  They run interleaved, A1 B1 B2 A2 (halves of K each), so
    # both measure the same stretch of the run -- the same drift events and
    # landings -- with the same instrumentation.
    halves = [K // 2, K - K // 2]
    t_start = t
    hq_all = qs[t + 1:t + 2 * K + 1].cpu().pin_memory()  # step s: hq_all[s - t_start - 1]
    hkv = [[x.cpu().pin_memory() for x in kv] for kv in kv_pool]
    hout = [torch.empty((w.batch,) + tuple(out.shape[1:]), dtype=out.dtype, pin_memory=True)
            for _ in range(2)]
    hout_par = torch.empty_like(hout[0], pin_memory=True)
    dbuf = [tuple(torch.empty_like(x) for x in inputs(1)) for _ in range(2)]
    # the job's result: O of the whole batch (batch mode: this rank's sequences
    # are one contiguous slab of it, gathered in place)
    obuf = [torch.empty((w.batch,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
            for _ in range(2)]
    oview = [o[seqs[0]:seqs[-1] + 1] if seqs else o for o in obuf]
    copy = torch.cuda.Stream()
    mk = lambda: torch.cuda.Event(enable_timing=False)  # noqa: E731
    ev_in, ev_used, ev_out = [mk(), mk()], [mk(), mk()], [mk(), mk()]
    gather_o = None
    if mode in ("batch", "slabs", "units"):
        import torch.distributed as dist

        if mode in ("batch", "slabs") and BACKEND == "nccl":
            def gather_o(o):  # rank r's rows are slab r of O: gather in place
                flat = o.view(world, -1)
                dist.all_gather_into_tensor(o.view(-1), flat[rank])
        elif mode == "batch":
            def gather_o(o):  # gloo (functional tests): host staging, rank-major slabs
                parts = list(o.cpu().view(world, -1).unbind(0))
                dist.all_gather(parts, parts[rank].clone())
                o.copy_(torch.stack(parts).view(o.shape))
        else:
            from paper_2601_13684_b200.parallel import combine_unit_outputs

            def gather_o(o):  # gloo (functional tests) / bin-packed units: host staging
                parts = [x.clone() for x in o.cpu()[None].expand(world, *o.shape)]
                dist.all_gather(parts, o.cpu())
                o.copy_(combine_unit_outputs(parts, owned_all, m.group))
    h2d = hq_all[0].numel() * hq_all[0].element_size() + sum(
        x.numel() * x.element_size() for x in hkv[0])
    d2h = hout[0].numel() * hout[0].element_size()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def upload(tt, slot):
        src = (hq_all[tt - t_start - 1],) + tuple(hkv[tt % 4])
        with torch.cuda.stream(copy):
            copy.wait_event(ev_used[slot])  # the decode that last read this slot is done
            for dst, x in zip(dbuf[slot], src):
                dst.copy_(x, non_blocking=True)
            ev_in[slot].record(copy)

    def loop_a(n):
        nonlocal t
        # light timing: two events per step around the K4 phase (the roofline's
        # launch duration); the full phase timeline is the block after the timed
        # region, so its host cost does not slow launch-bound configurations
        dec.kernel_timing(True, light=True)  # (discards the previous block's phases)
        dec.retrieval_stats()
        l0 = lib.hc_launch_count()
        barrier()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx-include "timed/" selects loop A
        ev0.record(stream)
        lo = t
        for i in range(n):
            t += 1
            if flush:
                flush_l2(i)
            dec.decode_step(t, *inputs(t), par_out if t == t_par else out, rows=False)
            if flush:
                dec.join()
                fe[i].record(stream)
        dec.join()  # the last step's monitor runs on the engine's side stream
        ev1.record(stream)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        barrier()
        return (flushed_ms(n) if flush else ev0.elapsed_time(ev1), lib.hc_launch_count() - l0,
                dec.kernel_timing(True, light=True), dec.retrieval_stats(), (lo, t))

    def loop_b(n):
        nonlocal t
        for e in ev_used + ev_out:
            e.record(stream)
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        if world == 1 and dec.devdec:
            # the C-ABI per-step call with HOST buffers (hc_engine_decode_step_host):
            # inputs H2D and O D2H on the engine's copy streams, one call per step
            for i in range(n):
                t += 1
                if flush:
                    flush_l2(i)
                dec.decode_step_host(t, hq_all[t - t_start - 1], *hkv[t % 4],
                                     hout_par if t == t_par else hout[i % 2], rows=False)
                if flush:
                    dec.join()
                    fe[i].record(stream)
            n_py = 0
        else:
            n_py = n
            upload(t + 1, 0)
        for i in range(n_py):
            t += 1
            slot = i % 2
            if i + 1 < n_py:
                upload(t + 1, 1 - slot)
            stream.wait_event(ev_in[slot])
            stream.wait_event(ev_out[slot])  # previous download of this output slot finished
            dec.decode_step(t, *dbuf[slot], oview[slot], rows=False)
            ev_used[slot].record(stream)
            with torch.cuda.stream(copy):
                copy.wait_event(ev_used[slot])
                if gather_o is not None:
                    gather_o(obuf[slot])
                hout[slot].copy_(obuf[slot], non_blocking=True)
                ev_out[slot].record(copy)
        stream.wait_stream(copy)
        dec.join()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return flushed_ms(n) if flush and n_py == 0 else ev0.elapsed_time(ev1)

    # L2 flush between timed steps (small configurations): a 252 MB write, then the
    # step between two events -- its time excludes the flush
    flush = l2_flush(args, w, plan.rho, world) and (world == 1 and dec.devdec)
    if l2_flush(args, w, plan.rho, world) and not flush:
        raise SystemExit("--l2 flush needs one GPU and device decisions")
    l2buf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device="cuda") if flush else None
    fs = [torch.cuda.Event(enable_timing=True) for _ in range(K)] if flush else []
    fe = [torch.cuda.Event(enable_timing=True) for _ in range(K)] if flush else []

    def flush_l2(i):
        l2buf.fill_(i & 0xff)
        fs[i].record(stream)

    def flushed_ms(n):
        return sum(a.elapsed_time(b) for a, b in zip(fs[:n], fe[:n]))

    clocks = ClockSampler(torch.cuda.current_device())
    if not os.environ.get("HC_BENCH_NO_CLOCKS"):
        clocks.start()
    ms = ms_e2e = 0.0
    launches = 0
    phases, retr_parts, a_ranges = {}, [], []
    rows_first = rows_last = None
    blocks = {"A": [], "B": []}
    rows_first = dec.resident_rows(t + 1)
    # palindromic order A1 B1 B2 A2: a drift rate that ramps up over the run (the
    # staggered shifts begin with the timed region) weighs both loops alike
    for kind, h in (("A", halves[0]), ("B", halves[0]), ("B", halves[1]), ("A", halves[1])):
        if kind == "B":
            m_b = loop_b(h)
            ms_e2e += m_b
            blocks["B"].append(m_b)
            continue
        m_a, l_a, ph, rs, rng = loop_a(h)
        blocks["A"].append(m_a)
        ms += m_a
        launches += l_a
        for key, val in ph.items():
            phases[key] = phases.get(key, 0) + val
        retr_parts.append(rs)
        a_ranges.append(rng)
    rows_last = dec.resident_rows(t)
    clk = clocks.stop()
    # the instrumented block: every phase event (append | K4 | combine | rows |
    # monitor | tail | gap), not part of any timed number
    n_ph = phase_steps(args)
    dec.kernel_timing(True)
    for _ in range(n_ph):
        t += 1
        dec.decode_step(t, *inputs(t), out, rows=False)
    dec.join()
    phases_full = dec.kernel_timing(False)
    dec.retrieval_stats()
    dec.finish()
    dec.sync()
    attn_ms, attn_n = phases["attention"], phases["steps"]
    rb = sum(r["bytes"] for r in retr_parts)
    rg = sum(r["gather_ms"] for r in retr_parts)
    retr = {"bytes": rb, "gather_ms": rg,
            "landing_stall_ms": sum(r["landing_stall_ms"] for r in retr_parts),
            "batches": sum(r["batches"] for r in retr_parts),
            "host_link_gbs": (rb / (rg * 1e-3) / 1e9) if rg > 0 else None}
    if world == 1 and dec.devdec and t_par > 0 and \
            t_par not in range(*(x + 1 for x in a_ranges[0])) and \
            t_par not in range(*(x + 1 for x in a_ranges[1])) and t_par > t_start:
        par_out.copy_(hout_par)  # the parity step ran through the host-buffer path

    # fires of loop A (its last boundary is decided during loop B) and the
    # reference's exposed-transfer measure (reporting.py:127-132): steps a
    # satellite served its stale set beyond trigger + update_delay_steps
    timed_ev = [e for s in dec.states for e in s.raw_events
                if any(lo < e.trigger_step <= hi for lo, hi in a_ranges)]
    events = len(timed_ev)
    exposed = sum(max(0, e.completion_step - (e.trigger_step + cfg.update_delay_steps))
                  for e in timed_ev)
    ref_bytes = sum(e.transfer_bytes for e in timed_ev)  # engine.py:330-333 accounting
    if world > 1:
        from paper_2601_13684_b200.parallel import max_over_ranks
        ms, ms_e2e = max_over_ranks([ms, ms_e2e], device=COLL_DEV)
    jobs = world if mode == "sequences" else 1  # batches decoded per step by the whole job
    own_rows = (rows_first + rows_last) / 2.0  # this rank's (K4 bytes per launch)
    if mode in ("batch", "slabs", "units"):  # one batch over all ranks: the ranks' sum
        import torch.distributed as dist

        tot = torch.tensor([rows_first, rows_last, events, exposed, ref_bytes],
                           dtype=torch.float64, device=COLL_DEV)
        dist.all_reduce(tot)
        rows_first, rows_last, events, exposed, ref_bytes = (int(x) for x in tot.tolist())
    rows_avg = (rows_first + rows_last) / 2.0
    step_bytes = algorithmic_bytes(int(rows_avg), w.batch, w.num_layers, m.q_heads)
    # the dominant kernel's bytes per launch: this rank's own resident rows
    q_rows = int(dec.owned.sum()) * m.group
    attn_bytes = own_rows * 2 * m.head_dim * 2 + q_rows * m.head_dim * 2 * 2
    # K4 phase as measured (it includes any residual landing wait inside it)
    attn_avg_ms = attn_ms / max(1, attn_n)
    stall_avg_ms = max(0.0, attn_ms - retr["landing_stall_ms"]) / max(1, attn_n)
    peak, peak_src, pk = peaks()
    rprobe = None
    if world == 1 and os.environ.get("HC_NO_READ_PROBE") != "1":
        try:
            rprobe = read_probe()
        except (RuntimeError, torch.OutOfMemoryError):  # a diagnostic: never fails the run
            rprobe = None
    achieved = attn_bytes / (attn_avg_ms * 1e-3) / 1e9 if attn_avg_ms > 0 else 0.0
    traffic = None
    tf = ROOT / "profiles" / f"traffic_{args.workload}.json"
    if tf.exists() and args.policy == "heterocache" and world == 1:
        traffic = json.loads(tf.read_text()).get("dram_bytes_per_launch")
    roles = {hd: p.role for hd, p in tax.heads.items()}
    res = {
        "metric": METRIC,
        "value": jobs * K / (ms * 1e-3),
        "unit": "steps/s",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": ms / K,
        "higher_is_better": True,
        "scaling": scaling_of(args, mode),
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic: counter-generated bf16 K/V/Q with planted per-cluster hot sets "
                "and topic shifts (random-init shapes; no checkpoint)",
        "config": make_config(args, w, cfg, plan.rho, plan.l_base_int, roles, world, mode),
        "hbm_gbs_step": jobs * step_bytes / (ms / K * 1e-3) / 1e9,
        "algorithmic_bytes_per_step": int(step_bytes),
        "e2e": {"value": jobs * K / (ms_e2e * 1e-3), "unit": "steps/s",
                # batch mode: every rank uploads its own sequences' inputs
                "h2d_bytes_per_step": int(h2d * (world if mode == "batch" else 1)),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "attn_tiles_kernel (K4)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_src,
                     "traffic": traffic,
                     "bytes_per_launch": int(attn_bytes), "avg_launch_ms": attn_avg_ms,
                     "launches_timed": attn_n,
                     "frac_excluding_landing_waits":
                         attn_bytes / (stall_avg_ms * 1e-3) / 1e9 / peak if stall_avg_ms else None,
                     "vs_nominal_8tbs": achieved / 8000.0,
                     "read_only_peak_gbs": rprobe["gbs"] if rprobe else None,
                     "frac_vs_read_only_peak": achieved / rprobe["gbs"] if rprobe else None,
                     "read_only_probe": rprobe},
        "clocks": clk,
        "phase_ms_per_step": {k: v / max(1, phases_full["steps"])
                              for k, v in phases_full.items() if k != "steps"},
        "phase_block": {"steps": phases_full["steps"],
                        "what": "every phase event recorded, in a block after the timed "
                                "region (the timed loops record only the two events "
                                "around K4)"},
        "timed_blocks_ms": blocks,  # run order A1 B1 B2 A2 (device-input / e2e halves)
        "profiling": prof,
        "prefill_scoring": {
            "kernel": "obs_score_kernel (K5, tcgen05.mma kind::f16 M=128 N=128, TMEM accumulators)",
            "obs_window": obs, "rows_valid": obs * m.group, "ms_per_layer": score_ms,
            "k_reads": passes_k,
            "hbm_gbs": score_bytes / (score_ms * 1e-3) / 1e9 if score_ms else None,
            "tflops_issued": score_flops / (score_ms * 1e-3) / 1e12 if score_ms else None,
            "tensor_peak_tflops": pk.get("bf16_tflops"),
        },
        "retrieval_events_timed_run": events,
        "exposed_transfer_steps_timed_run": exposed,
        # bytes: rows the timed loop's gathers moved over the host link (fetched set +
        # sinks + recency tail, an upper bound); reference_accounted_bytes: what the
        # reference charges for the timed loop's fires (fetched indices x bytes_per_kv_entry)
        "retrieval": {"host_link_gbs": retr["host_link_gbs"], "bytes": retr["bytes"],
                      "reference_accounted_bytes_timed_run": ref_bytes,
                      "gather_ms": retr["gather_ms"],
                      "landing_stall_ms_total": retr["landing_stall_ms"],
                      "batches": retr["batches"]},
        "prefill_seconds": prefill_s,
        "device_bytes": dec.device_bytes, "pinned_host_bytes": dec.host_bytes,
    }
    capture = None
    if t_par > 0 and world == 1:
        capture = dict(t=t_par, out=par_out.cpu(),
                       events=[[dict(trigger_step=e.trigger_step, pivot=tuple(e.pivot),
                                     completion_step=e.completion_step,
                                     transfer_bytes=e.transfer_bytes, fetches=e.fetches)
                                for e in st.events if e.trigger_step <= t_par]
                               for st in dec.states])
    dec.close()
    del dec
    torch.cuda.empty_cache()
    return res, capture, (roles, [(c.pivot, tuple(c.satellites)) for c in tax.clusters],
                          dict(plan.lengths), plan.l_base_int)


# ---------------------------------------------------------------------------
# CPU decoder (oracle port): cpu_baseline + parity leg, and the reference arm
# ---------------------------------------------------------------------------


def cpu_decode(args, w, roles, clusters, lengths, l_base_int, seqs, n_steps, warmup_steps=0,
               capture=None):
    """Decode `seqs` of the workload on the host cores with the CPU decoder
    oracle over the same seeded inputs as the GPU arm.  Returns (per-step seconds
    of the sample over the timed steps, cores, parity or None)."""
    import numpy as np
    import torch

    from oracle.cpu_decoder import CpuDecoder
    from oracle.synth import HostNormal
    from paper_2601_13684_b200.workload import SyntheticKV, decode_queries

    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    m = w.model
    shifts, T = schedule(args, w)
    cfg = engine_config(args, w)
    gen = SyntheticKV(m, batch=w.batch, prefill_len=w.prefill_len, num_layers=w.num_layers,
                      hot=hot_of(w), seed=seed_of(args), normal=HostNormal(), seqs=seqs)
    qs = decode_queries(gen, n_steps, shifts)
    kv_pool = [gen.step_inputs(100 + i, None)[1:] for i in range(4)]
    decs = [CpuDecoder(roles=roles, clusters=clusters, lengths=lengths, l_base_int=l_base_int,
                       prefill_len=w.prefill_len, max_decode=n_steps, group=m.group,
                       tau_drift=cfg.tau_drift, window=cfg.window,
                       transfer_bandwidth=cfg.transfer_bandwidth,
                       update_delay_steps=cfg.update_delay_steps, sink_count=cfg.sink_count,
                       recency_window=cfg.recency_window, bytes_per_kv_entry=512)
            for _ in seqs]
    obs = obs_of(args, w)
    t0 = time.perf_counter()
    for l in range(w.num_layers):
        k, v, q = gen.layer_kv(l, obs)
        for i, d in enumerate(decs):
            d.prefill(l, k[i], v[i], q[i])
        del k, v, q
    prefill_s = time.perf_counter() - t0
    times = []
    outs = None
    for t in range(1, n_steps + 1):
        kn, vn = kv_pool[t % 4]
        s0 = time.perf_counter()
        outs = [d.step(t, qs[t][i], kn[i], vn[i])[0] for i, d in enumerate(decs)]
        if t > warmup_steps:
            times.append(time.perf_counter() - s0)
    per_step = sum(times) / max(1, len(times))
    parity = None
    if capture is not None:
        got = capture["out"][seqs].float()
        ref = torch.stack(outs)
        err = (got - ref).abs()
        ok = bool((err <= O_ATOL + O_RTOL * ref.abs()).all())
        ev_ok = all(capture["events"][b] == d.events for b, d in zip(seqs, decs))
        parity = {"step": capture["t"], "sequences": list(seqs),
                  "units": len(seqs) * w.num_layers * m.kv_heads,
                  "max_abs": float(err.max()),
                  "max_rel": float((err / ref.abs().clamp_min(1e-3)).max()),
                  "tolerance": f"|O - O_cpu| <= {O_ATOL} + {O_RTOL} |O_cpu| (bf16 in/out, "
                               f"fp32 accumulate)",
                  "within_tolerance": ok,
                  "events_compared": sum(len(d.events) for d in decs),
                  "events_identical": ev_ok,
                  "reference": "oracle/cpu_decoder.py (fp32 attention over the CacheView sets + "
                               "the reference decision sequence), same seeded inputs"}
    return per_step, cores, parity, prefill_s, len(times)


def cpu_sample(w, args):
    n = max(1, min(args.cpu_seqs, w.batch))
    return list(range(n))


def reference_engine_timing(seconds_cap: float = 60.0):
    """The reference package's OWN engine (heterocache.engine.CacheEngine, the
    unmodified install in baseline/_ref, pure Python, one core) replaying the
    committed HCTRACE1 export of a 128K GPU run (tests/golden/scale_128k: a
    cfg3-shaped slice, 2 layers x 4 KV heads x 1 sequence, every head's records
    so its _measure runs too) -- SURVEY.md 8d CPU baseline (i).  Decision
    bookkeeping only: the reference has no attention."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "heterocache").exists():
        return {"unavailable": "reference not installed into baseline/_ref"}
    import numpy as np

    sys.path[:0] = [str(ref), str(ROOT / "tests")]
    from golden_io import key
    from heterocache.budget import BudgetPlan
    from heterocache.engine import CacheEngine, EngineConfig
    from heterocache.profiling import Cluster, HeadProfile, TaxonomyResult
    from heterocache.trace import TraceManifest, make_trace

    d = ROOT / "tests" / "golden" / "scale_128k"
    run = json.loads((d / "scale_run.json").read_text())
    z = np.load(d / "scale_trace.npz")
    tr = make_trace(TraceManifest(**run["manifest"]), z["indices"], z["scores"])
    cid, clusters = {}, []
    for i, (p, sats) in enumerate(run["clusters"]):
        clusters.append(Cluster(i, tuple(p), tuple(tuple(x) for x in sats)))
        for mm in [tuple(p)] + [tuple(x) for x in sats]:
            cid[mm] = i
    heads = {key(h): HeadProfile(layer=key(h)[0], head=key(h)[1], s_stable=run["s_stable"][h],
                                 s_sim=0.0, role=r, cluster_id=cid.get(key(h)))
             for h, r in run["roles"].items()}
    m = run["manifest"]
    tax = TaxonomyResult(num_layers=m["num_layers"], heads_per_layer=m["heads_per_layer"],
                         tau_stable=0.5, tau_sim=0.5, profiling_topk=None, heads=heads,
                         clusters=tuple(clusters))
    p = run["plan"]
    plan = BudgetPlan(rho=p["rho"], prefill_len=p["prefill_len"], num_heads=p["num_heads"],
                      num_full=p["num_full"], num_comp=p["num_comp"], l_base=p["l_base"],
                      l_base_int=p["l_base_int"],
                      lengths={key(h): n for h, n in p["lengths"].items()})
    eng = CacheEngine(tr, tax, plan, EngineConfig(**run["config"]))
    st = eng.prefill_init()
    t0 = time.perf_counter()
    n = 0
    for t in range(1, m["decode_steps"] + 1):
        eng.decode_step(st, t)
        n += 1
        if time.perf_counter() - t0 > seconds_cap:
            break
    dt = (time.perf_counter() - t0) / n
    scale = 28 * 4 / m["num_layers"]  # cfg3: 28 layers x 4 sequences
    return {"engine": "heterocache.engine.CacheEngine (baseline/_ref, unmodified)",
            "cores": 1, "sample": f"HCTRACE1 export of a 128K GPU run: {m['num_layers']} layers x "
                                  f"{m['heads_per_layer']} KV heads x 1 sequence, {n} decode steps",
            "ms_per_step_sample": dt * 1e3,
            "cfg3_steps_per_s": 1.0 / (dt * scale), "cfg3_extrapolation_factor": scale}


def run_reference(args, world):
    """--impl reference: the CPU path (oracle port) on the host cores."""
    import torch

    from oracle import calibration as OC
    from paper_2601_13684_b200.workload import plan_for

    torch.set_num_threads(os.cpu_count() or 1)
    w = workload_of(args)
    m = w.model
    t0 = time.time()
    if args.roles == "profiled":
        roles, clusters, lengths, lbase, rho, stab, prof_s = OC.calibrate(
            m, w.num_layers, w.compression, w.prefill_len, calib_spec(args))
        clusters = [(tuple(p), tuple(tuple(s) for s in sats)) for p, sats in clusters]
    else:
        tax, plan = plan_for(w)
        roles = {hd: p.role for hd, p in tax.heads.items()}
        clusters = [(c.pivot, tuple(c.satellites)) for c in tax.clusters]
        lengths, lbase, rho, prof_s = dict(plan.lengths), plan.l_base_int, plan.rho, 0.0
    profiling_s = time.time() - t0
    seqs = cpu_sample(w, args)
    K, W = args.steps, args.warmup
    per_step, cores, _, prefill_s, n = cpu_decode(args, w, roles, clusters, lengths, lbase,
                                                  seqs, W + K, warmup_steps=W)
    factor = w.batch / len(seqs)
    v = 1.0 / (per_step * factor)
    cfg = engine_config(args, w)
    sample = (f"{len(seqs)} of {w.batch} sequences (all {w.num_layers} layers and heads: "
              f"prefill selection, attention, drift monitor, fires, landings); "
              f"{n} timed steps after {W} warm-up steps; a sequence is one reference engine "
              f"(SURVEY 8b), so the full-batch step time is the sample's x {factor:g}")
    res = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "steps/s",
        "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": scaling_of(args, shard_mode(args, w, world)),
        "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic: counter-generated bf16 K/V/Q with planted per-cluster hot sets "
                "and topic shifts (random-init shapes; no checkpoint)",
        "config": make_config(args, w, cfg, rho, lbase, roles, world,
                              shard_mode(args, w, world)),
        "extrapolation": {"factor": factor, "ms_per_step_measured_sample": per_step * 1e3,
                          "ms_per_full_step": per_step * factor * 1e3},
        "cpu_baseline": {"value": v, "unit": "steps/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "profiling": {"source": "oracle/calibration.py (fp32 rows, hc_oracle.run_taxonomy, "
                                "hc_oracle.plan_budget)" if args.roles == "profiled" else
                      "fixed survey mix", "profiling_s": profiling_s},
        "prefill_seconds": prefill_s,
        # SURVEY 8d baseline (i): the reference's own engine, decision bookkeeping only
        "reference_engine": reference_engine_timing(),
    }
    return res


# ---------------------------------------------------------------------------


def spawn(args) -> int:
    """`bench.py --gpus N` without torchrun: re-launch under torchrun."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd)


def secondary(args):
    """The secondary workload's line (child process, after this one's memory is free)."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--workload", args.secondary, "--steps",
           str(args.steps), "--warmup", str(args.warmup), "--secondary", "none",
           "--cpu-seqs", str(args.cpu_seqs), "--roles", args.roles,
           "--score-material", args.score_material]
    if args.no_cpu_baseline:
        cmd.append("--no-cpu-baseline")
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
        line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
        d = json.loads(line)
    except Exception as exc:  # noqa: BLE001
        return {"workload": args.secondary, "error": f"{type(exc).__name__}: {exc}"[:300]}
    keep = ("value", "e2e", "ms_per_step", "roofline", "clocks", "parity", "cpu_baseline",
            "hbm_gbs_step", "algorithmic_bytes_per_step", "config", "retrieval",
            "exposed_transfer_steps_timed_run", "prefill_scoring", "profiling", "gpu_launches",
            "phase_ms_per_step")
    return {"workload": args.secondary, **{k: d.get(k) for k in keep}}


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        return spawn(args)
    world = int(env_world or "1")
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(run_reference(args, world)))
        return 0

    import torch

    from paper_2601_13684_b200 import build as _build
    _build.ensure_built()  # no-op when the in-tree library shipped with the checkout
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(BACKEND)
    res, capture, plan_info = run_b200(args, rank, world)
    if rank == 0:
        res["cpu_baseline"] = None
        res["parity"] = None
        w = workload_of(args)
        if world == 1 and not args.no_cpu_baseline:
            seqs = cpu_sample(w, args)
            roles, clusters, lengths, lbase = plan_info
            n_steps = capture["t"] if capture else min(PARITY_STEP, args.warmup + args.steps)
            per_step, cores, parity, _, n = cpu_decode(args, w, roles, clusters, lengths, lbase,
                                                       seqs, n_steps, warmup_steps=2,
                                                       capture=capture)
            factor = w.batch / len(seqs)
            res["cpu_baseline"] = {
                "value": 1.0 / (per_step * factor), "unit": "steps/s", "cores": cores,
                "cpu_model": cpu_model(), "kind": "port",
                "sample": f"oracle/cpu_decoder.py on {len(seqs)} of {w.batch} sequences (all "
                          f"layers and heads, same seeded inputs), {n} timed steps of "
                          f"{n_steps}; per-step time x {factor:g}"}
            res["parity"] = parity
        if world == 1 and args.secondary not in ("none", "", args.workload):
            res["secondary"] = secondary(args)
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
