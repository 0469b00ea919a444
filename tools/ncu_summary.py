"""Summarise ncu reports / launch lists into profiles/ (tracked).

  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep profiles/r01_full_cfg3.md
  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches_cfg3.md
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: `{rep}`", ""]
    js = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        lines += [f"## {name}", "", "| metric | value | unit |", "|---|---|---|"]
        rec = {"kernel": name}
        for m in METRICS:
            hits = [j for j, h in enumerate(hdr) if h == m or h.endswith("." + m)]
            if hits:
                i = hits[0]
                lines.append(f"| {m} | {r[i]} | {units[i]} |")
                rec[m] = r[i]
        js.append(rec)
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    return js


def _us(value, unit):
    v = float(value)
    return {"nsecond": v * 1e-3, "ns": v * 1e-3, "usecond": v, "us": v, "msecond": v * 1e3,
            "ms": v * 1e3, "second": v * 1e6, "s": v * 1e6}.get(unit, v)


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"]][0] += 1
                agg[d["Kernel Name"]][1] += _us(d["Metric Value"], d.get("Metric Unit", ""))
    tot = sum(v for _, v in agg.values()) or 1.0
    # kernels of the retrieval stream run beside the step (host-link bound); the
    # step's own share is the one to compare with the bench's phase timeline
    side = ("gather_host_rows_kernel", "build_positions_batch_kernel")
    tot_step = sum(v for k, (_, v) in agg.items() if not any(x in k for x in side)) or 1.0
    lines = [f"# ncu launch list (gpu__time_duration.sum; serialised, cold caches): `{path}`", "",
             "| kernel | launches | total us | avg us | share | share of the step (excl. retrieval stream) |",
             "|---|---|---|---|---|---|"]
    for k, (n, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
        st = "—" if any(x in k for x in side) else f"{s / tot_step:.1%}"
        lines.append(f"| {k[:90]} | {n} | {s:.1f} | {s / n:.1f} | {s / tot:.1%} | {st} |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    if mode == "full":
        print(json.dumps(full(src, dst), indent=1))
    else:
        launches(src, dst)
