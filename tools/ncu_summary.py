"""Summarise ncu output into the small text / JSON files kept under profiles/.

  python tools/ncu_summary.py launches <launches.csv>          -> per-kernel share table
  python tools/ncu_summary.py full <report.ncu-rep> <out.json>  -> key metrics of one capture
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_utchmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_bytes.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "smsp__warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    ni = hdr.index("Metric Name")
    agg = defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi and r[ni] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", ""))
            if r[ui] == "usecond":
                v *= 1e3
            elif r[ui] == "msecond":
                v *= 1e6
            agg[r[ki]].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = io.StringIO()
    out.write(f"{'launches':>8} {'total_us':>10} {'avg_us':>9} {'share':>6}  kernel\n")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.write(f"{len(v):8d} {sum(v)/1e3:10.1f} {sum(v)/len(v)/1e3:9.1f} {100*sum(v)/tot:5.1f}%  {k[:110]}\n")
    return out.getvalue()


def full(path, out_json):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = {"value": vals[i], "unit": units[i]}
        res.append(d)
    json.dump(res, open(out_json, "w"), indent=1)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]), end="")
    else:
        print(json.dumps(full(sys.argv[2], sys.argv[3]), indent=1))
