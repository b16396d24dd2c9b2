"""Summarise ncu reports / launch lists (run here, no GPU).  Usage:
    python tools/ncu_summary.py launches gpurun_out/launches_X.csv
    python tools/ncu_summary.py report gpurun_out/prof_X.ncu-rep [more...]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_active.avg", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    own = sum(sum(v) for k, v in d.items() if "rrs::" in k) or 1  # the library's kernels only (no flush / copies)
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        s_own = f"  share of rrs kernels={100*sum(v)/own:5.1f}%" if "rrs::" in k else ""
        print(f"{k:72s} n={len(v):3d} mean={sum(v)/len(v)/1e3:9.2f} us  share={100*sum(v)/tot:5.1f}%{s_own}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units, v = r[0], r[1], r[2]
    print(f"== {path}: {v[h.index('Kernel Name')][:90]}")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k:80s} {v[i]:>14s} {units[i]}")
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                st.append((float(v[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    print("  stalls: " + ", ".join(f"{n} {100*x/tot:.0f}%" for x, n in sorted(st, reverse=True)[:8]))


if __name__ == "__main__":
    mode = sys.argv[1]
    for p in sys.argv[2:]:
        (launches if mode == "launches" else report)(p)
