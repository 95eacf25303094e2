"""Key figures of an `ncu --page raw --csv` export (one launch): duration, pipe
utilisation, issue, occupancy, registers, DRAM bytes.

usage: python tools/ncu_raw_keys.py raw.csv [more.csv ...]
"""
import csv, sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst %"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "SM inst thru %"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__occupancy_limit_registers", "occ limit regs"),
    ("launch__occupancy_limit_shared_mem", "occ limit smem"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram thru %"),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall barrier"),
]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    names, units, vals = rows[hdr], rows[hdr + 1], rows[hdr + 2]
    col = {n: i for i, n in enumerate(names)}
    print(f"== {path}: {vals[col.get('Kernel Name', 4)][:60]}")
    for k, label in KEYS:
        if k in col:
            print(f"  {label:22s} {vals[col[k]]:>16s} {units[col[k]]}")
    stalls = [(n, vals[i]) for n, i in col.items() if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued")]
    tot = sum(float(v.replace(",", "") or 0) for _, v in stalls)
    top = sorted(stalls, key=lambda kv: -float(kv[1].replace(",", "") or 0))[:8]
    if tot:
        print("  stalls: " + ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * float(v.replace(',', '')) / tot:.1f}%" for n, v in top))
