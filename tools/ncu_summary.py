"""Dev helper: key counters + stall mix of each kernel in an ncu report (`ncu -i X --page raw --csv`)."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__block_size", "launch__grid_size",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for v in rows[2:]:
    print("----")
    for k in keys:
        if k in h:
            print(f"  {k:60s} {v[h.index(k)][:70]}")
    st = [(h[i], v[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")]
    tot = sum(float(x[1] or 0) for x in st) or 1
    print("  stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * float(x) / tot:.1f}"
                                 for k, x in sorted(st, key=lambda t: -float(t[1] or 0))[:8]))
