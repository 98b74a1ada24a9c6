"""Print the headline counters and stall ratios of every kernel in an .ncu-rep
(ncu --set full capture): duration, instructions, issue / FP64 activity,
shared bank conflicts, registers, and the stall reasons above 0.05 per issue."""
import csv, subprocess, sys

WANT = ["gpu__time_duration.sum", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for v in rows[2:]:
    print("==", v[h.index("Kernel Name")][:100])
    for k in WANT:
        if k in h:
            print(f"  {k:64s} {v[h.index(k)]}")
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                if float(v[i]) > 0.05:
                    print(f"  stall {k[34:-23]:58s} {v[i]}")
            except ValueError:
                pass
