"""Summarise an ncu report: key metrics per kernel + stall reasons by opcode.
    python tools/ncu_summary.py report.ncu-rep"""
import csv, io, subprocess, sys
from collections import Counter, defaultdict

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smsp__inst_executed.sum']
for r in rows[2:]:
    for w in want:
        if w in hdr:
            print(f"  {w:60s} {r[hdr.index(w)][:70]} {units[hdr.index(w)]}")
    stalls = [h for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued')]
    vals = sorted(((float(r[hdr.index(h)] or 0), h) for h in stalls), reverse=True)[:8]
    tot = sum(float(r[hdr.index(h)] or 0) for h in stalls) or 1
    print("  stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v / tot * 100:.0f}%" for v, h in vals))
    print('---')
