"""Per-expectation instruction counts of config 3 from an ncu CSV (--metrics
gpu__time_duration.sum, smsp__inst_executed.sum, smsp__sass_thread_inst_
executed_op_{dfma,dmul,dadd}_pred_on.sum, dram__bytes_read.sum) over all the
sweep launches of ONE expectation; writes profiles/r02_expect30_counts.json
for bench.py's expect30 roofline.
    python tools/ncu_expect_counts.py launches.csv > profiles/r02_expect30_counts.json"""
import csv
import io
import json
import sys
from collections import defaultdict

text = open(sys.argv[1]).read()
text = text[text.index('"ID"'):]
L = defaultdict(dict)
names = {}
for r in csv.DictReader(io.StringIO(text)):
    i = int(r["ID"])
    L[i][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    names[i] = r["Kernel Name"]
sweeps = [i for i in sorted(L) if names[i] == "qsv_sweep" or "expect_sweep2" in names[i]
          or "reduce_columns" in names[i]]
out = {"launches": len(sweeps)}
for key, m in (("warp_inst", "smsp__inst_executed.sum"),
               ("dfma", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"),
               ("dmul", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"),
               ("dadd", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"),
               ("dram_read_bytes", "dram__bytes_read.sum")):
    out[key] = int(sum(L[i].get(m, 0) for i in sweeps))
out["ncu_ms"] = sum(L[i].get("gpu__time_duration.sum", 0) for i in sweeps) / 1e6
out["sweeps"] = sum(1 for i in sweeps if "reduce_columns" not in names[i])
out["source"] = ("ncu --metrics smsp__inst_executed.sum, smsp__sass_thread_inst_executed_op_"
                 "{dfma,dmul,dadd}_pred_on.sum over the qsv_sweep / expect_sweep2 / reduce_columns "
                 "launches of one config-3 expectation (tools/time_expect30.py 1)")
print(json.dumps(out, indent=1))
