"""FP64-pipe instruction counts of one config-2 step from an ncu CSV
(--csv --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_
{dfma,dmul,dadd}_pred_on.sum): sums the first `passes` qsv_pass launches after
`skip` of them and writes profiles/r02_fp64_counts.json for bench.py.
    python tools/ncu_fp64_counts.py launches.csv PASSES [SKIP] > profiles/r02_fp64_counts.json"""
import csv
import io
import json
import sys

path, passes = sys.argv[1], int(sys.argv[2])
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
text = open(path).read()
text = text[text.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(text)))
launch = {}
for r in rows:
    if "qsv_pass" not in r["Kernel Name"]:
        continue
    d = launch.setdefault(int(r["ID"]), {})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
ids = sorted(launch)[skip:skip + passes]
key = {"dfma": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
       "dmul": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
       "dadd": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"}
out = {k: int(sum(launch[i].get(m, 0) for i in ids)) for k, m in key.items()}
out["passes"] = len(ids)
out["ncu_ms"] = sum(launch[i].get("gpu__time_duration.sum", 0) for i in ids) / 1e6
out["source"] = ("ncu --metrics smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum, "
                 f"qsv_pass launches {skip}..{skip + len(ids) - 1} of `python bench.py --steps 1 "
                 "--warmup 3 --extra none --no-cpu-baseline` (one config-2 step)")
print(json.dumps(out, indent=1))
