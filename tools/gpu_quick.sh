# quick GPU check: parity tests + short bench (+ launch list)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
for v in ${VARIANTS:-"QSV_FUSE_QUBITS=2"}; do
  echo "== $v"; env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --extra none > gpurun_out/bench_quick.log 2>&1; echo rc=$?; tail -1 gpurun_out/bench_quick.log | cut -c1-300; grep -o '"frac": [0-9.]*' gpurun_out/bench_quick.log
done
if [ -n "$LAUNCHES" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_quick.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --extra none > /dev/null 2>&1; echo ncu rc=$?
fi
