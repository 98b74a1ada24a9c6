# quick GPU check: parity tests + short bench (+ launch list)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_quick.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/bench_quick.log | cut -c1-1500
if [ -n "$LAUNCHES" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_quick.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
fi
