mkdir -p gpurun_out
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02_full_c.log 2>&1; echo bench rc=$?; tail -c 1500 gpurun_out/bench_r02_full_c.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_final_launches.csv python bench.py --steps 2 --warmup 3 --extra none --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
