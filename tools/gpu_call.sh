mkdir -p gpurun_out
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02_full_b.log 2>&1; echo bench rc=$?; tail -c 8000 gpurun_out/bench_r02_full_b.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_r02_ref.log 2>&1; echo ref rc=$?; tail -c 1500 gpurun_out/bench_r02_ref.log
