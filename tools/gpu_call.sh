mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dropin.py -x -q -m gpu 2>&1 | tail -25
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full_r02a.log 2>&1; echo bench rc=$?; tail -c 6000 gpurun_out/bench_full_r02a.log
