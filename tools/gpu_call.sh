mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "expectation or sweep or config3 or h2 or golden_expectation or dense or jit_ucc" 2>&1 | tail -3
echo "== warps (default)"; timeout 600 python tools/time_expect30.py 2
echo "== warps TERMS=16"; QSV_SWEEP_TERMS=16 timeout 600 python tools/time_expect30.py 2
echo "== warps TERMS=12"; QSV_SWEEP_TERMS=12 timeout 600 python tools/time_expect30.py 2
echo "== legacy"; QSV_SWEEP_WARPS=0 timeout 600 python tools/time_expect30.py 2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -c 200 --csv --log-file gpurun_out/r02_expect30_warps_launches.csv python tools/time_expect30.py 1 > /dev/null 2>&1; echo launches rc=$?
