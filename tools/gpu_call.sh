mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "expectation or sweep or config3 or h2 or golden_expectation or dense" 2>&1 | tail -4
echo "== coset"; timeout 600 python tools/time_expect30.py 3
echo "== pairbit"; QSV_SWEEP_COSET=0 timeout 600 python tools/time_expect30.py 3
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_expect30_coset_launches.csv python tools/time_expect30.py 1 > /dev/null 2>&1; echo launches rc=$?
