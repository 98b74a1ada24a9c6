mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_geometry.py tests/test_gpu_dropin.py -x -q -m gpu -k "expectation or sweep or config3 or h2 or golden_expectation or dense or jit_ucc or ucc or parallel" 2>&1 | tail -3
echo "== fuse1 (default)"; timeout 600 python tools/time_expect30.py 3
echo "== no fuse"; QSV_SWEEP_FUSE1=0 timeout 600 python tools/time_expect30.py 3
timeout 1200 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_expect30_counts_f1.csv python tools/time_expect30.py 1 > /dev/null 2>&1; echo ncu rc=$?
