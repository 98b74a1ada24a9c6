mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
for u in 0 1; do echo "== QSV_CZ_DEFER=$u"; QSV_CZ_DEFER=$u timeout 300 python bench.py --steps 10 --warmup 3 --extra none --no-cpu-baseline 2>&1 | tail -1 | cut -c1-150; done
timeout 900 python tools/parity_config2_full.py 2>&1 | tail -3 | tee gpurun_out/r02_parity_config2_full_cz.log
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:qsv_pass -c 60 --csv --log-file gpurun_out/fp64_launches_cz.csv python bench.py --steps 1 --warmup 3 --extra none --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
