mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qsv_pass --launch-skip 16 --launch-count 2 -o gpurun_out/r02_c2_pass_full python bench.py --steps 1 --warmup 2 --extra none --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1; echo ncu rc=$?
