mkdir -p gpurun_out
for t in 16 32 48; do echo "== QSV_SWEEP_TERMS=$t"; QSV_SWEEP_TERMS=$t timeout 300 python tools/time_expect30.py 2; done
timeout 300 python tools/time_ucc12.py
timeout 300 python tools/host_profile_ucc12.py 2>&1 | tail -12
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -c 60 --csv --log-file gpurun_out/r02_ucc12_launches.csv python tools/time_ucc12.py > /dev/null 2>&1; echo ncu rc=$?
