# One ncu --set full capture of a heavy tile pass of the config-2 bench (launch 6 of the step)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_block_kernel --launch-skip 40 --launch-count 2 \
  -o gpurun_out/r01_tile_full python tools/profile_evolve.py brick28 3 > gpurun_out/ncu_full.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/ncu_full.log
