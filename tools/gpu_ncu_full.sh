# ncu --set full capture of two tile passes of the config-2 bench (launches 40-41)
mkdir -p gpurun_out
export QSV_FUSE_QUBITS=${QSV_FUSE_QUBITS:-1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tile_|qsv_pass" --launch-skip 45 --launch-count 3 \
  -o gpurun_out/${TAG:-tile}_full python tools/profile_evolve.py brick28 3 > gpurun_out/ncu_full.log 2>&1
echo ncu rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/${TAG:-tile}_launches.csv python tools/profile_evolve.py brick28 2 > /dev/null 2>&1; echo launches rc=$?
