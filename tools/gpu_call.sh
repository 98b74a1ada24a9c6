mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q -m gpu -k "config1 or hot or jit or ucc or golden or gradient" 2>&1 | tail -4
echo "== compact (default)"; timeout 600 python tools/time_ucc12.py 2>&1 | tail -2
echo "== straight"; QSV_COMPACT_GMAT=0 timeout 600 python tools/time_ucc12.py 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none -k regex:qsv_pass --launch-skip 8 --launch-count 2 -o gpurun_out/r02_ucc12_pass_compact python tools/time_ucc12.py > /dev/null 2>&1; echo ncu rc=$?
