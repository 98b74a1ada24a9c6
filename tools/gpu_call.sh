mkdir -p gpurun_out
QSV_SWEEP_ONETILE=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_geometry.py -x -q -m gpu -k "expectation or sweep or config3 or h2 or golden_expectation or dense or jit_ucc or ucc" 2>&1 | tail -3
for v in 0 1; do echo "== ONETILE=$v"; QSV_SWEEP_ONETILE=$v timeout 600 python tools/time_expect30.py 3 | tail -2; QSV_SWEEP_ONETILE=$v timeout 600 python tools/time_expect32.py | tail -1; done
