mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_geometry.py -x -q -m gpu 2>&1 | tail -8
