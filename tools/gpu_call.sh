mkdir -p gpurun_out
(nproc; lscpu | head -20; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv) > gpurun_out/host_info.txt 2>&1
./tools/peaks_probe > gpurun_out/peaks.json 2>&1; cat gpurun_out/peaks.json
timeout 900 python -m pytest tests/test_gpu_geometry.py -x -q -m gpu --durations=10 2>&1 | tail -15
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
