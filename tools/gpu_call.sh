mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
QSV_PASS_TMA=1 timeout 600 python -m pytest tests/test_gpu_geometry.py -x -q -m gpu 2>&1 | tail -15
QSV_PASS_TMA=1 timeout 600 python tools/time_fused30.py
QSV_PASS_TMA=1 QSV_MIN_CONTIG=3 timeout 600 python tools/time_fused30.py
cuobjdump -sass paper_2208_10978_b200/libqsv.so 2>/dev/null | grep -c UTMALDG
