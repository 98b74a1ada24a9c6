mkdir -p gpurun_out
for n in 20 22 24 26; do
  QSV_TILE_RING=0 timeout 30 python tools/diag_ring.py $n 2>&1 | tail -1
  QSV_TILE_RING=1 timeout 30 python tools/diag_ring.py $n 2>&1 | tail -1
done
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for v in "QSV_FUSE_QUBITS=2" "QSV_FUSE_QUBITS=0" "QSV_FUSE_QUBITS=1"; do
  echo "== $v"; env $v timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --extra none > gpurun_out/ab.log 2>&1; tail -1 gpurun_out/ab.log | cut -c1-200; grep -o '"frac": [0-9.]*' gpurun_out/ab.log
done
