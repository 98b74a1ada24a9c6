# A/B of kernel / planner variants on the config-2 bench
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for v in "QSV_FUSE_QUBITS=2" "QSV_FUSE_QUBITS=0" "QSV_FUSE_QUBITS=0 QSV_TILE_RING=0"; do
  echo "== $v"; env $v timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --extra none > gpurun_out/ab.log 2>&1; tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['config']['hbm_passes_per_step'])" || tail -3 gpurun_out/ab.log
done
