mkdir -p gpurun_out
for m in 12 11 10; do echo "== QSV_TILE_BITS=$m"; QSV_TILE_BITS=$m timeout 600 python tools/time_ucc12.py 2>&1 | tail -2; done
