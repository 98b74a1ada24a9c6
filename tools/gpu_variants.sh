# bench variants (env settings) on the config-2 bench, ms/step + frac
mkdir -p gpurun_out
for v in $VARIANTS; do
  vv=$(echo $v | tr ',' ' ')
  env $vv timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --extra none > gpurun_out/var.log 2>&1
  echo "$v $(python -c "import json;d=json.loads(open('gpurun_out/var.log').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],2), round(d['roofline']['frac'],3), d['config']['hbm_passes_per_step'])" 2>&1 | tail -1)"
done
