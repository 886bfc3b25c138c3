O=gpurun_out
for e in "X=1" "SG_PCG_K1=t" "SG_PCG_K23=t" "SG_PCG_K1=t SG_PCG_K23=t" "SG_PCG_NOSTAGE=1" "SG_SW_RANGE=1024" "SG_SW_RANGE=4096"; do
  echo "== $e" >> $O/r03_c1var.txt
  env $e timeout 300 python bench_configs.py --config c1 --steps 3 --warmup 1 2>> $O/r03_c1var.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(round(d['value'],3), d['k'], round(d['ms_per_solve'],1), {k:round(x['avg_ms']*1000,1) for k,x in d['per_kernel'].items()})" >> $O/r03_c1var.txt
done
