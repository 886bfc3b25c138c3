# GPU suite on the new library (fused partial gathers + two-line strip K1), then A/B against the
# library before the gather fusion (profiles/scratch/lib_pairs.so).
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r03f_pytest_gpu.log 2>&1; echo rc=$? >> $O/r03f_pytest_gpu.log
for v in new old new old; do
  if [ $v = old ]; then L=profiles/scratch/lib_pairs.so; else L=""; fi
  SG_LIB_PATH=$L timeout 400 python bench_configs.py --config c5 --steps 3 --warmup 1 >> $O/r03f_g2_c5_$v.jsonl 2>> $O/r03f_g2.err
  SG_LIB_PATH=$L timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 >> $O/r03f_g2_c2_$v.jsonl 2>> $O/r03f_g2.err
  SG_LIB_PATH=$L timeout 400 python bench_configs.py --config c1 --steps 3 --warmup 1 >> $O/r03f_g2_c1_$v.jsonl 2>> $O/r03f_g2.err
done
