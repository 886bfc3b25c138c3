O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r03_swblk_tests.log 2>&1; echo rc=$? >> $O/r03_swblk_tests.log
for v in new base new base; do
  if [ $v = new ]; then L=""; else L=profiles/scratch/lib_$v.so; fi
  SG_LIB_PATH=$L timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 >> $O/r03_swblk_$v.jsonl 2>> $O/r03_swblk.err
done
timeout 400 python bench_configs.py --config c5 --steps 3 --warmup 1 >> $O/r03_swblk_c5.jsonl 2>> $O/r03_swblk.err
