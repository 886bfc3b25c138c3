O=gpurun_out
SG_LIB_PATH=profiles/scratch/lib_strip128.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowpart.py -m gpu -q -p no:cacheprovider -k "strip or wide or partitioned" > $O/r03_strip128_tests.log 2>&1; echo rc=$? >> $O/r03_strip128_tests.log
for v in base 128 base 128; do
  if [ $v = base ]; then L=""; else L=profiles/scratch/lib_strip128.so; fi
  SG_LIB_PATH=$L timeout 400 python bench_configs.py --config c5 --steps 3 --warmup 1 >> $O/r03_strip_$v.jsonl 2>> $O/r03_strip.err
done
