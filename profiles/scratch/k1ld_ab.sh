O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowpart.py tests/test_gpu_config_parity.py -m gpu -q -p no:cacheprovider -k "strip or wide or partition or c5 or C5 or control_flow" > $O/r03_k1ld_tests.log 2>&1; echo rc=$? >> $O/r03_k1ld_tests.log
for v in new base new base; do
  if [ $v = new ]; then L=""; else L=profiles/scratch/lib_$v.so; fi
  SG_LIB_PATH=$L timeout 400 python bench_configs.py --config c5 --steps 3 --warmup 1 >> $O/r03_k1ld_$v.jsonl 2>> $O/r03_k1ld.err
done
