O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_parity.py tests/test_gpu_rowpart.py tests/test_gpu_boundary.py -m gpu -q -p no:cacheprovider > $O/r03_rpt2_tests.log 2>&1; echo rc=$? >> $O/r03_rpt2_tests.log
for v in 2 1 4 2 1 4; do
  if [ $v = 2 ]; then L=""; else L=profiles/scratch/lib_rpt$v.so; fi
  SG_LIB_PATH=$L timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 >> $O/r03_rpt_$v.jsonl 2>> $O/r03_rpt.err
done
