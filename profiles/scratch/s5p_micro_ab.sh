# A/B: strip K1 (k_iter1_s5p) d' phase with per-line uniform bounds and incremental slot / phase
# (in-tree) vs the committed kernel (lib_base.so).
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_parity.py tests/test_gpu_rowpart.py -m gpu -q -p no:cacheprovider -k "strip or wide or c5 or C5 or partition or timeline" > $O/r03j_tests.log 2>&1; echo rc=$? >> $O/r03j_tests.log
for v in new base new base; do
  if [ $v = base ]; then L=profiles/scratch/lib_base.so; else L=""; fi
  SG_LIB_PATH=$L timeout 400 python bench_configs.py --config c5 --steps 3 --warmup 1 >> $O/r03j_c5_$v.jsonl 2>> $O/r03j.err
done
