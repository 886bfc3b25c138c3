# A/B: strip K1 with two grid lines per step (k_iter1_s5p, SG_STRIP_K1_PAIRS=1) vs one (=0).
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_parity.py tests/test_gpu_rowpart.py -m gpu -q -p no:cacheprovider -k "strip or wide or c5 or C5 or partition" > $O/r03e_pairs_tests.log 2>&1; echo rc=$? >> $O/r03e_pairs_tests.log
for v in 1 0 1 0; do
  SG_STRIP_K1_PAIRS=$v timeout 400 python bench_configs.py --config c5 --steps 3 --warmup 1 >> $O/r03e_pairs_c5_$v.jsonl 2>> $O/r03e_pairs.err
done
