# A/B: the strip K1 on its own residency-weighted line ranges (SG_STRIP_K1_WEIGHTS=1) vs K2+K3's
# uniform ranges (=0); strip / C5 tests first; then the timeline probe with the weights on.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_parity.py tests/test_gpu_rowpart.py -m gpu -q -p no:cacheprovider -k "strip or wide or c5 or C5 or partition" > $O/r03g_w_tests.log 2>&1; echo rc=$? >> $O/r03g_w_tests.log
for v in 1 0 1 0; do
  SG_STRIP_K1_WEIGHTS=$v timeout 400 python bench_configs.py --config c5 --steps 3 --warmup 1 >> $O/r03g_w_c5_$v.jsonl 2>> $O/r03g_w.err
done
SG_STRIP_K1_WEIGHTS=1 timeout 300 python profiles/trace_probe.py > $O/r03g_trace_weighted.json 2>> $O/r03g_w.err
