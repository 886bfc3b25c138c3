O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "timeline or synthetic" > $O/r03h_tests.log 2>&1; echo rc=$? >> $O/r03h_tests.log
timeout 900 python bench.py --no-cpu-baseline > $O/r03h_bench.jsonl 2> $O/r03h_bench.err
