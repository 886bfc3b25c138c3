# Re-entry check of this round's HEAD on a fresh box: GPU suite, smoke, default bench line.
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/r03b_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r03b_pytest_gpu.log 2>&1; echo rc=$? >> $O/r03b_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r03b_smoke.log 2>&1; echo rc=$? >> $O/r03b_smoke.log
timeout 900 python bench.py > $O/r03b_bench_c2.jsonl 2> $O/r03b_bench_c2.err; echo rc=$? >> $O/r03b_bench_c2.err
