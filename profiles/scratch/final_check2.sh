# The committed library at the end of the session: GPU suite, smoke, default bench line.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r03s3_final_pytest_gpu.log 2>&1; echo rc=$? >> $O/r03s3_final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r03s3_final_smoke.log 2>&1; echo rc=$? >> $O/r03s3_final_smoke.log
timeout 900 python bench.py > $O/r03s3_final_bench.jsonl 2> $O/r03s3_final_bench.err
