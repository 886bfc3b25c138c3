# Final library of the session (trace probe compiled in, off): GPU suite, smoke, C5 config line.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r03s2_final_pytest_gpu.log 2>&1; echo rc=$? >> $O/r03s2_final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r03s2_final_smoke.log 2>&1; echo rc=$? >> $O/r03s2_final_smoke.log
timeout 400 python bench_configs.py --config c5 --steps 3 --warmup 1 > $O/r03s2_final_c5.jsonl 2>> $O/r03s2_final.err
