# Final round-3 pass on the final kernels: GPU suite + smoke, then the measurement script.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r03_pytest_gpu.log 2>&1; echo rc=$? >> $O/r03_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r03_smoke.log 2>&1; echo rc=$? >> $O/r03_smoke.log
bash profiles/measure_r03.sh > $O/r03_measure.log 2>&1
