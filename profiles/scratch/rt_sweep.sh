O=gpurun_out
SG_PCG_K23RT=2 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowpart.py -m gpu -q -p no:cacheprovider -k "sliding or stencil or deferred or control_flow or batch or 3d or partitioned" > $O/r03_pytest_rt2.log 2>&1; echo rc=$? >> $O/r03_pytest_rt2.log
for rt in 1 2 1 2; do SG_PCG_K23RT=$rt timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 >> $O/r03_rt_$rt.jsonl 2>> $O/r03_rt.err; done
