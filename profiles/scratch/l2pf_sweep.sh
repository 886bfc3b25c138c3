O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_rowpart.py tests/test_gpu_formats.py -m gpu -q -p no:cacheprovider > $O/r03_pytest5.log 2>&1; echo rc=$? >> $O/r03_pytest5.log
for pf in 0 2 4 8; do SG_PCG_L2PF=$pf timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/r03_l2pf_$pf.jsonl 2> $O/r03_l2pf_$pf.err; done
