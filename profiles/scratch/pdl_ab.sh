# A/B: programmatic dependent launch of the streamed PCG kernels (SG_PCG_PDL=1, default) vs plain
# launches (SG_PCG_PDL=0).  GPU suite with PDL on first.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r03d_pytest_gpu.log 2>&1; echo rc=$? >> $O/r03d_pytest_gpu.log
for v in 1 0 1 0; do
  SG_PCG_PDL=$v timeout 400 python bench_configs.py --config c5 --steps 3 --warmup 1 >> $O/r03d_pdl_c5_$v.jsonl 2>> $O/r03d_pdl.err
  SG_PCG_PDL=$v timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 >> $O/r03d_pdl_c2_$v.jsonl 2>> $O/r03d_pdl.err
done
