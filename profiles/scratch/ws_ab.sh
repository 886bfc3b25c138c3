# A/B: producer-warp K1 (SG_STRIP1_WS / SG_SW1_WS = 1, the in-tree library) vs the previous
# single-barrier K1 (profiles/scratch/lib_ws0.so, both macros 0).  GPU suite on the new library first.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r03c_pytest_gpu.log 2>&1; echo rc=$? >> $O/r03c_pytest_gpu.log
for v in ws base ws base; do
  if [ $v = base ]; then L=profiles/scratch/lib_ws0.so; else L=""; fi
  SG_LIB_PATH=$L timeout 400 python bench_configs.py --config c5 --steps 3 --warmup 1 >> $O/r03c_ws_c5_$v.jsonl 2>> $O/r03c_ws.err
  SG_LIB_PATH=$L timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 >> $O/r03c_ws_c2_$v.jsonl 2>> $O/r03c_ws.err
done
