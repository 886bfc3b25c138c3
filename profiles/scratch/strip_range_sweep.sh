# C5 strip kernels: range length (lines per CTA) sweep.  Default planner: 38 lines (432 CTAs, one wave).
O=gpurun_out
for r in 0 19 13 10 26 0 19 13; do
  if [ $r = 0 ]; then unset SG_SW_RANGE; else export SG_SW_RANGE=$r; fi
  echo "range=$r" >> $O/r03s2_range_sweep.jsonl
  timeout 300 python bench_configs.py --config c5 --steps 3 --warmup 1 >> $O/r03s2_range_sweep.jsonl 2>> $O/r03s2_range_sweep.err
done
unset SG_SW_RANGE
for r in 0 19; do
  if [ $r = 0 ]; then unset SG_SW_RANGE; else export SG_SW_RANGE=$r; fi
  echo "range=$r" >> $O/r03s2_range_trace.txt
  timeout 300 python profiles/trace_probe.py >> $O/r03s2_range_trace.txt 2>> $O/r03s2_range_sweep.err
done
