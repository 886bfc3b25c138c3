# Round-3 second-session measurement pass (after the K1 loop change) on the final kernels (one gpurun call): GPU suite, smoke,
# bench lines (C2 headline with the C5 block, reference arm, C1/C3/C4/C5 configs), launch list of
# the C2 step, ncu --set full of the C2 and C5 PCG kernels (summarised on the box).
set -x
O=gpurun_out
T=r03s3
summ() {
  python profiles/summarize_ncu.py $O/$1.ncu-rep > $O/$1_summary.txt 2>&1
  ncu -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>&1
  ncu -i $O/$1.ncu-rep --page source --csv --print-source sass > $O/$1_source.csv 2>&1
  gzip -f $O/$1_source.csv
  rm -f $O/$1.ncu-rep
}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,power.draw --format=csv > $O/${T}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${T}_pytest_gpu.log 2>&1; echo rc=$? >> $O/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${T}_smoke.log 2>&1; echo rc=$? >> $O/${T}_smoke.log
timeout 900 python bench.py > $O/${T}_bench_c2.jsonl 2> $O/${T}_bench_c2.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/${T}_bench_reference_arm.jsonl 2> $O/${T}_ref.err
timeout 400 python bench_configs.py --config c1 >> $O/${T}_bench_configs.jsonl 2>> $O/${T}_cfg.err
timeout 400 python bench_configs.py --config c5 >> $O/${T}_bench_configs.jsonl 2>> $O/${T}_cfg.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/${T}_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-c5 > $O/${T}_ncu1.log 2>&1
python profiles/summarize_launches.py $O/${T}_launches.csv 25 > $O/${T}_launches_c2_128sys.txt 2>&1
gzip -f $O/${T}_launches.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_iter1_sw|k_iter23_sw" --launch-skip 300 -c 2 -o $O/${T}_pcg_sw python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-c5 > $O/${T}_ncu2.log 2>&1
summ ${T}_pcg_sw
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_iter1_s5p|k_iter23_s5" --launch-skip 60 -c 2 -o $O/${T}_pcg_s5 python bench_configs.py --config c5 --steps 1 --warmup 0 --max-iters 100 > $O/${T}_ncu3.log 2>&1
summ ${T}_pcg_s5
ls -la $O
