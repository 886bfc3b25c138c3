# Round-3 measurement script (one gpurun call): bench lines, configs, launch list, ncu captures.
# ncu reports are summarised on the box and deleted (gpurun brings back <= 64 MiB).
set -x
O=gpurun_out
summ() {  # $1 = report basename: raw metrics summary + details page, then drop the report
  python profiles/summarize_ncu.py $O/$1.ncu-rep > $O/$1_summary.txt 2>&1
  ncu -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>&1
  ncu -i $O/$1.ncu-rep --page source --csv --print-source sass > $O/$1_source.csv 2>&1
  gzip -f $O/$1_source.csv
  rm -f $O/$1.ncu-rep
}
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.limit,power.draw --format=csv > $O/r03_smi.txt
./profiles/micro/dmma_peak > $O/r03_dmma_peak.json 2>&1
timeout 600 python bench.py > $O/r03_bench_c2.jsonl 2> $O/r03_bench_c2.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/r03_bench_reference_arm.jsonl 2> $O/r03_ref.err
for c in c1 c3 c5; do timeout 400 python bench_configs.py --config $c >> $O/r03_bench_configs.jsonl 2>> $O/r03_cfg.err; done
for p in 2 4 8; do timeout 400 python bench_configs.py --config c5 --parts $p --steps 3 >> $O/r03_bench_c5_parts.jsonl 2>> $O/r03_cfg.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/r03_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-c5 > $O/r03_ncu1.log 2>&1
gzip -f $O/r03_launches.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_iter1_sw|k_iter23_sw" --launch-skip 300 -c 2 -o $O/r03_pcg_sw python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-c5 > $O/r03_ncu2.log 2>&1
summ r03_pcg_sw
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_iter1_s5|k_iter23_s5" --launch-skip 60 -c 2 -o $O/r03_pcg_s5 python bench_configs.py --config c5 --steps 1 --warmup 0 --max-iters 100 > $O/r03_ncu3.log 2>&1
summ r03_pcg_s5
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_node_layer|k_edge_pass|k_node_encode" -c 6 -o $O/r03_gnn python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-c5 > $O/r03_ncu4.log 2>&1
summ r03_gnn
ls -la $O
du -sh $O
