set -x
O=gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.limit,power.draw --format=csv > $O/r02_smi.txt
timeout 400 python bench.py > $O/r02_bench_c2.jsonl 2> $O/r02_bench_c2.err
timeout 400 python bench.py --impl reference --steps 1 --warmup 0 > $O/r02_bench_reference_arm.jsonl 2> $O/r02_ref.err
for c in c1 c3 c5; do timeout 400 python bench_configs.py --config $c >> $O/r02_bench_configs.jsonl 2>> $O/r02_cfg.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $O/r02_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02_ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_iter1_sw|k_iter23_sw" --launch-skip 300 -c 2 -o $O/r02_pcg_sw python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/r02_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_node_layer|k_edge_pass|k_node_encode" -c 3 -o $O/r02_gnn python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/r02_ncu3.log 2>&1
ls -la $O
