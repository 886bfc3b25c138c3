# C5 through the row partition (group mode, 2 / 4 / 8 partitions on one GPU) on the final library.
O=gpurun_out
for p in 2 4 8; do timeout 400 python bench_configs.py --config c5 --parts $p --steps 3 >> $O/r03s3_bench_c5_parts.jsonl 2>> $O/r03s3_parts.err; done
