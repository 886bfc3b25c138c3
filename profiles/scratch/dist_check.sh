O=gpurun_out
export SG_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 --systems-per-gpu 32 > $O/r03_dist2.jsonl 2> $O/r03_dist2.err; echo rc=$? >> $O/r03_dist2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 --systems-per-gpu 32 > $O/r03_dist2_ref.jsonl 2> $O/r03_dist2_ref.err; echo rc=$? >> $O/r03_dist2_ref.err
