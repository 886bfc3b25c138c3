O=gpurun_out
for v in 3072 8192 3072 8192; do
  SG_PCG_SMALL_ROWS=$v timeout 400 python bench_configs.py --config c1 --steps 3 --warmup 1 >> $O/r03_small_$v.jsonl 2>> $O/r03_small.err
done
for nx in 96 128; do for v in 3072 20000; do
  SG_PCG_SMALL_ROWS=$v timeout 400 python -c "
import time, numpy as np, torch, paper_2510_27517_b200 as P
A, meta = P.gen_poisson2d($nx, $nx, coeff_seed=1)
m = P.init_model(P.GnnConfig(d_node=3, seed=0))
G = P.forward(m, P.build_graph(A, meta)).G
M = P.build_learned_spai(G, m.config.epsilon)
b = P.gen_rhs(meta, 5)
cfg = P.SolveConfig(rtol=1e-6)
rep = P.pcg_solve(A, b, M, cfg)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(3): rep = P.pcg_solve(A, b, M, cfg)
torch.cuda.synchronize(); t = (time.perf_counter() - t0) / 3
print('nx', $nx, 'small_rows', $v, 'k', rep.k, 'ms', round(1000 * t, 2), 'us/iter', round(1e6 * t / rep.k, 2))
" >> $O/r03_small_grid.txt 2>> $O/r03_small.err
done; done
