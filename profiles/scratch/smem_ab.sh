O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -m gpu -q -p no:cacheprovider -k "control_flow or small or deferred or apply_time or golden or train" > $O/r03_smem_tests.log 2>&1; echo rc=$? >> $O/r03_smem_tests.log
for v in 1 0; do
  SG_PCG_SMEM=$v timeout 300 python bench_configs.py --config c1 --steps 3 --warmup 1 >> $O/r03_smem_c1_$v.jsonl 2>> $O/r03_smem.err
done
for nx in 16 32 48 64 96 128; do for v in 1 0; do
  SG_PCG_SMEM=$v timeout 400 python -c "
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
print('nx', $nx, 'smem', $v, 'k', rep.k, 'conv', rep.converged, 'ms', round(1000 * t, 2), 'us/iter', round(1e6 * t / rep.k, 2))
" >> $O/r03_smem_grid.txt 2>> $O/r03_smem.err
done; done
