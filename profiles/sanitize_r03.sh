# compute-sanitizer over the streamed (bulk-copy / mbarrier ring) PCG kernels and the row partition.
O=gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
K='tests/test_gpu_parity.py::test_coefficient_stencil_k1_bit_identical tests/test_gpu_parity.py::test_sliding_window_two_chunk_halo tests/test_gpu_parity.py::test_pcg_wide_grid_strip_kernels'
timeout 1500 $S --tool racecheck --racecheck-report all python -m pytest $K -q -p no:cacheprovider > $O/r03_sanitize_racecheck.log 2>&1; echo rc=$? >> $O/r03_sanitize_racecheck.log
timeout 1500 $S --tool synccheck python -m pytest $K -q -p no:cacheprovider > $O/r03_sanitize_synccheck.log 2>&1; echo rc=$? >> $O/r03_sanitize_synccheck.log
timeout 1500 $S --tool memcheck python -m pytest $K "tests/test_gpu_rowpart.py::test_partitioned_solve_matches_whole_system" tests/test_gpu_rowpart.py::test_peer_mode_single_rank_runs_the_peer_reduction_path -q -p no:cacheprovider > $O/r03_sanitize_memcheck.log 2>&1; echo rc=$? >> $O/r03_sanitize_memcheck.log
