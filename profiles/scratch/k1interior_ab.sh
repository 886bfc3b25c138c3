# A/B: 1-D K1 stencil regeneration without wall selects for interior rows (mask 0x1f)
# -- in-tree library -- vs the committed kernel (lib_base.so).
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r03m_pytest_gpu.log 2>&1; echo rc=$? >> $O/r03m_pytest_gpu.log
for v in new base new base; do
  if [ $v = base ]; then L=profiles/scratch/lib_base.so; else L=""; fi
  SG_LIB_PATH=$L timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-c5 >> $O/r03m_k1_c2_$v.jsonl 2>> $O/r03m_k1.err
done
