O=gpurun_out
summ() {
  python profiles/summarize_ncu.py $O/$1.ncu-rep > $O/$1_summary.txt 2>&1
  ncu -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>&1
  ncu -i $O/$1.ncu-rep --page source --csv --print-source sass > $O/$1_source.csv 2>&1
  gzip -f $O/$1_source.csv
  rm -f $O/$1.ncu-rep
}
for v in new xd0 pg3 ld pg3ld new xd0 pg3 ld pg3ld; do
  if [ $v = new ]; then L=""; else L=profiles/scratch/lib_$v.so; fi
  SG_LIB_PATH=$L timeout 400 python bench_configs.py --config c5 --steps 3 --warmup 1 >> $O/r03_blk2_$v.jsonl 2>> $O/r03_blk2.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_iter1_s5|k_iter23_s5" --launch-skip 60 -c 2 -o $O/r03_pcg_s5blk python bench_configs.py --config c5 --steps 1 --warmup 0 --max-iters 100 > $O/r03_ncu5.log 2>&1
summ r03_pcg_s5blk
