# r02 call F: c5 parity (new test), ncu captures of c2/c3 kernels (full set) + c2 launch list
export TOMO_PARITY_LOG=gpurun_out/parity_c5.jsonl; rm -f $TOMO_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_configs.py -k c5 -x -q -s > gpurun_out/c5.log 2>&1; echo "rc=$?" >> gpurun_out/c5.log
OUT=gpurun_out; REP=/tmp/ncu; mkdir -p $REP; TAG=r02a
K='k_(t2_rows|t2_cols|w_sep|task_spmv|t1_cols|t1_rows)|k_cg_update|k_cgcg_final|k_sb_post'
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" -s 600 -c 400 --csv \
    --log-file $OUT/${TAG}_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/${TAG}_launches_c2.log 2>&1
for c in c2 c3; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 60 -c 7 \
      -o $REP/${TAG}_full_$c python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > $OUT/${TAG}_full_$c.log 2>&1
  ncu -i $REP/${TAG}_full_$c.ncu-rep --page raw --csv > $OUT/${TAG}_full_${c}_raw.csv 2>/dev/null
  ncu -i $REP/${TAG}_full_$c.ncu-rep --page details --csv > $OUT/${TAG}_full_${c}_details.csv 2>/dev/null
  cp $REP/${TAG}_full_$c.ncu-rep $OUT/
done
