# r02 call G: c5 parity (perturbation bound), c3 bench, GPU suite, c3 ncu capture
export TOMO_PARITY_LOG=gpurun_out/parity_c5.jsonl; rm -f $TOMO_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_configs.py -k c5 -x -q -s > gpurun_out/c5.log 2>&1; echo "rc=$?" >> gpurun_out/c5.log
timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "rc=$?" >> gpurun_out/bench_c3.err
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_configs.py::test_c5_apply_and_chambolle_pock > gpurun_out/gpu_suite.log 2>&1; echo "suite rc=$?" >> gpurun_out/gpu_suite.log
OUT=gpurun_out; REP=/tmp/ncu; mkdir -p $REP; TAG=r02a
K='k_(t2_rows|t2_cols|w_sep|task_spmv|t1_cols|t1_rows)|k_cg_update|k_cgcg_final|k_sb_post'
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 60 -c 7 \
      -o $REP/${TAG}_full_c3 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > $OUT/${TAG}_full_c3.log 2>&1
ncu -i $REP/${TAG}_full_c3.ncu-rep --page raw --csv > $OUT/${TAG}_full_c3_raw.csv 2>/dev/null
ncu -i $REP/${TAG}_full_c3.ncu-rep --page details --csv > $OUT/${TAG}_full_c3_details.csv 2>/dev/null
cp $REP/${TAG}_full_c3.ncu-rep $OUT/
