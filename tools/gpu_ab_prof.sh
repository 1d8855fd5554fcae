#!/usr/bin/env bash
# A/B bench runs (ab_run.sh specs in $AB) followed by an ncu --set full capture of one solver step
# of each config in $PCFG (default c2): reports stay in /tmp/ncu on the box; the raw page (CSV) and
# the hot-instruction summary of each kernel come back in gpurun_out/.
TAG=${TAG:-r02b}
mkdir -p /tmp/ncu
[ -n "$AB" ] && bash tools/ab_run.sh $AB
for c in ${PCFG:-c2}; do
  case $c in c4) skip=800; cnt=3;; c5) skip=40; cnt=9;; *) skip=60; cnt=7;; esac
  K='k_(t2_rows|t2_cols|w_sep|task_spmv|t1_cols|t1_rows)|k_cg_update|k_sb_post|k_stencil'
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $skip -c $cnt \
      -o /tmp/ncu/${TAG}_full_$c python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline \
      > gpurun_out/${TAG}_full_$c.log 2>&1
  echo "ncu $c rc=$?"
  ncu -i /tmp/ncu/${TAG}_full_$c.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_${c}_raw.csv 2>/dev/null
  for k in k_t2_rows k_t2_cols k_w_sep k_task_spmv k_t1_cols k_t1_rows; do
    python tools/ncu_hot.py /tmp/ncu/${TAG}_full_$c.ncu-rep "$k" 25 > gpurun_out/${TAG}_hot_${c}_$k.txt 2>&1
  done
done
