#!/usr/bin/env bash
# ncu evidence for profiles/ (run on the GPU box, one GPU, after the same bench commands exited 0
# without ncu). Usage: tools/profile.sh <tag>. Reports stay in /tmp/ncu on the box; the raw and
# details pages (CSV) and the launch list come back in gpurun_out/.
set -u
TAG=${1:-r01}
OUT=gpurun_out
REP=/tmp/ncu
mkdir -p $OUT $REP
K='k_(t2_rows|t2_cols|w_sep|w_pair|pair_sigma|task_spmv|t1_cols|t1_rows)|k_cg_update|k_sb_post|k_stencil|k_cp_dual'
# launch list of the default bench (c2) inside the timed solve: cold-cache, serialised per-launch times
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" -s 600 -c 400 --csv \
    --log-file $OUT/${TAG}_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-other-configs > $OUT/${TAG}_launches_c2.log 2>&1
# one full capture of each kernel of one solver step per config
for c in c2 c3 c4 c5; do
  case $c in c4) skip=800; cnt=3;; c5) skip=40; cnt=9;; *) skip=60; cnt=8;; esac
  KK=$K; [ $c = c4 ] && KK='k_stencil|k_cg_update|k_sb_post'
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KK" -s $skip -c $cnt \
      -o $REP/${TAG}_full_$c python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline \
      > $OUT/${TAG}_full_$c.log 2>&1
  echo "$c rc=$?"
  ncu -i $REP/${TAG}_full_$c.ncu-rep --page raw --csv > $OUT/${TAG}_full_${c}_raw.csv 2>/dev/null
  ncu -i $REP/${TAG}_full_$c.ncu-rep --page details --csv > $OUT/${TAG}_full_${c}_details.csv 2>/dev/null
done
ls -la $OUT | tail -20
