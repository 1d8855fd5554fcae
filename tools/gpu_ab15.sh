#!/bin/bash
# A/B: fused W^T + PA (k_wt_t1) threads per CTA vs the two-kernel path (c2, c3, c1)
out=gpurun_out/ab15; mkdir -p $out
for c in c2 c3 c1; do
  for v in "1 512" "1 256" "1 1024" "0 512"; do
    set -- $v
    TOMO_WT_FUSE=$1 TOMO_WT_T1_THREADS=$2 timeout 300 python bench.py --config $c --no-cpu-baseline \
      > $out/${c}_f$1_t$2.json 2> $out/${c}_f$1_t$2.err
  done
done
