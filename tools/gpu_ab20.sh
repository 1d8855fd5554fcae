#!/bin/bash
# c1 call size x lanes sweep after the grid.y batching of W / W^T
out=gpurun_out/ab20; mkdir -p $out
for bl in "20 3" "25 2" "50 2" "50 3" "50 4" "100 3" "100 4" "34 3"; do
  set -- $bl
  TOMO_LANES=$2 timeout 300 python bench.py --config c1 --batch $1 --no-cpu-baseline > $out/c1_b$1_l$2.json 2> $out/c1_b$1_l$2.err
done
