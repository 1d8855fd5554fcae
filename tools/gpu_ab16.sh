#!/bin/bash
# A/B: batched W / W^T slices across grid.y (TOMO_BATCH_Y) on c1 (calls of 20 on 3 lanes); GPU tests
out=gpurun_out/ab16; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/gputests.log 2>&1; echo "tests exit $?" >> $out/gputests.log
for v in 1 0; do
  TOMO_BATCH_Y=$v timeout 300 python bench.py --config c1 --no-cpu-baseline > $out/c1_y$v.json 2> $out/c1_y$v.err
done
TOMO_BATCH_Y=1 timeout 300 python bench.py --config c3 --no-cpu-baseline > $out/c3_y1.json 2> $out/c3_y1.err
