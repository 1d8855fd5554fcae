#!/bin/bash
# grid.y batching (BY template) check: GPU tests, c1/c2/c3 benches, then the r01k ncu captures
out=gpurun_out/ab17; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/gputests.log 2>&1; echo "tests exit $?" >> $out/gputests.log
for c in c1 c2 c3; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > $out/${c}.json 2> $out/${c}.err
done
TOMO_BATCH_Y=0 timeout 300 python bench.py --config c1 --no-cpu-baseline > $out/c1_y0.json 2> $out/c1_y0.err
bash tools/profile.sh r01k
