#!/usr/bin/env bash
# Baseline check on the GPU box: GPU tests, then quick bench lines for c2/c3/c1/c5/c4.
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
for c in ${CFGS:-c2 c3 c1 c5 c4}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/chk_$c.json 2> gpurun_out/chk_$c.err; echo "$c rc=$?"
done
