#!/usr/bin/env bash
# Hermitian half-grid path: its own equivalence tests, the full GPU suite, quick bench lines.
timeout 600 python -m pytest tests/test_gpu_herm.py -x -q -s -p no:cacheprovider > gpurun_out/herm_tests.log 2>&1; echo "herm rc=$?" >> gpurun_out/herm_tests.log
tail -3 gpurun_out/herm_tests.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
for c in ${CFGS:-c2 c5 c1 c3}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/h_$c.json 2> gpurun_out/h_$c.err; echo "$c rc=$?"
done
