#!/bin/bash
# same-box A/B: current library vs the previous commit's (libtomo_b200_head.so), c3 and c1, alternating
out=gpurun_out/ab18; mkdir -p $out
for r in 1 2; do
  for v in head cur; do
    lib=libtomo_b200.so; [ $v = head ] && lib=libtomo_b200_head.so
    for c in c3 c1; do
      TOMO_LIB_NAME=$lib timeout 300 python bench.py --config $c --no-cpu-baseline > $out/${c}_${v}_$r.json 2> $out/${c}_${v}_$r.err
    done
  done
done
timeout 600 python -m pytest tests -m gpu -x -q > $out/gputests.log 2>&1; echo "tests exit $?" >> $out/gputests.log
