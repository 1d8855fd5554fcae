#!/usr/bin/env bash
# Round-2 bench lines for every BASELINE config (one GPU): our arm (device + e2e + roofline + CPU
# baseline on the box's host cores) and the reference arm, into gpurun_out/bench_<cfg>.json and
# gpurun_out/ref_<cfg>.json. Usage on the GPU box: bash tools/bench_all.sh [tag]
tag=${1:-r02}
for c in c2 c1 c3 c4 c5; do
  steps=20; warm=5
  [ $c = c5 ] && { steps=3; warm=3; }
  timeout 900 python bench.py --config $c --steps $steps --warmup $warm > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
  echo "$c ours rc=$?"
  rs=20; rw=5
  [ $c != c2 ] && { rs=5; rw=2; }
  timeout 900 python bench.py --config $c --impl reference --steps $rs --warmup $rw > gpurun_out/${tag}_ref_$c.json 2> gpurun_out/${tag}_ref_$c.err
  echo "$c reference rc=$?"
done
