# bench sweep helper: tools/gpu_sweep.sh <config> "<batch list>" [extra bench args]; one JSON line per batch
cfg=$1; shift; batches=$1; shift
for b in $batches; do
  timeout 600 python bench.py --config $cfg --batch $b --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/sweep_${cfg}_b$b.json 2> gpurun_out/sweep_${cfg}_b$b.err
done
