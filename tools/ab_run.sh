# A/B of env-selected kernel variants (the knobs are honoured only with TOMO_AB=1, set here):
#   bash tools/ab_run.sh "<cfg>:<ENV=..,ENV=..>:<tag>[:<extra bench args, comma-separated>]" ...
for spec in "$@"; do
  IFS=: read c envs tag extra <<< "$spec"
  env TOMO_AB=1 $(echo $envs | tr ',' ' ') timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline \
    $(echo $extra | tr ',' ' ') > gpurun_out/ab_${tag}_$c.json 2> gpurun_out/ab_${tag}_$c.err
  echo "$c $tag rc=$?"
done
