for c in c2 c1 c3 c4 c5; do timeout 900 python bench.py --config $c > gpurun_out/s2_bench_$c.json 2> gpurun_out/s2_bench_$c.err; echo "$c rc=$?"; done
