set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s1_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s1_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s1_smoke.log 2>&1; echo "smoke rc=$?"
for c in c2 c1 c3 c4 c5; do timeout 900 python bench.py --config $c > gpurun_out/s1_bench_$c.json 2> gpurun_out/s1_bench_$c.err; echo "$c rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s1_ref_c2.json 2>&1; echo "ref rc=$?"
