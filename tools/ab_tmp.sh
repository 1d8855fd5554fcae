timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -p no:cacheprovider --deselect tests/test_gpu_configs.py::test_c5_apply_and_chambolle_pock > gpurun_out/par.log 2>&1; echo "rc=$?" >> gpurun_out/par.log
for c in c2 c3 c1 c5; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_new_$c.json 2>&1; done
