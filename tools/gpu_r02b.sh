# round-2 call B: config parity (c1-c5), the 2-rank sharded test, c2 bench + reference arm
export TOMO_PARITY_LOG=gpurun_out/parity_configs.jsonl
rm -f $TOMO_PARITY_LOG
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_sharded.py -q -s --durations=0 > gpurun_out/configs.log 2>&1; echo "configs rc=$?" >> gpurun_out/configs.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench rc=$?" >> gpurun_out/bench_c2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err; echo "ref rc=$?" >> gpurun_out/ref_c2.err
