# Round-end check on the GPU box: the whole GPU suite with the config-parity log, the default bench line + reference arm, smoke()
export TOMO_PARITY_LOG=gpurun_out/parity_configs.jsonl; rm -f $TOMO_PARITY_LOG
timeout 1800 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > gpurun_out/gpu_suite.log 2>&1; echo "suite rc=$?" >> gpurun_out/gpu_suite.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "rc=$?" >> gpurun_out/bench_c2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err; echo "rc=$?" >> gpurun_out/ref_c2.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
