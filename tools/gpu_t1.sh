timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "long_rows" --durations=5 > gpurun_out/t1_pytest.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/t1_pytest.log
