timeout 900 python -m pytest tests -m gpu -x -q -k "c5 or cp or 8192 or chambolle or fft" > gpurun_out/ab11_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab11_pytest.log
bash tools/ab_run.sh "c5::split" "c5:TOMO_LIB_NAME=libtomo_nosplit.so:nosplit"
