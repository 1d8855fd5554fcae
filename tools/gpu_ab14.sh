timeout 900 python -m pytest tests -m gpu -x -q -k "parity" > gpurun_out/ab14_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab14_pytest.log
bash tools/ab_run.sh "c3::tws2" "c2::tws2" "c5::tws2"
