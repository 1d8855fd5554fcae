timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab9_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab9_pytest.log
bash tools/ab_run.sh "c4::st9" "c2::st9"
