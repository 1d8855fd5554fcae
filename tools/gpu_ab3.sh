timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab3_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab3_pytest.log
bash tools/ab_run.sh "c2::half" "c3::half" "c1::half" "c4::half"
