timeout 900 python -m pytest tests -m gpu -x -q -k "parity or edge or fused" > gpurun_out/ab2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab2_pytest.log
bash tools/ab_run.sh "c2::tr" "c3::tr" "c1::tr" "c5::tr"
