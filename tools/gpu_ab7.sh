timeout 900 python -m pytest tests -m gpu -x -q -k "surrogate or stencil or c4 or sb or edge" > gpurun_out/ab7_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab7_pytest.log
bash tools/ab_run.sh "c4::st3"
