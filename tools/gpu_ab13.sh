timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab13_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ab13_pytest.log
bash tools/ab_run.sh "c3::tws1" "c3:TOMO_LIB_NAME=libtomo_notws.so:tws0" "c2::tws1" "c2:TOMO_LIB_NAME=libtomo_notws.so:tws0" "c5::tws1" "c1::tws1"
